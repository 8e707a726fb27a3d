import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path through the C ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


class _OracleRuns:
    """Session cache of full oracle runs (slots, edge flags) and trees per config: the oracle's
    C2b run replays 7968 dense leaves and several GPU tests compare against it."""

    def __init__(self, O):
        self.O, self.trees, self.runs = O, {}, {}

    def tree(self, name):
        if name not in self.trees:
            from workloads import circuits as W
            self.trees[name] = self.O.Tree.from_config(W.config(name))
        return self.trees[name]

    def run(self, name):
        if name not in self.runs:
            self.runs[name] = self.tree(name).run()
        return self.runs[name]

    def sparse_run(self, name, eps=1e-9):
        """Full-run slots of an Adder config from the oracle's sparse replay (oracle/sparse.py,
        pinned to the dense oracle): each leaf's core replayed, sampled, XORed with its readout mask;
        eps = the edge-draw window (1e-9 for c128, 1e-5 for c64, DESIGN reading #17)."""
        key = ("sparse", name, eps)
        if key not in self.runs:
            import numpy as np
            from oracle import sparse as SP
            from workloads import circuits as W
            cfg = W.config(name)
            ot = self.tree(name)
            ref = np.zeros(cfg.shots, dtype=np.uint64)
            edge = np.zeros(cfg.shots, dtype=bool)
            for l in range(ot.n_leaves):
                tr, cnt, off = ot.leaf(l)
                psi = SP.replay(cfg.ops, SP.core_triples(tr, len(cfg.ops)), drop_below=1e-14)
                k, e = SP.sample(psi, cfg.seed, l, cnt, eps, ot.terminal_mask(l))
                ref[off:off + cnt], edge[off:off + cnt] = k, e
            self.runs[key] = (ref, edge)
        return self.runs[key]


@pytest.fixture(scope="session")
def oracle_runs(oracle):
    return _OracleRuns(oracle)


def edge_budget(draws: int) -> int:
    """Most edge draws (excluded from slot parity) a c128 slot test may see: a broken edge flag
    would otherwise make every slot comparison vacuous."""
    return max(3, draws // 1000)


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run under gpurun)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
