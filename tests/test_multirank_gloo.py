"""World-size-2 gloo test of the replica multi-GPU path on CPU: identical trees on both ranks,
contiguous cost-balanced leaf ranges, and the SUM reduction of disjoint slot arrays reproducing
the single-rank result bit for bit.  The device run of each range is stood in for by the oracle
(test infrastructure) because this container has no GPU; the GPU tests cover run_tree itself."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from workloads import circuits as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_dir, real=False):
    import torch.distributed as dist

    import paper_2508_04880_b200 as T
    from oracle import oracle as O
    from paper_2508_04880_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = W.config(name)
    nz = cfg.noise
    tree = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    ot = O.Tree.from_config(cfg)

    def run_range(b, e):
        out = np.zeros(cfg.shots, dtype=np.uint64)
        if real:   # the library's own tusq_run_tree on cuda:0 (both ranks share the device)
            if e > b:
                T.run_tree(tree, 128, leaf_begin=b, leaf_end=e, out_slots=out)
            return out
        for l in range(b, e):
            _, cnt, off = ot.leaf(l)
            k, _ = ot.sample_leaf(ot.replay_leaf_core(l), l)
            out[off:off + cnt] = k
        return out

    slots, (lb, le) = D.run_tree_distributed(tree, run_range=run_range, device="cpu")
    np.save(os.path.join(out_dir, f"slots{rank}.npy"), slots)
    np.save(os.path.join(out_dir, f"range{rank}.npy"), np.array([lb, le]))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C2a", "C3"])
def test_gloo_world2_real_run_tree(tmp_path, oracle_runs, name):
    # both ranks run the real tusq_run_tree on cuda:0 over their tusq_tree_partition ranges; the gloo
    # SUM of the disjoint slot arrays equals the single-rank library run and the oracle (non-edge)
    port = _free_port()
    mp.spawn(_worker, args=(2, port, name, str(tmp_path), True), nprocs=2, join=True)
    s0, s1 = np.load(tmp_path / "slots0.npy"), np.load(tmp_path / "slots1.npy")
    r0, r1 = np.load(tmp_path / "range0.npy"), np.load(tmp_path / "range1.npy")
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] > r1[0]
    assert np.array_equal(s0, s1)
    import paper_2508_04880_b200 as T
    cfg = W.config(name)
    nz = cfg.noise
    tree = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    single, _ = T.run_tree(tree, 128)
    assert np.array_equal(s0, single)
    ref, edge = oracle_runs.run(name) if name != "C3" else oracle_runs.sparse_run(name)
    assert int(edge.sum()) <= max(3, cfg.shots // 1000)
    assert ((s0 != ref) & ~edge).sum() == 0


@pytest.mark.parametrize("name", ["C1", "C2a"])
def test_gloo_world2_matches_single_rank(tmp_path, oracle, name):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, name, str(tmp_path)), nprocs=2, join=True)
    s0 = np.load(tmp_path / "slots0.npy")
    s1 = np.load(tmp_path / "slots1.npy")
    r0, r1 = np.load(tmp_path / "range0.npy"), np.load(tmp_path / "range1.npy")
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] > r1[0]
    assert np.array_equal(s0, s1)
    ref, _ = oracle.Tree.from_config(W.config(name)).run()
    assert np.array_equal(s0, ref)


def _sharded_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2508_04880_b200 as T
    from paper_2508_04880_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the NCCL unique id travels over the process group (a stand-in id: no GPU/NCCL here)
    uid = D.share_unique_id(unique_id=lambda: bytes(range(128)))
    # every rank's sharded host plan is identical (deterministic, no communication)
    cfg = W.config("C2b")
    nz = cfg.noise
    tree = T.build_error_tree(cfg.n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    _, st = T.run_tree(tree, 128, flags=T.EXEC_PLAN_ONLY, comm=T.Comm.local(world))
    np.save(os.path.join(out_dir, f"uid{rank}.npy"), np.frombuffer(uid, dtype=np.uint8))
    np.save(os.path.join(out_dir, f"plan{rank}.npy"), np.array([st["exchanges"], st["gate_apps"], st["hbm_bytes"]]))
    # without a GPU the NCCL communicator must fail loudly (no silent fallback)
    try:
        T.Comm.nccl(uid, world, rank, 0)
        ok = 1
    except T.TusqError:
        ok = 0
    np.save(os.path.join(out_dir, f"nccl{rank}.npy"), np.array([ok]))
    dist.destroy_process_group()


def test_gloo_world2_sharded_plumbing(tmp_path, oracle):
    port = _free_port()
    mp.spawn(_sharded_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    u0, u1 = np.load(tmp_path / "uid0.npy"), np.load(tmp_path / "uid1.npy")
    assert np.array_equal(u0, u1) and np.array_equal(u0, np.arange(128, dtype=np.uint8))
    p0, p1 = np.load(tmp_path / "plan0.npy"), np.load(tmp_path / "plan1.npy")
    assert np.array_equal(p0, p1) and p0[0] > 0
    assert np.load(tmp_path / "nccl0.npy")[0] == 0 and np.load(tmp_path / "nccl1.npy")[0] == 0
