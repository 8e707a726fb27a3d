#!/usr/bin/env python
"""TUSQ hot-path benchmark (BASELINE.json metric: noisy-sim wall s per circuit, 30q Adder; gate HBM GB/s).

One step = one pass of the whole hot path over one batch: the ECM + tree (a1-a6, host, the full
circuit) and the DFS traversal of the next B leaves of this rank's DFS range with uncompute /
re-anchor, fused gate sweeps and leaf sampling (a7-a10, device).  `value` is the projected wall
seconds per circuit: ECM seconds + (this rank's total algorithmic bytes from the exact host plan)
/ (bytes per second measured over the timed steps), max over ranks.  `--full` runs every leaf of
every rank's range inside the timed region instead (no projection).

Launch: python bench.py --gpus N --steps K --warmup W   (N > 1 under torch.distributed.run)
        python bench.py --impl reference ...              (the CPU oracle on host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import circuits as W  # noqa: E402

METRIC = "noisy-sim wall s per circuit (30q Adder) at 1/2/4/8 B200; gate HBM GB/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, idx: int):
        self.idx, self.rows, self.stop = idx, [], threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_oracle_rate(cfg, max_seconds: float = 20.0):
    """Time the oracle (as it stands) applying gates of leaf 0 at the config's size on the host cores.
    Returns (seconds per gate application, cores, sample description)."""
    import numpy as np
    from oracle import oracle as O
    n = cfg.n
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    nn = n
    while (16 << nn) * 1.5 > avail and nn > 20:
        nn -= 1
    st = np.zeros(1 << nn, dtype=np.complex128)
    st[0] = 1
    ops = [g for g in cfg.ops if max(g[1], g[2] if g[0] in W.TWO_QUBIT else 0) < nn] or cfg.ops
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < max_seconds and k < len(ops):
        O.apply_gate(st, nn, ops[k])
        k += 1
    dt = (time.perf_counter() - t0) / max(k, 1) * (1 << (n - nn))
    del st
    desc = (f"oracle or_apply_gate on {k} gates of the {cfg.name} circuit at {nn} qubits"
            + (f" (scaled x2^{n - nn} to {n} qubits: host RAM)" if nn < n else "")
            + "; seconds per gate application x the oracle's naive gate count (each leaf replayed from |0..0>)")
    return dt, cores, desc


def workload_desc(cfg) -> str:
    nz = cfg.noise
    kind = "Cuccaro adder" if cfg.name in ("C1", "C3", "C4") else ("GHZ" if cfg.name == "C2a" else "QFT")
    return (f"{cfg.name}: {cfg.n}q {kind} (L={len(cfg.ops)}), depolarizing p1={nz.p1} p2={nz.p2}"
            + (f" p_meas={nz.p_meas}" if nz.p_meas else "") + f", {cfg.shots} shots, seed {cfg.seed}, alpha 1/100, beta 100")


def ncu_traffic(prec, no_fuse):
    """DRAM bytes per k_fused launch from the committed ncu --set full capture of this bench (c128)."""
    path = os.path.join(ROOT, "profiles", "r1_ncu_k_fused_in_bench.json")
    if no_fuse or prec != 128 or not os.path.exists(path):
        return None
    try:
        caps = json.load(open(path))["full_capture"]
        return caps[0].get("dram_traffic_bytes")
    except (OSError, ValueError, KeyError, IndexError):
        return None


def run_reference(args, rank, world):
    """The CPU oracle (test infrastructure) timed on the host cores on this workload."""
    if rank != 0:
        return
    cfg = W.config(args.config)
    from oracle import oracle as O
    O.build()
    t0 = time.perf_counter()
    tree = O.Tree.from_config(cfg)
    t_ecm = time.perf_counter() - t0
    naive = sum(len(cfg.ops) + len(tree.leaf(l)[0]) for l in range(tree.n_leaves))
    per, cores, desc = None, None, None
    times = []
    for s in range(args.warmup + args.steps):
        per, cores, desc = cpu_oracle_rate(cfg, max_seconds=args.cpu_seconds / 2)
        if s >= args.warmup:
            times.append(per)
    per = sorted(times)[len(times) // 2]
    value = t_ecm + per * naive
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "extrapolated": True,
                       "projection": "oracle ECM s + (oracle s per gate application) x naive gate applications"},
            "cpu_baseline": {"value": value, "unit": "s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tusq", choices=["tusq", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--precision", type=int, default=128, choices=[128, 64])
    ap.add_argument("--leaves-per-step", type=int, default=0)
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="replica", choices=["replica", "sharded"],
                    help="sharded: amplitudes split over the N ranks by global qubits (e.g. --config C5 on 8 GPUs)")
    ap.add_argument("--shards", type=int, default=0,
                    help="sharded mode on ONE GPU: this many shards driven by one process (local communicator)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_04880_b200 as T

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.config(args.config)
    nz = cfg.noise
    n = cfg.n
    prec = args.precision

    # ---- ECM + tree (host): timed on the host clock (it is host work)
    t0 = time.perf_counter()
    tree = T.build_error_tree(n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    t_ecm = time.perf_counter() - t0
    info = tree.info()
    flags = T.EXEC_PROFILE | (T.EXEC_NO_FUSE if args.no_fuse else 0)
    dt = torch.complex128 if prec == 128 else torch.complex64
    comm = None
    nshards = 0
    if args.mode == "sharded":
        # every rank runs every leaf on its 2^(n-g) shard; the host plan is the same on all ranks
        if world > 1:
            from paper_2508_04880_b200 import dist as D
            comm, _ = D.make_sharded_comm(local)
            nshards = world
            state = torch.empty(1 << (n - (world.bit_length() - 1)), dtype=dt, device="cuda")
        else:
            # one GPU: all shards in this process (the local communicator; exchanges are device swaps)
            nshards = args.shards or 2
            comm = T.Comm.local(nshards)
            state = torch.empty(1 << n, dtype=dt, device="cuda")
        lb, le = 0, info["n_leaves"]
        _, plan = T.run_tree(tree, prec, flags=flags | T.EXEC_PLAN_ONLY, comm=T.Comm.local(nshards))
    else:
        bounds = tree.partition(world, prec)
        lb, le = int(bounds[rank]), int(bounds[rank + 1])
        _, plan = T.run_tree(tree, prec, leaf_begin=lb, leaf_end=le, flags=flags | T.EXEC_PLAN_ONLY)
        state = torch.empty(1 << n, dtype=dt, device="cuda")
    plan_bytes = plan["hbm_bytes"] + plan["sample_bytes"]
    stream = torch.cuda.current_stream()
    nleaf = max(le - lb, 1)
    B = args.leaves_per_step or max(1, min(nleaf, (16 if comm is not None else 64) if n >= 28 else 256))
    slots = np.zeros(cfg.shots, dtype=np.uint64)

    # batches spread evenly over the rank's DFS range (the cost of a transition depends on where
    # in the tree it is: early DFS leaves diverge late in the circuit); each batch starts with a
    # re-anchor.  Warm-up batches come from the same spread, interleaved.
    nb_total = args.warmup + (1 if args.full else args.steps)
    stride = max(1, nleaf // max(nb_total, 1))

    def step(s, full=False):
        b = lb if full else lb + (s * stride) % nleaf
        e = le if full else min(b + B, le)
        _, st = T.run_tree(tree, prec, d_state=state, stream=stream, leaf_begin=b, leaf_end=e, flags=flags,
                           out_slots=slots, comm=comm)
        return st

    order = list(range(nb_total))
    warm, timed = order[1::2][:args.warmup], [s for s in order if s not in order[1::2][:args.warmup]]
    for s in warm:
        step(s)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        w0 = time.perf_counter()
        ev0.record(stream)
        for s in ([0] if args.full else timed[:args.steps]):
            stats.append(step(s, args.full))
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    if world > 1:
        dist.barrier()
    t_dev = ev0.elapsed_time(ev1) / 1e3
    tot = {k: sum(st[k] for st in stats) for k in stats[0]}
    done_bytes = tot["hbm_bytes"] + tot["sample_bytes"]
    rate = done_bytes / t_dev
    proj = t_dev if args.full else plan_bytes / rate
    proj_wall = wall if args.full else plan_bytes / (done_bytes / wall)
    # max over ranks
    vals = torch.tensor([proj, proj_wall, t_dev], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    proj, proj_wall, t_dev_max = [float(x) for x in vals.cpu()]
    value = t_ecm + proj
    hbm_peak, peak_src = peaks()
    gk_s, gk_b, gk_n = tot["gate_kernel_seconds"], tot["gate_kernel_bytes"], tot["gate_kernel_launches"]
    achieved = gk_b / gk_s / 1e9 if gk_s > 0 else None
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
        "steps": 1 if args.full else args.steps, "warmup": args.warmup,
        "ms_per_step": t_dev_max * 1e3 / (1 if args.full else args.steps),
        "higher_is_better": False, "scaling": "strong" if args.full else "weak", "vs_baseline": None,
        "dtype": "c128" if prec == 128 else "c64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg),
                   "leaves": info["n_leaves"], "leaves_per_step": B, "rank_leaves": [lb, le],
                   "extrapolated": not args.full,
                   "projection": "ECM s + rank plan bytes / measured bytes-per-s over the timed steps (max over ranks)",
                   "ecm_s": t_ecm, "gpu_projected_s": proj, "plan_sweeps": plan["sweeps"],
                   "plan_gate_apps": plan["gate_apps"], "plan_hbm_GB": plan_bytes / 1e9,
                   "dftt_ops": info["dftt_ops"], "naive_ops": info["naive_ops"],
                   "l2": f"state {state.numel() * state.element_size() / 2**30:.0f} GiB >> 126 MB L2 (no flush needed)",
                   "fused": not args.no_fuse,
                   "parallelism": (f"sharded x{nshards} over {world} GPU(s): amplitudes split by "
                                   f"{nshards.bit_length() - 1} global qubits, half-shard exchanges "
                                   + ("(NCCL)" if world > 1 else "(local communicator, device swaps)")
                                   if comm is not None
                                   else f"replica x{world}, contiguous DFS leaf ranges")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": (achieved / hbm_peak) if achieved else None, "traffic": ncu_traffic(prec, args.no_fuse),
                     "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of one k_fused launch of this "
                                       "bench under ncu --set full (profiles/r1_ncu_k_fused_in_bench.json)",
                     "kernel": "k_fused (K5)" if not args.no_fuse else "K1-K4",
                     "launches_timed": gk_n, "bytes_per_launch": gk_b / max(gk_n, 1),
                     "avg_launch_ms": gk_s / max(gk_n, 1) * 1e3, "peak_source": peak_src,
                     "step_share": gk_s / t_dev if t_dev > 0 else None},
        "e2e": {"value": t_ecm + proj_wall, "unit": "s", "h2d_bytes_per_step": 24 * len(cfg.ops),
                "d2h_bytes_per_step": int(8 * sum(st["draws"] for st in stats) / len(stats)),
                "note": "public API (build_error_tree + run_tree, host out_slots) on the host clock"},
        "gpu_launches": int(tot["launches"]),
        "clocks": clk.summary(),
        "stats": {k: tot[k] for k in ("leaves", "resets", "gate_apps", "sweeps", "draws", "edge_draws",
                                      "fused_launches", "exchanges")},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        per, cores, desc = cpu_oracle_rate(cfg, args.cpu_seconds)
        v = per * info["naive_ops"]
        line["cpu_baseline"] = {"value": v, "unit": "s", "cores": cores, "kind": "oracle", "sample": desc,
                                "extrapolated": True}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
