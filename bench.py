#!/usr/bin/env python
"""TUSQ hot-path benchmark (BASELINE.json metric: noisy-sim wall s per circuit, 30q Adder; gate HBM GB/s).

The measured quantity is ONE WHOLE CIRCUIT (C4 by default: 30-qubit noisy Adder, 8192 shots):
the ECM + tree (a1-a6, host) and then the DFS traversal of EVERY leaf (a7-a10, device) -- uncompute /
re-anchor, fused gate sweeps, leaf sampling -- with, for N > 1, the slot reduction over the ranks.
A "step" is one contiguous, cost-balanced batch of this rank's DFS range: --steps K batches cover
the whole range (each continues the DFS state of the previous one), so
    value = ecm_s + (device seconds of the K timed steps + the reduction), max over ranks
is the measured wall time of one circuit -- nothing is projected.  Warm-up runs W short separate
batches first.  After the timed region an untimed PROFILE pass (per-launch CUDA events) over a few
short batches gives the K5 per-launch time behind `roofline` and the stage shares.

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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
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
            self.stop.wait(0.5)

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


def workload_desc(cfg) -> str:
    nz = cfg.noise
    kind = "Cuccaro adder" if cfg.name in ("C1", "C3", "C4") else ("GHZ" if cfg.name == "C2a" else "QFT")
    return (f"{cfg.name}: {cfg.n}q {kind} (L={len(cfg.ops)}), depolarizing p1={nz.p1} p2={nz.p2}"
            + (f" p_meas={nz.p_meas}" if nz.p_meas else "") + f", {cfg.shots} shots, seed {cfg.seed}, alpha 1/100, beta 100")


def config_dict(cfg, prec, world):
    """The config both arms report (identical keys and values for the same workload)."""
    return {"workload": workload_desc(cfg), "precision": f"c{prec}", "shots": cfg.shots,
            "l2": f"state {(16 if prec == 128 else 8) * 2 ** cfg.n / 2 ** 30:.0f} GiB >> 126 MB L2 (no flush needed)",
            "parallelism": f"replica x{world}, cost-balanced DFS leaf chunks (interleaved over the ranks)"}


def cpu_oracle_rate(cfg, max_seconds: float = 20.0):
    """Time the oracle (as it stands) applying gates of the circuit at the config's size on the host
    cores.  Returns (seconds per gate application, cores, sample description)."""
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


def ncu_traffic(prec):
    """DRAM bytes of one DENSE k_fused sweep (2 x 2^30 x 16 B algorithmic) from the committed
    ncu --set full capture (c128): traffic ~= algorithmic means no wasted re-reads."""
    for name in ("r2_ncu_k_fused_dense.json", "r1_ncu_k_fused_in_bench.json"):
        path = os.path.join(ROOT, "profiles", name)
        if prec != 128 or not os.path.exists(path):
            continue
        try:
            caps = json.load(open(path))["full_capture"]
            return caps[0].get("dram_traffic_bytes"), f"profiles/{name}"
        except (OSError, ValueError, KeyError, IndexError):
            continue
    return None, None


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
        per, cores, desc = cpu_oracle_rate(cfg, max_seconds=args.cpu_seconds / 4)
        if s >= args.warmup:
            times.append(per)
    per = sorted(times)[len(times) // 2]
    value = t_ecm + per * naive
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": f"c{args.precision}", "data": "synthetic",
            "config": config_dict(cfg, args.precision, world),
            "extrapolated": True,
            "projection": "oracle ECM s + (oracle s per gate application) x naive gate applications",
            "cpu_baseline": {"value": value, "unit": "s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def dense_line(ptot, peak):
    """The dense K5 sweeps of the profile pass (every tile of a fully valid state: 2 x 2^n x s bytes)."""
    if not ptot or not ptot.get("dense_sweep_launches"):
        return None
    a = ptot["dense_sweep_bytes"] / ptot["dense_sweep_seconds"] / 1e9
    return {"launches": int(ptot["dense_sweep_launches"]),
            "avg_ms": ptot["dense_sweep_seconds"] / ptot["dense_sweep_launches"] * 1e3,
            "achieved": a, "frac": a / peak,
            "share_of_K5_time": ptot["dense_sweep_seconds"] / max(ptot["gate_kernel_seconds"], 1e-12)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tusq", choices=["tusq", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--precision", type=int, default=128, choices=[128, 64])
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--no-live", action="store_true",
                    help="plain dense path: no live tiles / valid sets / sums-only sampling (TUSQ_EXEC_NO_LIVE)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-leaves", type=int, default=100,
                    help="leaves per slice of the untimed per-launch profile pass (8 slices spread over the range)")
    ap.add_argument("--mode", default="replica", choices=["replica", "sharded"],
                    help="sharded: amplitudes split over the N ranks by global qubits (e.g. --config C5 on 8 GPUs)")
    ap.add_argument("--shards", type=int, default=0,
                    help="sharded mode on ONE GPU: this many shards driven by one process (local communicator)")
    ap.add_argument("--leaves", type=int, default=0,
                    help="sharded mode only: time the first this-many DFS leaves (C5 at full size is ~16 GPU-hours)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.mode == "sharded":
        return run_sharded(args, rank, world, local)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_04880_b200 as T

    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2508_04880_b200 import dist as D
        comm, _ = D.make_comm(local)
    cfg = W.config(args.config)
    nz = cfg.noise
    n = cfg.n
    prec = args.precision
    K = max(1, args.steps)
    flags = (T.EXEC_NO_FUSE if args.no_fuse else 0) | (T.EXEC_NO_LIVE if args.no_live else 0)
    dt = torch.complex128 if prec == 128 else torch.complex64
    state = torch.empty(1 << n, dtype=dt, device="cuda")
    stream = torch.cuda.current_stream()
    slots = np.zeros(cfg.shots, dtype=np.uint64)

    # ---- warm-up: W short separate batches (untimed), ECM included
    tree = T.build_error_tree(n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    nl = tree.n_leaves
    for w in range(args.warmup):
        b = (w * 997) % max(nl - 8, 1)
        T.run_tree(tree, prec, d_state=state, stream=stream, leaf_begin=b, leaf_end=min(b + 8, nl), flags=flags,
                   out_slots=np.zeros(cfg.shots, dtype=np.uint64))
    del tree
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed: ECM (host) + K contiguous batches of this rank's range + the reduction
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    stats = []
    with Clocks(local) as clk:
        w0 = time.perf_counter()
        tree = T.build_error_tree(n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
        t_ecm = time.perf_counter() - w0
        # world * K cost-balanced chunks in DFS order; rank r takes chunks r, r + world, ... (interleaved:
        # the partition balances gate applications, while device time follows the full sweeps, which
        # cluster in DFS order -- interleaving spreads them over the ranks).  One rank: contiguous.
        bounds = tree.partition(world * K, prec)
        batches = [(int(bounds[s * world + rank]), int(bounds[s * world + rank + 1])) for s in range(K)]
        ev[0].record(stream)
        for s, (b, e) in enumerate(batches):
            cont = s > 0 and batches[s - 1][1] == b   # continue the DFS state only across contiguous batches
            _, st = T.run_tree(tree, prec, d_state=state, stream=stream, leaf_begin=b, leaf_end=e,
                               flags=flags | (T.EXEC_CONTINUE if cont else 0), out_slots=slots)
            stats.append(st)
        ev[1].record(stream)
        if comm is not None:
            ev[2].record(stream)
            T.reduce_slots(comm, slots, stream)
            ev[3].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    t_dev = ev[0].elapsed_time(ev[1]) / 1e3
    t_red = ev[2].elapsed_time(ev[3]) / 1e3 if comm is not None else 0.0
    tot = {k: sum(st[k] for st in stats) for k in stats[0]}
    vals = torch.tensor([t_ecm + t_dev + t_red, wall, t_dev, t_red], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    value, wall_max, t_dev_max, t_red_max = [float(x) for x in vals.cpu()]
    info = tree.info()

    # ---- untimed profile pass: per-launch CUDA events over 8 slices spread evenly over the range
    # (slices of ~100 leaves: the per-call fixed work stays ~1 % of a slice's device time)
    lb, le = batches[0][0], batches[-1][1]
    prof = []
    for frac in [(i + 0.5) / 8 for i in range(8)]:
        b = lb + int((le - lb) * frac)
        e = min(le, b + args.profile_leaves)
        if e > b:
            _, st = T.run_tree(tree, prec, d_state=state, stream=stream, leaf_begin=b, leaf_end=e,
                               flags=flags | T.EXEC_PROFILE, out_slots=np.zeros(cfg.shots, dtype=np.uint64))
            prof.append(st)
    ptot = {k: sum(st[k] for st in prof) for k in prof[0]} if prof else None
    hbm_peak, peak_src = peaks()
    achieved = share_gate = share_sample = None
    if ptot and ptot["gate_kernel_seconds"] > 0:
        achieved = ptot["gate_kernel_bytes"] / ptot["gate_kernel_seconds"] / 1e9
        share_gate = ptot["gate_kernel_seconds"] / ptot["device_seconds"]
        share_sample = ptot["sample_kernel_seconds"] / ptot["device_seconds"]
    # the same kernel's rate inside the timed steps: its bytes / (its profile share x step time)
    in_step = (tot["hbm_bytes"] / (share_gate * t_dev) / 1e9) if share_gate else None
    traffic, traffic_src = ncu_traffic(prec)
    n_launch = ptot["gate_kernel_launches"] if ptot else 0
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": t_dev_max * 1e3 / K,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": f"c{prec}", "data": "synthetic",
        "config": config_dict(cfg, prec, world),
        "extrapolated": False,
        "measured": "ECM + every DFS leaf of every rank (K contiguous batches) + slot reduction, max over ranks",
        "stages": {"ecm_s": t_ecm, "device_s": t_dev_max, "reduce_s": t_red_max,
                   "traversal_s": share_gate * t_dev_max if share_gate else None,
                   "sampling_s": share_sample * t_dev_max if share_sample else None,
                   "note": "traversal/sampling = device_s x the gate/sampler kernel shares of the profile pass"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": (achieved / hbm_peak) if achieved else None, "traffic": traffic,
                     "traffic_source": (f"dram__bytes_read.sum + dram__bytes_write.sum of one dense k_fused sweep "
                                        f"(algorithmic 2 x 2^n x 16 B) under ncu --set full ({traffic_src})")
                     if traffic_src else None,
                     "kernel": "k_fused (K5)" if not args.no_fuse else "K1-K4",
                     "per_unit": ("one fused sweep = 2 x 2^n x 16 B over every tile it visits: a live-tile sweep "
                                  "(after a reset) moves 2 x its live tiles x 64 KiB, a reset sweep writes one tile, "
                                  "the first sweep on a partly valid state writes 2^n x 16 B and reads its valid "
                                  "elements (DESIGN.md 'Live tiles')"),
                     "launches_profiled": n_launch,
                     "bytes_per_launch": ptot["gate_kernel_bytes"] / max(n_launch, 1) if ptot else None,
                     "avg_launch_ms": ptot["gate_kernel_seconds"] / max(n_launch, 1) * 1e3 if ptot else None,
                     "achieved_in_timed_steps": in_step, "frac_in_timed_steps": in_step / hbm_peak if in_step else None,
                     "step_share": share_gate, "peak_source": peak_src,
                     "dense_sweeps": dense_line(ptot, hbm_peak)},
        "e2e": {"value": wall_max, "unit": "s",
                "h2d_bytes_per_step": int(tot["h2d_bytes"] / K), "d2h_bytes_per_step": int(tot["d2h_bytes"] / K),
                "note": "host clock around build_error_tree + every run_tree call (host op list in, host slots out) "
                        "+ the slot reduction; h2d = kernel parameter blocks + draw tables, d2h = slots + counters"},
        "gpu_launches": int(tot["launches"]),
        "clocks": clk.summary(),
        "stats": {"leaves": int(tot["leaves"]), "draws": int(tot["draws"]), "edge_draws": int(tot["edge_draws"]),
                  "sampled_vectors": int(tot["sampled_vectors"]), "resets": int(tot["resets"]),
                  "gate_apps": int(tot["gate_apps"]), "sweeps": int(tot["sweeps"]),
                  "fused_launches": int(tot["fused_launches"]), "hbm_GB": tot["hbm_bytes"] / 1e9,
                  "tree_leaves": info["n_leaves"], "dftt_ops": info["dftt_ops"], "naive_ops": info["naive_ops"],
                  "rank_leaves": int(sum(e - b for b, e in batches))},
    }
    line["path"] = ("dense state-vector path (TUSQ_EXEC_NO_LIVE: every sweep visits the whole state)" if args.no_live
                    else "live tiles + valid sets + sums-only sampling (DESIGN.md)")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        per, cores, desc = cpu_oracle_rate(cfg, args.cpu_seconds)
        line["cpu_baseline"] = {"value": per * info["naive_ops"], "unit": "s", "cores": cores, "kind": "oracle",
                                "sample": desc, "extrapolated": True}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        comm.free()
        dist.destroy_process_group()


def run_sharded(args, rank, world, local):
    """Sharded mode: the first --leaves DFS leaves of C5-size states, amplitudes split by
    global qubits over N ranks (or --shards local shards on one GPU).  A full C5 circuit is ~16
    GPU-hours, so this line times a leaf prefix and is labelled as such (not the headline)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_04880_b200 as T

    torch.cuda.set_device(local)
    cfg = W.config(args.config)
    nz = cfg.noise
    n, prec = cfg.n, args.precision
    dt = torch.complex128 if prec == 128 else torch.complex64
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2508_04880_b200 import dist as D
        comm, _ = D.make_comm(local)
        nshards = world
        state = torch.empty(1 << (n - (world.bit_length() - 1)), dtype=dt, device="cuda")
    else:
        nshards = args.shards or 2
        comm = T.Comm.local(nshards)
        state = torch.empty(1 << n, dtype=dt, device="cuda")
    t0 = time.perf_counter()
    tree = T.build_error_tree(n, cfg.ops, nz.p1, nz.p2, nz.p_meas, cfg.shots, cfg.seed)
    t_ecm = time.perf_counter() - t0
    nl = tree.n_leaves
    per = max(1, args.leaves // max(args.steps, 1)) if args.leaves else 2
    stream = torch.cuda.current_stream()
    slots = np.zeros(cfg.shots, dtype=np.uint64)
    for w in range(args.warmup):
        T.run_tree(tree, prec, d_state=state, stream=stream, leaf_begin=w, leaf_end=w + 1, comm=comm,
                   out_slots=slots)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    with Clocks(local) as clk:
        e0.record(stream)
        for s in range(args.steps):
            b = s * per
            st = T.run_tree(tree, prec, d_state=state, stream=stream, leaf_begin=b, leaf_end=min(nl, b + per),
                            flags=T.EXEC_CONTINUE if s else 0, comm=comm, out_slots=slots)[1]
            stats.append(st)
        e1.record(stream)
        torch.cuda.synchronize()
    t_dev = e0.elapsed_time(e1) / 1e3
    tot = {k: sum(st[k] for st in stats) for k in stats[0]}
    _, plan = T.run_tree(tree, prec, flags=T.EXEC_PLAN_ONLY, comm=T.Comm.local(nshards))
    proj = t_ecm + t_dev * (plan["hbm_bytes"] + plan["sample_bytes"]) / max(tot["hbm_bytes"] + tot["sample_bytes"], 1)
    if rank == 0:
        print(json.dumps({
            "metric": f"noisy-sim wall s per circuit ({cfg.name}, sharded x{nshards})", "value": proj, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev * 1e3 / args.steps,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": f"c{prec}",
            "data": "synthetic", "config": config_dict(cfg, prec, world),
            "extrapolated": True, "timed_leaves": int(tot["leaves"]), "tree_leaves": nl,
            "projection": "ECM s + timed device s x (plan bytes / timed bytes)",
            "gpu_launches": int(tot["launches"]), "clocks": clk.summary(),
            "stats": {k: tot[k] for k in ("leaves", "resets", "gate_apps", "sweeps", "draws", "exchanges")},
            "e2e": None}), flush=True)
    if world > 1:
        comm.free()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
