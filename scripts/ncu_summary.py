#!/usr/bin/env python
"""Summarize an ncu report (--set full capture) and an ncu launch list into profiles/.

usage: python scripts/ncu_summary.py <prof.ncu-rep> <launches.csv> <out.json> [algorithmic_bytes_per_launch]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_bytes",
    "dram__bytes_read.sum.per_second": "dram_read_bytes_per_s",
    "smsp__average_warp_latency_issue_stalled_barrier": "stall_barrier",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    # ncu prints memory sizes in decimal (Kbyte = 1e3 B) and shared-memory sizes in binary units
    # (KiB, "Kibyte"): both are scaled to plain bytes here
    scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "Kibyte": 1024, "Mibyte": 1 << 20, "Gibyte": 1 << 30, "KB": 1e3, "KiB": 1024, "MiB": 1 << 20}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    unit = units.get(k, "")
                    if unit.endswith("/block"):   # e.g. dynamic shared memory in "Kbyte/block"
                        unit = unit[:-len("/block")]
                    e[name] = float(d[k].replace(",", "")) * scale.get(unit, 1)
                except ValueError:
                    e[name] = d[k]
        res.append(e)
    return res


def launches(path):
    agg = defaultdict(lambda: [0, 0.0])
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:80]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(x[1] for x in agg.values()) or 1.0
    return {k: {"launches": n, "total_ms": t / 1e6, "share": t / tot} for k, (n, t) in
            sorted(agg.items(), key=lambda kv: -kv[1][1])}


def main():
    rep, lcsv, out = sys.argv[1:4]
    alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
    full = raw(rep)
    for e in full:
        if "dram_read_bytes" in e and "dram_write_bytes" in e:
            e["dram_traffic_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
            if alg:
                e["algorithmic_bytes"] = alg
                e["traffic_over_algorithmic"] = e["dram_traffic_bytes"] / alg
            if e.get("duration_ns"):
                e["achieved_GBps_dram"] = e["dram_traffic_bytes"] / e["duration_ns"]
                if alg:
                    e["achieved_GBps_algorithmic"] = alg / e["duration_ns"]
    res = {"full_capture": full, "launch_list": launches(lcsv) if lcsv != "-" else None}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
