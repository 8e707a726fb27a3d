#!/usr/bin/env python
"""Per-kernel DRAM bandwidth from an ncu launch list of scripts/kernel_bench.py (n = 30):
   ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv ...
Groups consecutive launches of the same kernel name with the bench's row order and prints
GB/s = (dram read + write bytes) / duration per launch (median), against MEASURED_PEAKS.json."""
import csv, io, json, os, sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, out):
    txt = open(path).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    hdr = rows[0]
    launches = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        lid = int(d["ID"])
        e = launches.setdefault(lid, {"kernel": d["Kernel Name"].split("(")[0][:60]})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6, "byte": 1, "Kbyte": 1e3,
              "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        e[d["Metric Name"]] = v
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    res = []
    for lid, e in launches.items():
        t = e.get("gpu__time_duration.sum")
        b = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
        if t:
            res.append({"id": lid, "kernel": e["kernel"], "ms": t / 1e6, "dram_GB": b / 1e9, "GBps": b / t,
                        "frac": b / t / peak})
    json.dump({"peak_GBs": peak, "launches": res}, open(out, "w"), indent=1)
    for r in res:
        print(f"{r['id']:5d} {r['kernel']:40s} {r['ms']:8.3f} ms {r['dram_GB']:7.2f} GB {r['GBps']:8.1f} GB/s {r['frac']:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
