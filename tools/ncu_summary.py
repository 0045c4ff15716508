"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name:
launches, total device time, share of the summed kernel time. Usage:
  python tools/ncu_summary.py launches.csv [--json out.json]"""
import csv
import json
import sys
from collections import defaultdict


def load(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        rows.append((short, v * scale, r.get("Grid Size"), r.get("Block Size")))
    return rows


def summarise(rows):
    agg = defaultdict(lambda: [0, 0.0])
    for name, ms, _, _ in rows:
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(a[1] for a in agg.values())
    out = [{"kernel": k, "launches": a[0], "ms": round(a[1], 4), "share": round(a[1] / tot, 4) if tot else 0.0,
            "mean_us": round(1e3 * a[1] / a[0], 2)} for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    return {"total_kernel_ms": round(tot, 3), "launches": len(rows), "kernels": out}


if __name__ == "__main__":
    s = summarise(load(sys.argv[1]))
    print(f"{s['launches']} launches, {s['total_kernel_ms']:.2f} ms kernel time")
    for k in s["kernels"][:40]:
        print(f"{k['share']*100:6.2f}%  {k['ms']:10.3f} ms  {k['launches']:6d} x {k['mean_us']:9.2f} us  {k['kernel'][:90]}")
    if "--json" in sys.argv:
        json.dump(s, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
