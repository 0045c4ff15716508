"""Aggregate ncu source-page samples (--print-source cuda,sass --csv) per CUDA source line.
Usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(lambda: [0, 0, 0, ""])
hdr = None
line = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < 7:
        continue
    if r[0].strip():
        line = (int(r[0]), r[1])
    if line is None:
        continue
    try:
        smp = int(r[hdr["# Samples"]] or 0)
        bar = int(r[hdr["stall_barrier"]] or 0)
        ex = int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, KeyError):
        continue
    a = agg[line[0]]
    a[0] += smp; a[1] += bar; a[2] += ex; a[3] = line[1]
tot = sum(a[0] for a in agg.values()) or 1
for ln, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a[0]:7d} {100 * a[0] / tot:5.1f}%  bar={a[1]:6d} inst={a[2]:9d}  L{ln:<4d} {a[3].strip()[:80]}")
