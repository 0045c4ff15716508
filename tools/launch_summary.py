"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per psdproj_project call:
calls are delimited by nonfinite_kernel (the first kernel of every call). Prints the kernel-time
shares of call `which` (default: the last one, the timed warm step).

  python tools/launch_summary.py launches.csv [which] > summary.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else -1
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
calls, cur = [], None
for r in data:
    name = r[ki].split("(")[0].replace("void ", "")
    if "nonfinite_kernel" in name:
        cur = []
        calls.append(cur)
    if cur is not None:
        cur.append((name, float(r[vi])))
sel = calls[which]
agg = collections.defaultdict(lambda: [0, 0.0])
for name, ns in sel:
    agg[name][0] += 1
    agg[name][1] += ns
tot = sum(v[1] for v in agg.values())
print(f"call {which if which >= 0 else len(calls) + which} of {len(calls)}: {len(sel)} launches, {tot / 1e6:.2f} ms kernel time "
      f"(ncu-serialised, cold caches: compare shares, not absolutes)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{100 * v[1] / tot:6.2f}% {v[1] / 1e6:9.3f} ms {v[0]:6d} x {v[1] / v[0] / 1e3:9.2f} us  {k[:80]}")
