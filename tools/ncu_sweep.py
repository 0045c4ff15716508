"""Per-launch durations (and DRAM bytes) of an ncu --csv launch list, one line per kernel launch."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
by = {}
for r in rows[1:]:
    by.setdefault(int(r[iid]), [r[ik].split("(")[0][:48], {}])[1][r[im]] = float(r[iv].replace(",", ""))
for i in sorted(by):
    name, m = by[i]
    t = m.get("gpu__time_duration.sum", 0.0) / 1e3
    b = m.get("dram__bytes_read.sum", 0.0) / 1e6
    print(f"{i:4d} {t:9.2f} us {b:9.1f} MB  {name}")
