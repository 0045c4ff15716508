"""Compact text form of `ncu -i rep --page details --csv`: kernel name, then one line per metric
(`section | metric | value unit`), rule texts dropped. Usage:
  python tools/ncu_details_txt.py details.csv > summary.txt"""
import csv
import sys

rows = list(csv.DictReader(ln for ln in open(sys.argv[1]) if ln.startswith('"')))
if not rows:
    sys.exit("no rows")
print("kernel:", rows[0]["Kernel Name"][:160])
print("grid", rows[0]["Grid Size"], "block", rows[0]["Block Size"])
for r in rows:
    if not r.get("Metric Name"):
        continue
    print(f'{r["Section Name"][:28]} | {r["Metric Name"]} | {r["Metric Value"]} {r["Metric Unit"]}')
