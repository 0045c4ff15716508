# PSDPROJ_S_CAP sweep on the headline command (late-sequence line included)
for w in 512 -512 448; do
  PSDPROJ_S_CAP=$w python bench.py --no-e2e --no-cpu --no-r63 > gpurun_out/scap_$w.log 2> gpurun_out/scap_$w.err
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/scap_$w.log").read().strip().splitlines()[-1])
    l = d["late_sequence"]
    print("s_cap $w:", round(d["value"], 4), "proj/s iters", d["iters_per_projection"]["warm"], "ms/it", round(d["ms_per_iteration"], 4),
          "err", d["accuracy"]["max_rel_err"], "ok", d["accuracy"]["bound_dominates"], d["accuracy"]["status_counts"],
          "| late", round(l["value"], 3), l["iters"], l["status"])
except Exception as e:
    print("s_cap $w: ERR", e)
PY
done
