# PSDPROJ_WIDE_NO_P sweep on the headline command (no companions except the late-sequence line)
for w in 0 96 128 160 192; do
  PSDPROJ_WIDE_NO_P=$w python bench.py --no-e2e --no-cpu --no-r63 > gpurun_out/wide_$w.log 2> gpurun_out/wide_$w.err
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/wide_$w.log").read().strip().splitlines()[-1])
    l = d["late_sequence"]
    print("wide_no_p $w:", round(d["value"], 4), "proj/s iters", d["iters_per_projection"]["warm"], "ms/it", round(d["ms_per_iteration"], 4),
          "err", d["accuracy"]["max_rel_err"], "ok", d["accuracy"]["bound_dominates"], d["accuracy"]["status_counts"],
          "| late", round(l["value"], 3), l["iters"], l["status"])
except Exception as e:
    print("wide_no_p $w: ERR", e)
PY
done
