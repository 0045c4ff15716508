# R63 sweep on the headline command (no companions): krylov_depth x krylov_max_active
for cfg in ${KMA_CFGS:-"1 0" "2 48" "2 96" "3 48" "3 64" "4 48" "2 0"}; do
  set -- $cfg
  python bench.py --no-extra --no-e2e --no-cpu --krylov-depth $1 --krylov-max-active $2 > gpurun_out/kma_$1_$2.log 2> gpurun_out/kma_$1_$2.err
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/kma_$1_$2.log").read().strip().splitlines()[-1])
    print("depth $1 max_active $2:", round(d["value"], 4), "proj/s iters", d["iters_per_projection"]["warm"], "ms/it", round(d["ms_per_iteration"], 4),
          "err", d["accuracy"]["max_rel_err"], "bound_ok", d["accuracy"]["bound_dominates"], "status", d["accuracy"]["status_counts"])
except Exception as e:
    print("depth $1 max_active $2: ERR", e)
PY
done
