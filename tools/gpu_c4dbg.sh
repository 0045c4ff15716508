mkdir -p gpurun_out
: > gpurun_out/c4dbg.txt
for cfg in "X=1" "PSDPROJ_LINV_MAX=0" "PSDPROJ_LINV_MAX=0 PSDPROJ_RESTART=0" "PSDPROJ_LINV_MAX=1e12"; do
  echo "=== $cfg" >> gpurun_out/c4dbg.txt
  env $cfg timeout 600 python bench.py --workload c4 --steps 2 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['iters_per_projection'])" >> gpurun_out/c4dbg.txt
done
