mkdir -p gpurun_out
: > gpurun_out/atile.txt
for cfg in "PSDPROJ_AMUL_TILE=128" "PSDPROJ_AMUL_TILE=64"; do
  env $cfg timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['phase_ms_per_step']['a3_block_multiply'])" >> gpurun_out/atile.txt
done
