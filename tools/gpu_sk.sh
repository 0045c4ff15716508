mkdir -p gpurun_out
: > gpurun_out/minkt.txt
for cfg in "PSDPROJ_SPLITK_MINKT=8" "PSDPROJ_SPLITK_MINKT=24" "PSDPROJ_SPLITK_MINKT=48" "PSDPROJ_SPLITK_MINKT=100000"; do
  env $cfg timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['roofline']['frac'], {k: round(v,1) for k, v in d['phase_ms_per_step'].items()})" >> gpurun_out/minkt.txt
done
