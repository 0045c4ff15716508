mkdir -p gpurun_out
: > gpurun_out/reproj.txt
for cfg in "PSDPROJ_LOCK_REPROJ=0" "PSDPROJ_LOCK_REPROJ=1"; do
  echo "=== $cfg" >> gpurun_out/reproj.txt
  env $cfg timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 >> gpurun_out/reproj.txt
  env $cfg timeout 600 python tools/perf_probe.py 4000 3 500 2>&1 | cut -c1-60,215-290 >> gpurun_out/reproj.txt
done
