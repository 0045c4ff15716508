mkdir -p gpurun_out
: > gpurun_out/matrix.txt
for cfg in "PSDPROJ_LINV_MAX=1e8" "PSDPROJ_LINV_MAX=1e8 PSDPROJ_RESTART=0" "PSDPROJ_LINV_MAX=1e10" "PSDPROJ_LINV_MAX=1e10 PSDPROJ_RESTART=0"; do
  echo "=== cfg: $cfg" >> gpurun_out/matrix.txt
  env $cfg timeout 600 python -m pytest tests/test_admm.py tests/test_gpu_projection.py -m gpu -q 2>&1 | tail -2 >> gpurun_out/matrix.txt
  env $cfg timeout 300 python tools/check_exp.py 2>&1 | grep -v "trace\|rotation" >> gpurun_out/matrix.txt
  env $cfg timeout 600 python tools/perf_probe.py 4000 3 500 2>&1 | cut -c1-60,215-290 >> gpurun_out/matrix.txt
done
