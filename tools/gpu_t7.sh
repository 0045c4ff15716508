mkdir -p gpurun_out
: > gpurun_out/ovl.txt
for cfg in "PSDPROJ_CHOL_CS=8" "PSDPROJ_CHOL_CS=4" "PSDPROJ_CHOL_CS=16" "PSDPROJ_CHOL_CS=8 PSDPROJ_NO_OVERLAP=1"; do
  echo "=== $cfg" >> gpurun_out/ovl.txt
  env $cfg timeout 600 python tools/perf_probe.py 4000 3 500 2>&1 | tail -2 | cut -c1-40,300-420 >> gpurun_out/ovl.txt
done
