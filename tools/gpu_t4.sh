mkdir -p gpurun_out
: > gpurun_out/combo.txt
for cfg in "" "PSDPROJ_REFRESH=0" "PSDPROJ_LINV_MAX=0" "PSDPROJ_REFRESH=0 PSDPROJ_LINV_MAX=0" "PSDPROJ_TRI_NOREG=1"; do
  echo "cfg: $cfg" >> gpurun_out/combo.txt
  env $cfg timeout 300 python -m pytest tests/test_admm.py -m gpu -q 2>&1 | tail -1 >> gpurun_out/combo.txt
  env $cfg timeout 300 python tools/repro_admm.py 300 2>&1 | grep "^13 \|^39 \|^200 \|^250 " | cut -c1-120 >> gpurun_out/combo.txt
done
