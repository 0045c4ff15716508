mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_kernels.py > gpurun_out/bt_tests.txt 2>&1
: > gpurun_out/bt.txt
for v in 0 1; do
  if [ $v = 1 ]; then export PSDPROJ_BT_WARP=1; fi
  echo "warp=$v" >> gpurun_out/bt.txt
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:backtransform \
    --log-file gpurun_out/bt_$v.csv python tools/eigh_probe.py 200:70,300:100,400:130,500:170,700:230 > /dev/null 2>&1
  grep -o '"backtransform[^"]*".*' gpurun_out/bt_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' >> gpurun_out/bt.txt
  echo >> gpurun_out/bt.txt
done
