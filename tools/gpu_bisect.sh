# Multisection width sweep: tri_bisect(_ms) kernel time at s = 200 / 400 (ncu launch list) + eigensolver tests
mkdir -p gpurun_out; : > gpurun_out/bisect.txt
timeout 600 python -m pytest -q -x tests/test_gpu_kernels.py > gpurun_out/bisect_tests.txt 2>&1
PSDPROJ_BISECT_G=32 timeout 300 python -m pytest -q -x tests/test_gpu_kernels.py >> gpurun_out/bisect_tests.txt 2>&1
for g in 32 64 128 256 512; do
  PSDPROJ_BISECT_G=$g timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:tri_bisect \
    --log-file gpurun_out/bisect_$g.csv python tools/eigh_probe.py 200:70,400:130 > /dev/null 2>&1
  echo "G=$g" >> gpurun_out/bisect.txt
  grep -o '"tri_bisect[^"]*".*' gpurun_out/bisect_$g.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' >> gpurun_out/bisect.txt
  echo >> gpurun_out/bisect.txt
done
