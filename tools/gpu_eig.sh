mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_kernels.py > gpurun_out/eig_tests.txt 2>&1
timeout 300 python tools/eigh_probe.py 100:33,200:70,300:100,400:130,450:150,500:170 > gpurun_out/eig_probe.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eig_launches.csv python tools/eigh_probe.py 400:130 > /dev/null 2>&1
rm -f gpurun_out/tw.ncu-rep; timeout 600 ncu --set full --import-source on --clock-control none -k regex:tri_twisted -c 1 -o gpurun_out/tw python tools/eigh_probe.py 400:130 > /dev/null 2>&1
