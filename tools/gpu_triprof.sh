mkdir -p gpurun_out
PSDPROJ_TRI_PROF=1 python tools/eigh_probe.py 200:80,400:150,600:200 > gpurun_out/triprof.txt 2>&1
python -m pytest -q -x tests/test_gpu_kernels.py -k eigh >> gpurun_out/triprof.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:tridiag_cluster_kernel -c 1 -o gpurun_out/tri400 python tools/eigh_probe.py 400:150 > gpurun_out/tri400.log 2>&1
