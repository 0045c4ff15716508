mkdir -p gpurun_out
PSDPROJ_TRI_PROF=1 python tools/eigh_probe.py 200:80,400:150,600:200,800:250 > gpurun_out/triprof.txt 2>&1
python -m pytest -q -x tests/test_gpu_kernels.py -k eigh >> gpurun_out/triprof.txt 2>&1
