mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest -q -x tests/test_gpu_kernels.py > gpurun_out/triprof_tests.txt 2>&1
PSDPROJ_TRI_PROF=1 timeout 120 python tools/eigh_probe.py 100:33,200:70,300:100,400:130,450:150,500:170 > gpurun_out/triprof.txt 2>&1
timeout 120 python tools/eigh_probe.py 100:33,200:70,300:100,400:130,450:150,500:170 >> gpurun_out/triprof.txt 2>&1
PSDPROJ_TRI_NOREG=1 timeout 120 python tools/eigh_probe.py 100:33,200:70,300:100,400:130,450:150,500:170 >> gpurun_out/triprof.txt 2>&1
