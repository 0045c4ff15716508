S=32:10,64:20,100:33,128:40,160:50,192:64,224:70,256:90
PSDPROJ_TRI_TILE=0 python tools/eigh_probe.py $S > gpurun_out/eigh_cluster.log 2>&1
python tools/eigh_probe.py $S > gpurun_out/eigh_tile.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kern_tests.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tridiag --csv python tools/eigh_probe.py 64:20,128:40,192:64,256:90 > gpurun_out/ncu_tri_tile.csv 2>&1
PSDPROJ_TRI_TILE=0 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tridiag --csv python tools/eigh_probe.py 64:20,128:40,192:64,256:90 > gpurun_out/ncu_tri_cluster.csv 2>&1
