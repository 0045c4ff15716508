python tools/tri_debug.py > gpurun_out/tri_debug.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q > gpurun_out/kern_tests.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tridiag_tile --csv python tools/eigh_probe.py 64:20,96:30,128:40,160:50,192:64,224:70,256:90 > gpurun_out/ncu_tri_tile3.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:tridiag_tile -c 1 -s 2 -o gpurun_out/tri_tile_s192 python tools/eigh_probe.py 192:64 > gpurun_out/ncu_full.log 2>&1
