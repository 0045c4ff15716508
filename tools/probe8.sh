python tools/tri_debug.py > gpurun_out/tri_debug.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tridiag_tile -c 1 -s 2 -o gpurun_out/tri_tile_s128 python tools/eigh_probe.py 128:40 > gpurun_out/ncu_full.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q > gpurun_out/kern_tests.log 2>&1
