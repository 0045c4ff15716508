python tools/tri_debug.py > gpurun_out/tri_debug.log 2>&1
PSDPROJ_TRI_TILE=0 python tools/tri_debug.py > gpurun_out/tri_debug0.log 2>&1
python tools/eigh_probe.py 64:20,128:40,192:64,256:90 > gpurun_out/eigh_tile2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tridiag_tile --csv python tools/eigh_probe.py 64:20,128:40,192:64,256:90 > gpurun_out/ncu_tri_tile2.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:tridiag_tile -c 1 -s 12 -o gpurun_out/tri_tile_s128 python tools/eigh_probe.py 128:40 > gpurun_out/ncu_full.log 2>&1
