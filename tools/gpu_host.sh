mkdir -p gpurun_out
PSDPROJ_HOSTPROF=1 timeout 600 python tools/host_probe.py 4000 4 500 0 > gpurun_out/host.txt 2>&1
PSDPROJ_HOSTPROF=1 timeout 600 python tools/host_probe.py 4000 3 500 3 >> gpurun_out/host.txt 2>&1
