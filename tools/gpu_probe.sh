mkdir -p gpurun_out
timeout 600 python tools/perf_probe.py 4000 2 60 > gpurun_out/probe4000.log 2>&1
PSDPROJ_CLA_CS=8 timeout 600 python tools/perf_probe.py 4000 2 60 >> gpurun_out/probe4000.log 2>&1
