mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
timeout 600 python tools/perf_probe.py 4000 2 60 > gpurun_out/probe4000.log 2>&1
python tools/eigh_probe.py 200:80,400:150,600:220 > gpurun_out/eigh.log 2>&1
