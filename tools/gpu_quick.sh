# quick GPU pass: kernel + projection tests, eigensolver timings, per-phase probe at n=4000
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
python tools/eigh_probe.py 200:80,400:150,600:220,800:300,1200:400 > gpurun_out/eigh.log 2>&1
timeout 600 python tools/perf_probe.py 4000 3 60 > gpurun_out/probe4000.log 2>&1
