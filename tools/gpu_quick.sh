# quick GPU pass: kernel + projection tests, eigensolver timings, per-phase probe at n=4000
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
python tools/eigh_probe.py 100:40,160:60,200:80,300:120,400:150,500:200,600:220,640:220,1000:300 > gpurun_out/eigh.log 2>&1
timeout 600 python tools/perf_probe.py 4000 3 60 > gpurun_out/probe4000.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eig_launches.csv python tools/eigh_probe.py 400:150 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/eig_launches.csv > gpurun_out/eig_summary.txt 2>&1
