# Profiling pass (run under gpurun): per-call probe, eigensolver probes, ncu launch list of a short bench.
mkdir -p gpurun_out
python tools/perf_probe.py 4000 3 60 > gpurun_out/probe4000.log 2>&1
python tools/eigh_probe.py 100:40,160:60,200:80,300:120,400:150,500:200,600:220 > gpurun_out/eigh.log 2>&1
python tools/jacobi_probe.py 100,160,200,300,400,500,600 > gpurun_out/jac.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --max-iter 40 --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
