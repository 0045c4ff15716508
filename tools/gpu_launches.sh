mkdir -p gpurun_out
# launch list of one warm projection (skip the cold call's launches)
ncu --metrics gpu__time_duration.sum --clock-control none -s 3600 -c 2500 --csv --log-file gpurun_out/warm_launches.csv python tools/perf_probe.py 4000 2 40 > gpurun_out/warm_probe.log 2>&1
python tools/ncu_summary.py gpurun_out/warm_launches.csv > gpurun_out/warm_summary.txt 2>&1
