mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_kernels.py -k "eigh or cholesky" > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
ncu --metrics gpu__time_duration.sum --clock-control none -s 3200 -c 1400 --csv --log-file gpurun_out/warm_launches.csv python tools/perf_probe.py 4000 2 20 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/warm_launches.csv > gpurun_out/warm_summary.txt 2>&1
