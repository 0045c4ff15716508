mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eig_launches.csv python tools/eigh_probe.py 400:150 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/eig_launches.csv > gpurun_out/eig_summary.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:tridiag_cluster_kernel -c 1 -o gpurun_out/tri400 python tools/eigh_probe.py 400:150 > gpurun_out/tri400.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:cholesky_cluster_kernel -s 20 -c 1 -o gpurun_out/chol python tools/perf_probe.py 2000 1 30 > gpurun_out/chol.log 2>&1
