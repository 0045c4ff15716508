mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eig_launches.csv python tools/eigh_probe.py 400:150 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/eig_launches.csv > gpurun_out/eig_summary.txt 2>&1
