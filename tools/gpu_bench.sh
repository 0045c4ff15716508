# Round-end style measurement: bench line, ncu launch list of the same command, ncu --set full of one a3 launch.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$? >> gpurun_out/bench_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/bench_launches.csv python bench.py > gpurun_out/bench_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/bench_launches.csv --json gpurun_out/bench_launches_summary.json > gpurun_out/bench_launches_summary.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:dgemm_kp_kernel<0, 0, 64, 64, 4, 1>' -s 40 -c 1 -o gpurun_out/amul python bench.py --steps 1 --warmup 0 --max-iter 30 --no-e2e --no-cpu > gpurun_out/amul_ncu.log 2>&1
