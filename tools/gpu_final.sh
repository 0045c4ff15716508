# Measurement pass: bench line, ncu launch list of the same command (warm region), one a3 launch --set full.
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$? >> gpurun_out/bench_full.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 40000 -c 16000 --csv --log-file gpurun_out/bench_launches_warm.csv python bench.py --no-e2e --no-cpu > gpurun_out/bench_ncu_warm.log 2>&1
python tools/ncu_summary.py gpurun_out/bench_launches_warm.csv --json gpurun_out/bench_launches_warm_summary.json > gpurun_out/bench_launches_warm_summary.txt 2>&1
rm -f gpurun_out/amul.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:\(int\)4, \(int\)1>' -s 40 -c 1 -o gpurun_out/amul python bench.py --steps 1 --warmup 0 --max-iter 30 --no-e2e --no-cpu > gpurun_out/amul_ncu.log 2>&1
timeout 900 python bench.py --workload c4 --steps 2 --warmup 3 > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 > gpurun_out/bench_c5.log 2>&1
