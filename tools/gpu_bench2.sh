mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$? >> gpurun_out/bench_full.log
timeout 900 python bench.py --workload c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.log 2>&1
