mkdir -p gpurun_out
timeout 600 python bench.py --shard --steps 1 --warmup 1 --max-iter 100 --no-e2e --no-cpu > gpurun_out/bench_shard.log 2>&1; echo rc=$? >> gpurun_out/bench_shard.log
timeout 600 python bench.py --steps 1 --warmup 1 --max-iter 100 --no-e2e --no-cpu > gpurun_out/bench_noshard.log 2>&1
for t in 4 16 32; do PSDPROJ_BATCH_THREADS=$t timeout 600 python bench.py --workload c4 --steps 1 --warmup 1 > gpurun_out/bench_c4_t$t.log 2>&1; done
