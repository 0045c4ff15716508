mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
timeout 900 python bench.py --workload c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.log 2>&1
PSDPROJ_BATCH_THREADS=1 timeout 900 python bench.py --workload c4 --steps 1 --warmup 1 >> gpurun_out/bench_c4.log 2>&1
