mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_q.log 2>&1
