mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_sk.log 2>&1
PSDPROJ_NO_STREAMK=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_nosk.log 2>&1
