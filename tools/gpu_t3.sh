mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
timeout 300 python tools/repro_admm.py 300 > gpurun_out/repro_admm.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/bench.log
