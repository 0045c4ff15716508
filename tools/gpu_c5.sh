mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "not admm" > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
python tools/eigh_probe.py 1500:200,2000:300,2000:2000 > gpurun_out/eigh_big.log 2>&1
timeout 1500 python bench.py --workload c5 --warmup 0 > gpurun_out/bench_c5.log 2>&1; echo rc=$? >> gpurun_out/bench_c5.log
