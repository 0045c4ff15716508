mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_admm.py > gpurun_out/admm_tests.log 2>&1; echo rc=$? >> gpurun_out/admm_tests.log
timeout 1200 python bench.py --workload c5 --warmup 0 > gpurun_out/bench_c5.log 2>&1; echo rc=$? >> gpurun_out/bench_c5.log
