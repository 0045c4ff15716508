for cfg in "0 0" "0 0.01" "40 0.01" "40 0.1" "0 0.1"; do
  set -- $cfg
  timeout 600 python bench.py --workload c5 --steps 1 --warmup 3 --adapt-every $1 --tol-ratio $2 > gpurun_out/c5_$1_$2.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/c5_$1_$2.log').read().strip().splitlines()[-1])
print('$1 $2', {k:d[k] for k in ('value','solve_s','admm_iters','r_prim','r_dual','objective','lobpcg_iters_per_admm_iter')})"
done > gpurun_out/c5_summary.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_projection.py -q -k krylov > gpurun_out/krylov_tests.log 2>&1
python tools/seq_probe.py --cfg c3r --tol 1e-7 --steps 5 --param max_iter=4000 --param krylov_depth=2 > gpurun_out/c3r_depth2.log 2>&1
python tools/seq_probe.py --cfg c3r --tol 1e-7 --steps 5 --param max_iter=4000 --param krylov_depth=3 > gpurun_out/c3r_depth3.log 2>&1
