# Round-2 ncu evidence (B200_PROFILING.md recipe): each command first exits 0 without ncu. The launch list
# uses a short bench command (max_iter 60: the cold call and one timed warm step, ~8k launches) -- the
# full bench makes ~10^5 launches, too many to serialise under ncu.
CMD="python bench.py --steps 1 --warmup 0 --max-iter 60 --no-e2e --no-cpu --no-extra"
$CMD > gpurun_out/plain_bench_short.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
      --log-file gpurun_out/launches_r02.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python tools/c3r_probe.py --steps 2 --max-iter 40"
$CMD2 > gpurun_out/plain_probe.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tridiag_reg -s 30 -c 1 \
      -o gpurun_out/tri_reg_r02 $CMD2 > gpurun_out/ncu_tri.log 2>&1
$CMD2 > gpurun_out/plain_probe2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel -s 30 -c 1 \
      -o gpurun_out/a3_r02 $CMD2 > gpurun_out/ncu_a3.log 2>&1
