# Launch list of the bench command in its final configuration (B200_PROFILING.md recipe): the command
# first exits 0 without ncu. max_iter 60 bounds it (the cold call and one timed warm step, ~6k
# launches): the converged bench makes ~10^5 launches per step, too many to serialise under ncu.
CMD="python bench.py --steps 1 --warmup 0 --max-iter 60 --no-e2e --no-cpu --no-extra"
$CMD > gpurun_out/plain_bench_short.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
      --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
