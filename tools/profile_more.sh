# ncu --set full captures (one launch each) of the next kernels of a warm LOBPCG iteration after the
# tridiagonalisation and the a3 multiply (B200_PROFILING.md recipe: the command first exits 0 without ncu)
CMD="python tools/c3r_probe.py --steps 2 --max-iter 40"
$CMD > gpurun_out/plain_probe_more.log 2>&1 || { echo "plain run failed"; exit 1; }
for k in cholesky_cluster_kernel tri_bisect_ms_kernel dgemm_kp_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 -f \
      -o gpurun_out/ncu_$k $CMD > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
  ncu -i gpurun_out/ncu_$k.ncu-rep --page details --csv > gpurun_out/ncu_$k.details.csv 2>/dev/null
done
