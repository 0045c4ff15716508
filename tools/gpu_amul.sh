mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:\(int\)4, \(int\)1>' -s 40 -c 1 -o gpurun_out/amul python bench.py --steps 1 --warmup 0 --max-iter 30 --no-e2e --no-cpu > gpurun_out/amul_ncu.log 2>&1
