mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lb tools/micro/lat_bench.cu && /tmp/lb > gpurun_out/lat.txt 2>&1
rm -f gpurun_out/bt.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:backtransform_panel -c 1 -o gpurun_out/bt python tools/eigh_probe.py 400:150 > /dev/null 2>&1
