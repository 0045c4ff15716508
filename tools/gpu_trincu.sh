mkdir -p gpurun_out
rm -f gpurun_out/trireg.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tridiag_reg_kernel -c 1 -o gpurun_out/trireg python tools/eigh_probe.py 400:130 > gpurun_out/trireg_ncu.log 2>&1
