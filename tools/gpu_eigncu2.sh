mkdir -p gpurun_out
rm -f gpurun_out/eig3.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:tri_inviter|tri_bisect|backtransform_wy' -c 3 -o gpurun_out/eig3 python tools/eigh_probe.py 400:130 > gpurun_out/eig3_ncu.log 2>&1
