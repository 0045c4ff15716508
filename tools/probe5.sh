for ke in -1 20 40; do echo "keep_extra=$ke"; timeout 300 python tools/seq_probe.py --cfg c2cl --tol 1e-10 --steps 12 --param keep_extra=$ke; done > gpurun_out/probe_c2cl.log 2>&1
for lf in 1.0 0.1 0.01; do echo "lock_factor=$lf"; timeout 300 python tools/seq_probe.py --cfg c3r --n 1000 --tol 1e-10 --steps 3 --param lock_factor=$lf; done > gpurun_out/probe_c3r1000_lf.log 2>&1
echo soft; timeout 300 python tools/seq_probe.py --cfg c3r --n 1000 --tol 1e-10 --steps 3 --param locking=1 >> gpurun_out/probe_c3r1000_lf.log 2>&1
for lf in 1.0 0.1; do echo "n4000 lock_factor=$lf"; timeout 300 python tools/seq_probe.py --cfg c3r --tol 1e-7 --steps 4 --param lock_factor=$lf --param max_iter=4000; done > gpurun_out/probe_c3r4000_lf.log 2>&1
