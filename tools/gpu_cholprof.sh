mkdir -p gpurun_out
rm -f gpurun_out/chol.ncu-rep
cat > /tmp/chol_probe.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
rng = np.random.default_rng(0)
t = 300
M = rng.standard_normal((t + 20, t)); G = torch.from_numpy(M.T @ M).cuda()
for _ in range(3): api.cholesky(G)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): api.cholesky(G)
e1.record(); torch.cuda.synchronize()
print("chol t=300 ms/call (incl. alloc + sync)", e0.elapsed_time(e1) / 10)
PY
python /tmp/chol_probe.py > gpurun_out/chol_probe.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:cholesky_cluster -s 2 -c 1 -o gpurun_out/chol python /tmp/chol_probe.py > /dev/null 2>&1
