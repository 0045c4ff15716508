"""Measure torch float64 GEMM (cuBLAS DGEMM) burst and sustained throughput on cuda:0."""
import json, time, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = a @ b; torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2 * n**3 / best / 1e9
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
# copy bandwidth fp64
x = torch.empty(1 << 27, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
bw = 0
for _ in range(10):
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
    bw = max(bw, 2 * x.numel() * 8 / e0.elapsed_time(e1) / 1e6)
print(json.dumps({"dgemm_tflops_burst": burst, "dgemm_tflops_sustained": sus, "copy_gbs_fp64_1GiB": bw, "n": n}))
