"""a3 block multiply Y = A Z (A symmetric n x n) at n = 4000: the TMA kernel (psdproj_symm_multiply)
vs the cp.async DMMA kernel (psdproj_dgemm), device time (CUDA events, min of 10), TF/s and the
fraction of the measured DGEMM peak (35.46 TF/s) and of HBM (6457 GB/s, A streamed once)."""
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1912_02767_b200 import api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "8,16,32,48,64,70,96,128,200,300").split(",")]
g = torch.Generator(device="cuda").manual_seed(1)
M = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
A = api.colmajor(n, n)
A.copy_(0.5 * (M + M.T))
ws = torch.empty(32 * n * max(ks), dtype=torch.float64, device="cuda")
for k in ks:
    Z = api.colmajor(n, k)
    Z.copy_(torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g))
    Y1, Y2 = api.colmajor(n, k), api.colmajor(n, k)
    res = {}
    for name, fn in (("tma", lambda: api.symm_multiply(1.0, A, Z, Y=Y1, ws=ws)),
                     ("cp_async", lambda: api.dgemm(0, 0, 1.0, A, Z, 0.0, Y2, ws=ws))):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        tf = 2.0 * n * n * k / (best / 1e3) / 1e12
        res[name] = {"ms": round(best, 4), "tflops": round(tf, 2), "frac_p64": round(tf / 35.46, 3),
                     "hbm_frac": round(8.0 * n * n / (best / 1e3) / 1e9 / 6456.8, 3)}
    res["max_diff"] = float((Y1 - Y2).abs().max())
    print(json.dumps({"n": n, "k": k, **res}), flush=True)
