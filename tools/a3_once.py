"""One a3 block multiply per k in argv[2] at n = argv[1] (ncu target: psdproj_symm_multiply)."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1912_02767_b200 import api  # noqa: E402

n = int(sys.argv[1])
g = torch.Generator(device="cuda").manual_seed(1)
M = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
A = api.colmajor(n, n)
A.copy_(0.5 * (M + M.T))
for k in (int(x) for x in sys.argv[2].split(",")):
    Z = api.colmajor(n, k)
    Z.copy_(torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g))
    ws = torch.empty(32 * n * k, dtype=torch.float64, device="cuda")
    api.symm_multiply(1.0, A, Z, ws=ws)
    torch.cuda.synchronize()
