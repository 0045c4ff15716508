import sys
sys.path.insert(0, '.')
import numpy as np
from paper_1912_02767_b200.admm import MaxCutADMM
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
W = np.ones((n, n)) - np.eye(n)
L = np.diag(W.sum(1)) - W
s = MaxCutADMM(L)
for k in range(3000):
    rp, rd, info = s.step()
    if k % 200 == 0:
        print(k, rp, rd, info["side"], info["iters"], info["npos"], flush=True)
print("done", s.objective())
