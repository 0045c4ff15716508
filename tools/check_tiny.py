import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import api
for s in (4, 40, 100):
    for sc in (0.0, 1e-300, 1.0):
        A = np.diag(np.linspace(0, 1, s) * sc)
        At = torch.as_strided(torch.from_numpy(A.T.copy()).cuda(), (s, s), (1, s))
        w, V, npos = api.eigh(At, s)
        print(s, sc, "w max", w.max().item(), "w min", w.min().item(), "npos", npos, "ref npos", int((np.diag(A) > 0).sum()), flush=True)
