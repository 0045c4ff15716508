import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle.exact import project_exact, eig
from paper_1912_02767_b200 import api
from workloads.generators import BO, planted
cfg = BO(count=48, lo=8, hi=100)
mats = [planted(*cfg.block(i)) for i in range(cfg.count)]
b = int(sys.argv[1])
Q, lam = cfg.block(b)
print('block', b, 'n', cfg.sizes[b], 'top eigs', np.sort(lam)[::-1][:4])
batch = api.TinyLobpcgBatch(cfg.sizes, seed=7)
outs, res = batch.project([torch.from_numpy(A).cuda() for A in mats], 1e-10)
torch.cuda.synchronize()
A = mats[b]
print({k: v[b] for k, v in res.items()}, 'err', np.linalg.norm(outs[b].cpu().numpy() - project_exact(A)))
