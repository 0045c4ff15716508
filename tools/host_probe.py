"""Host-side split of psdproj_project (PSDPROJ_HOSTPROF=1 prints wall / in-sync / issuing per call)
on C3-R-like sequences, profile bits off (development tool)."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_1912_02767_b200 import api
from workloads import generators as G
n = int(sys.argv[1]); steps = int(sys.argv[2]); mi = int(sys.argv[3]); prof = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = G.C3R(n)
mats = [A for _, A, _, _ in G.rotation_sequence(cfg, steps=steps, device='cuda')]
ctx = api.Context(n, params=api.default_params(max_iter=mi, profile=prof))
out = torch.empty_like(mats[0])
for k, A in enumerate(mats):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, inf = ctx.project(A, 1e-7, out=out)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"k={k} ms={dt*1e3:.1f} iters={inf['iters']} launches={inf['launches']}", flush=True)
