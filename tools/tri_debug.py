"""Debug: d, e of the tridiagonalisation (psdproj_eigh workspace head) for a given matrix."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1912_02767_b200 import _lib, api
L = _lib.load()
for s, scale in ((4, 1e300), (40, 1e300), (4, 1.0), (6, 1.0)):
    A = np.diag(np.linspace(0.0, 1.0, s) * scale)
    if scale == 1.0:
        M = np.random.default_rng(s).standard_normal((s, s)); A = (M + M.T) / 2
    At = api.colmajor(s, s); At.copy_(torch.from_numpy(A))
    m = s
    w = torch.empty(m, dtype=torch.float64, device='cuda'); V = api.colmajor(s, m)
    npos = torch.zeros(1, dtype=torch.int32, device='cuda')
    ws = torch.zeros(int(L.psdproj_eigh_ws_elems(s, m)), dtype=torch.float64, device='cuda')
    rc = L.psdproj_eigh(s, ctypes.c_void_p(At.data_ptr()), s, m, ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(V.data_ptr()), s,
                        ctypes.c_void_p(npos.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    h = ws.cpu().numpy()
    print(s, scale, 'rc', rc, 'npos', int(npos.item()), 'd', h[:s][:6], 'e', h[s:2 * s - 1][:6], 'w', w.cpu().numpy()[:6])
    if scale == 1.0:
        T = np.diag(h[:s]) + np.diag(h[s:2*s-1], 1) + np.diag(h[s:2*s-1], -1)
        print('   eig T vs A', np.abs(np.sort(np.linalg.eigvalsh(T)) - np.sort(np.linalg.eigvalsh(A))).max())
