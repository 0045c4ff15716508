"""f1: approximate ADMM (Alg. 1) for the MaxCut SDP of BASELINE
configs[4]:  maximise 1/4 <L, X>  s.t.  diag(X) = 1,  X PSD.

Every arithmetic step runs in libpsdproj.so: `psdproj_admm_maxcut_step1` (line 3's elementwise
KKT solve -- A^T A is diagonal for A = [D; I] -- the relaxation of line 4 and the projection input
of line 5), `psdproj_project` (line 5's PSD projection by warm-started LOBPCG with the paper's
tolerance schedule 10/k^1.01) and `psdproj_admm_maxcut_step2` (line 6's dual update
and the residual maxima). This module only sequences the calls. Reading R43: line 5
projects alpha z~ + (1 - alpha) z^k + y^k/rho and line 6 uses the same relaxed z-hat (COSMO form).
Termination (R33): max(||x - z||_inf, ||diag X - 1||_inf) <= eps and ||q + A^T y||_inf <= eps.
"""
import ctypes

import torch

from . import _lib, api
from ._lib import check


def tol_schedule(k, c=10.0, p=1.01):
    """LOBPCG residual tolerance at ADMM iteration k >= 1."""
    return c / float(k) ** p


class MaxCutADMM:
    def __init__(self, L, rho=0.1, sigma=1e-6, alpha=1.6, device="cuda", params=None, tol_floor=0.0,
                 tol_override=None):
        n = L.shape[0]
        self.n, self.rho, self.sigma, self.alpha = n, float(rho), float(sigma), float(alpha)
        self.tol_floor, self.tol_override = tol_floor, tol_override
        dev = torch.device(device)
        Lt = torch.as_tensor(L, dtype=torch.float64, device=dev)
        self.Q = (-0.25 * Lt).contiguous()  # min <Q, X> = -max 1/4 <L, X>
        self.L = Lt
        z = lambda: torch.zeros(n, n, dtype=torch.float64, device=dev)  # noqa: E731
        self.X, self.Zp, self.Yp, self.Zh, self.V = z(), z(), z(), z(), z()
        self.ye = torch.zeros(n, dtype=torch.float64, device=dev)
        self.zeh = torch.zeros(n, dtype=torch.float64, device=dev)
        self.ctx = api.Context(n, params=params if params is not None else api.default_params(seed=1912))
        self.k = 0
        self.infos = []

    def step(self):
        """One iteration of Alg. 1; returns (r_prim, r_dual, projection info)."""
        L_ = _lib.load()
        n, st = self.n, api._stream_ptr(None)
        p = api._ptr
        check(L_.psdproj_admm_maxcut_step1(n, p(self.X), p(self.Zp), p(self.Yp), p(self.ye), p(self.Q), n,
                                           self.sigma, self.rho, self.alpha, p(self.Zh), p(self.V), p(self.zeh),
                                           st), "psdproj_admm_maxcut_step1")
        self.k += 1
        tol = self.tol_override if self.tol_override is not None else max(tol_schedule(self.k), self.tol_floor)
        _, info = self.ctx.project(self.V, tol, out=self.Zp)
        res = (ctypes.c_double * 3)()
        check(L_.psdproj_admm_maxcut_step2(n, p(self.X), p(self.Zp), p(self.Zh), p(self.Yp), p(self.ye),
                                           p(self.zeh), p(self.Q), n, self.rho, res, st),
              "psdproj_admm_maxcut_step2")
        self.infos.append(info)
        return max(res[0], res[1]), res[2], info

    def solve(self, eps=1e-4, max_iter=5000):
        r_p = r_d = float("inf")
        while self.k < max_iter:
            r_p, r_d, _ = self.step()
            if r_p <= eps and r_d <= eps:
                break
        return {"iters": self.k, "r_prim": r_p, "r_dual": r_d, "objective": self.objective(),
                "lobpcg_iters": sum(i["iters"] for i in self.infos)}

    def objective(self):
        """1/4 <L, X> at the current (relaxed) primal iterate."""
        return float(0.25 * (self.L * self.X).sum())

    def close(self):
        self.ctx.close()
