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


class DiagSDPADMM:
    """Alg. 1 on  min <Q, X>  s.t.  X_ii = b_i (i with w_i = 1),  X PSD  (b, w default to ones).
    f3: `certificates()` evaluates Theorem 1's infeasibility certificates in the
    practical form of PAPER.md:563-587 (reading R49) from the last two iterates; `solve(...,
    check_every=40)` stops on a certificate (status 'primal_infeasible' / 'dual_infeasible')."""

    def __init__(self, Q, b=None, w=None, rho=0.1, sigma=1e-6, alpha=1.6, device="cuda", params=None, tol_floor=0.0,
                 tol_override=None, adapt_every=0, adapt_ratio=5.0, tol_ratio=0.0):
        n = Q.shape[0]
        self.n, self.rho, self.sigma, self.alpha = n, float(rho), float(sigma), float(alpha)
        self.adapt_every, self.adapt_ratio = int(adapt_every), float(adapt_ratio)
        self.tol_ratio = float(tol_ratio)
        self.last_res = None
        self.rho_history = [(0, self.rho)]
        self.tol_floor, self.tol_override = tol_floor, tol_override
        dev = torch.device(device)
        self.Q = torch.as_tensor(Q, dtype=torch.float64, device=dev).contiguous()
        vec = lambda v: None if v is None else torch.as_tensor(v, dtype=torch.float64, device=dev).contiguous()  # noqa: E731
        self.b, self.w = vec(b), vec(w)
        z = lambda: torch.zeros(n, n, dtype=torch.float64, device=dev)  # noqa: E731
        self.X, self.Zp, self.Yp, self.Zh, self.V = z(), z(), z(), z(), z()
        self.ye = torch.zeros(n, dtype=torch.float64, device=dev)
        self.zeh = torch.zeros(n, dtype=torch.float64, device=dev)
        self.ctx = api.Context(n, params=params if params is not None else api.default_params(seed=1912))
        self.k = 0
        self.infos = []
        self.prev = None
        self._cert_ctx = None

    def step(self, save_prev=False):
        """One iteration of Alg. 1; returns (r_prim, r_dual, projection info)."""
        L_ = _lib.load()
        n, st = self.n, api._stream_ptr(None)
        p = api._ptr
        pb = p(self.b) if self.b is not None else None
        pw = p(self.w) if self.w is not None else None
        if save_prev:
            self.prev = (self.X.clone(), self.ye.clone(), self.Yp.clone())
        check(L_.psdproj_admm_maxcut_step1(n, p(self.X), p(self.Zp), p(self.Yp), p(self.ye), p(self.Q), n,
                                           self.sigma, self.rho, self.alpha, p(self.Zh), p(self.V), p(self.zeh),
                                           pb, pw, st), "psdproj_admm_maxcut_step1")
        self.k += 1
        tol = self.tol_override if self.tol_override is not None else max(tol_schedule(self.k), self.tol_floor)
        if self.tol_override is None and self.tol_ratio > 0 and self.last_res is not None:
            # R59: never looser than tol_ratio x the current ADMM residual (the paper's summable schedule
            # 10/k^1.01, stays the upper bound)
            tol = min(tol, max(self.tol_ratio * min(self.last_res), 1e-12))
        _, info = self.ctx.project(self.V, tol, out=self.Zp)
        res = (ctypes.c_double * 3)()
        check(L_.psdproj_admm_maxcut_step2(n, p(self.X), p(self.Zp), p(self.Zh), p(self.Yp), p(self.ye),
                                           p(self.zeh), p(self.Q), n, self.rho, res, pb, pw, st),
              "psdproj_admm_maxcut_step2")
        self.infos.append(info)
        r_p, r_d = max(res[0], res[1]), res[2]
        self.last_res = (r_p, r_d)
        self._adapt(r_p, r_d)
        return r_p, r_d, info

    def _adapt(self, r_p, r_d):
        """Reading R58 (COSMO-style residual balancing; the paper runs COSMO.jl): every
        `adapt_every` iterations (0 = fixed rho), if one residual exceeds the other by more than
        `adapt_ratio`, rho <- rho sqrt(r_prim / r_dual), clipped to [1e-6, 1e6]. Line 3's matrix
        sigma I + rho A^T A is diagonal here, so a new rho costs nothing; y is kept."""
        if self.adapt_every <= 0 or self.k % self.adapt_every or not (r_p > 0 and r_d > 0):
            return
        ratio = r_p / r_d
        if ratio > self.adapt_ratio or ratio < 1.0 / self.adapt_ratio:
            self.rho = min(1e6, max(1e-6, self.rho * ratio ** 0.5))
            self.rho_history.append((self.k, self.rho))

    def _psd_part(self, M):
        """||Pi_S+(M)||_F of a symmetric device matrix by the library's DIRECT path (exact
        eigendecomposition; info pi_fro = sqrt of the sum of the squared positive eigenvalues)."""
        if self._cert_ctx is None:
            self._cert_ctx = api.Context(self.n, params=api.default_params(side=2))
            self._cert_out = torch.empty_like(M)
        _, info = self._cert_ctx.project(M, 1e-12, out=self._cert_out)
        return info["pi_fro"]

    def certificates(self):
        """Theorem 1's certificates from the successive differences of the last step (needs
        step(save_prev=True)), reading R49. The terms are formed on the device in one pass
        (psdproj_admm_certificate_terms) and the two PSD-part distances by the DIRECT projection;
        only the normalisation of a few scalars happens here. With y = (w ye, Yp), x = vec(X):
          primal: ||A^T y-bar||_inf, dist_{C-polar}(y-bar) = ||Pi_S+(Y-bar)||_F, b^T y-bar_eq
          dual:   dist_{C-inf}(A x-bar) = (||w diag X-bar||^2 + ||Pi_S+(-X-bar)||_F^2)^(1/2), <Q, X-bar>"""
        L_ = _lib.load()
        X0, ye0, Yp0 = self.prev
        n, p = self.n, api._ptr
        if not hasattr(self, "_cert_buf"):
            self._cert_buf = (torch.empty_like(self.X), torch.empty_like(self.X),
                              torch.empty(7 * (2 * 148 * 4 + 1), dtype=torch.float64, device=self.X.device))
        dYs, mdXs, work = self._cert_buf
        t = (ctypes.c_double * 7)()
        check(L_.psdproj_admm_certificate_terms(n, p(self.X), p(X0), p(self.ye), p(ye0), p(self.Yp), p(Yp0),
                                                p(self.Q), n, p(self.b) if self.b is not None else None,
                                                p(self.w) if self.w is not None else None, p(dYs), p(mdXs),
                                                p(work), work.numel(), t, api._stream_ptr(None)),
              "psdproj_admm_certificate_terms")
        ndx, ndy = t[0] ** 0.5, (t[1] + t[2]) ** 0.5
        out = {"ndx": ndx, "ndy": ndy}
        if ndy > 1e-12:
            out["p_at"] = t[6] / ndy
            out["p_dist"] = self._psd_part(dYs) / ndy      # positive homogeneity of Pi_S+
            out["p_supp"] = t[3] / ndy
        if ndx > 1e-12:
            out["d_dist"] = (t[5] + self._psd_part(mdXs) ** 2) ** 0.5 / ndx
            out["d_qx"] = t[4] / ndx
        return out

    @staticmethod
    def infeasible(cert, eps_pinf=1e-4, eps_dinf=1e-4):
        """R49: primal if ||A^T y-bar|| < eps, dist < eps and the support b^T y-bar < -eps; dual if
        dist < eps and q^T x-bar < -eps (Theorem 1's strict inequalities)."""
        p = "p_at" in cert and cert["p_at"] < eps_pinf and cert["p_dist"] < eps_pinf and cert["p_supp"] < -eps_pinf
        d = "d_dist" in cert and cert["d_dist"] < eps_dinf and cert["d_qx"] < -eps_dinf
        return p, d

    def solve(self, eps=1e-4, max_iter=5000, check_every=0, eps_pinf=1e-4, eps_dinf=1e-4):
        r_p = r_d = float("inf")
        status, cert = "max_iter", None
        while self.k < max_iter:
            chk = check_every > 0 and (self.k + 1) % check_every == 0
            r_p, r_d, _ = self.step(save_prev=chk)
            if r_p <= eps and r_d <= eps:
                status = "solved"
                break
            if chk:
                cert = self.certificates()
                pinf, dinf = self.infeasible(cert, eps_pinf, eps_dinf)
                if pinf or dinf:
                    status = "primal_infeasible" if pinf else "dual_infeasible"
                    if pinf and dinf:
                        status = "primal_dual_infeasible"
                    break
        return {"iters": self.k, "r_prim": r_p, "r_dual": r_d, "objective": self.objective(), "status": status,
                "certificates": cert, "lobpcg_iters": sum(i["iters"] for i in self.infos)}

    def objective(self):
        """<Q, X> at the current (relaxed) primal iterate."""
        return float((self.Q * self.X).sum())

    def close(self):
        self.ctx.close()
        if self._cert_ctx is not None:
            self._cert_ctx.close()


class MaxCutADMM(DiagSDPADMM):
    """MaxCut SDP (BASELINE configs[4]): max 1/4 <L, X> s.t. diag(X) = 1, X PSD."""

    def __init__(self, L, **kw):
        self.L = torch.as_tensor(L, dtype=torch.float64, device=kw.get("device", "cuda"))
        super().__init__(-0.25 * self.L, **kw)

    def objective(self):
        """1/4 <L, X> at the current (relaxed) primal iterate."""
        return float(0.25 * (self.L * self.X).sum())
