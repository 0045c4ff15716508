"""Thin Python binding over the psdproj C ABI (same names; marshalling only).

Every step of the projection runs in libpsdproj.so's sm_100a kernels; torch supplies the
device memory (workspace, A, Pi) and the stream. Column-major convention: a torch tensor
M of shape (r, c) with M.stride(0) == 1 is an r x c column-major matrix with ld = M.stride(1);
symmetric matrices may be passed in either layout.
"""
import ctypes

import torch

from . import _lib
from ._lib import Info, Params, PsdprojError, check

__all__ = ["Context", "ShardedContext", "TinyLobpcgBatch", "default_params", "project_batched", "dgemm", "jacobi",
           "philox_raw",
           "philox_gauss", "workspace_bytes", "colmajor", "colmajor_copy", "nccl_uid", "row_blocks"]


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def colmajor(r, c, device="cuda", ld=None):
    """Allocate an r x c column-major fp64 matrix (torch view with stride (1, ld))."""
    ld = ld or r
    return torch.zeros(c, ld, dtype=torch.float64, device=device).T[:r, :]


def _ld_colmajor(M):
    if M.dim() != 2 or M.dtype != torch.float64:
        raise ValueError("expected a 2-D float64 tensor")
    if M.stride(0) == 1:
        return max(M.stride(1), M.shape[0]) if M.shape[1] > 1 else max(M.shape[0], 1)
    raise ValueError("matrix must be column-major (stride(0) == 1)")


def _ld_sym(A):
    """Leading dimension of a symmetric matrix in either layout."""
    if A.dim() != 2 or A.shape[0] != A.shape[1] or A.dtype != torch.float64:
        raise ValueError("expected a square float64 matrix")
    if A.stride(1) == 1:
        return A.stride(0) if A.shape[0] > 1 else 1
    if A.stride(0) == 1:
        return A.stride(1) if A.shape[0] > 1 else 1
    raise ValueError("A must have a unit stride in one dimension")


def default_params(**kw):
    p = Params()
    _lib.load().psdproj_default_params(ctypes.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p


def workspace_bytes(n, params=None):
    return int(_lib.load().psdproj_workspace_bytes(n, ctypes.byref(params) if params is not None else None))


class Context:
    """psdproj_create / psdproj_project / psdproj_reset / psdproj_destroy over a torch-owned
    device workspace. One context per cone block; it carries the warm block between calls."""

    def __init__(self, n, params=None, device="cuda", **kw):
        L = _lib.load()
        self.n = n
        self.params = params if params is not None else default_params(**kw)
        nbytes = workspace_bytes(n, self.params)
        self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
        base = self.ws.data_ptr()
        off = (-base) % 256
        self._h = ctypes.c_void_p()
        check(L.psdproj_create(n, ctypes.byref(self.params), ctypes.c_void_p(base + off), nbytes,
                               ctypes.byref(self._h)), "psdproj_create")

    def project(self, A, tol, out=None, stream=None):
        """Pi(A) for a device fp64 symmetric matrix A; returns (Pi, info dict). out may be A."""
        L = _lib.load()
        n = self.n
        if A.shape != (n, n) or not A.is_cuda:
            raise ValueError(f"A must be a CUDA ({n}, {n}) float64 tensor")
        lda = _ld_sym(A)
        if out is None:
            out = torch.empty_like(A)
        ldo = _ld_sym(out)
        info = Info()
        rc = L.psdproj_project(self._h, _ptr(A), lda, _ptr(out), ldo, float(tol), _stream_ptr(stream),
                               ctypes.byref(info))
        check(rc, "psdproj_project")
        return out, info.as_dict()

    def project_host(self, A_host, tol, out_host=None, stream=None):
        """End-to-end call with HOST A / Pi (the copies happen inside the C call)."""
        L = _lib.load()
        n = self.n
        if A_host.is_cuda:
            raise ValueError("project_host takes host tensors")
        lda = _ld_sym(A_host)
        if out_host is None:
            out_host = torch.empty_like(A_host)
        info = Info()
        rc = L.psdproj_project_host(self._h, _ptr(A_host), lda, _ptr(out_host), _ld_sym(out_host),
                                    float(tol), _stream_ptr(stream), ctypes.byref(info))
        check(rc, "psdproj_project_host")
        return out_host, info.as_dict()

    def get_ritz(self, cap=None, with_vectors=False):
        L = _lib.load()
        cap = cap or self.n
        vals = (ctypes.c_double * cap)()
        vecs = colmajor(self.n, cap) if with_vectors else None
        k = check(L.psdproj_get_ritz(self._h, vals, cap, _ptr(vecs) if vecs is not None else None,
                                     self.n), "psdproj_get_ritz")
        v = torch.tensor(list(vals)[:k], dtype=torch.float64)
        return (v, vecs[:, :k]) if with_vectors else v

    def reset(self):
        check(_lib.load().psdproj_reset(self._h), "psdproj_reset")

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().psdproj_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h


def nccl_uid():
    """128-byte NCCL unique id for psdproj_create_sharded (rank 0 creates it, then broadcasts)."""
    buf = ctypes.create_string_buffer(128)
    check(_lib.load().psdproj_get_nccl_uid(buf), "psdproj_get_nccl_uid")
    return buf.raw


def row_blocks(n, world):
    """Contiguous, balanced row blocks (offset, rows) of the row-sharded mode, rank order."""
    base, extra = divmod(n, world)
    out, off = [], 0
    for r in range(world):
        rows = base + (1 if r < extra else 0)
        out.append((off, rows))
        off += rows
    return out


def colmajor_copy(M):
    """Column-major (stride(0) == 1) copy of a 2-D float64 tensor."""
    out = colmajor(M.shape[0], M.shape[1], device=M.device)
    out.copy_(M)
    return out


class ShardedContext:
    """psdproj_create_sharded: rank `rank` of `world` holds rows [row0, row0 + nrows) of every
    n x n input (a column-major nrows x n block) and gets the same rows of Pi. All ranks call
    project() collectively (NCCL inside the library, on the current stream)."""

    def __init__(self, n, row0, nrows, uid, rank, world, params=None, device="cuda", nrows_max=None, **kw):
        L = _lib.load()
        self.n, self.row0, self.nrows = n, row0, nrows
        self.params = params if params is not None else default_params(**kw)
        nrmax = nrows_max or max(r for _, r in row_blocks(n, world))
        nbytes = int(L.psdproj_workspace_bytes_sharded(n, nrmax, world, ctypes.byref(self.params)))
        self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=device)
        base = self.ws.data_ptr()
        off = (-base) % 256
        self._h = ctypes.c_void_p()
        ub = ctypes.create_string_buffer(bytes(uid), 128)
        check(L.psdproj_create_sharded(n, row0, nrows, ub, rank, world, ctypes.byref(self.params),
                                       ctypes.c_void_p(base + off), nbytes, ctypes.byref(self._h)),
              "psdproj_create_sharded")

    def project(self, A_local, tol, out=None, stream=None):
        L = _lib.load()
        if A_local.shape != (self.nrows, self.n) or not A_local.is_cuda:
            raise ValueError(f"A_local must be a CUDA ({self.nrows}, {self.n}) float64 tensor")
        lda = _ld_colmajor(A_local)
        if out is None:
            out = colmajor(self.nrows, self.n, device=A_local.device)
        info = Info()
        rc = L.psdproj_project(self._h, _ptr(A_local), lda, _ptr(out), _ld_colmajor(out), float(tol),
                               _stream_ptr(stream), ctypes.byref(info))
        check(rc, "psdproj_project (sharded)")
        return out, info.as_dict()

    def reset(self):
        check(_lib.load().psdproj_reset(self._h), "psdproj_reset")

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().psdproj_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def project_batched(ctxs, As, tols, outs=None, stream=None):
    """psdproj_project_batched over independent contexts (one per block)."""
    L = _lib.load()
    k = len(ctxs)
    outs = outs if outs is not None else [torch.empty_like(a) for a in As]
    H = (ctypes.c_void_p * k)(*[c.handle.value for c in ctxs])
    Ap = (ctypes.c_void_p * k)(*[a.data_ptr() for a in As])
    Op = (ctypes.c_void_p * k)(*[o.data_ptr() for o in outs])
    la = (ctypes.c_int * k)(*[_ld_sym(a) for a in As])
    lo = (ctypes.c_int * k)(*[_ld_sym(o) for o in outs])
    tl = (ctypes.c_double * k)(*[float(t) for t in tols])
    infos = (Info * k)()
    rc = L.psdproj_project_batched(H, k, Ap, la, Op, lo, tl, _stream_ptr(stream), infos)
    check(rc, "psdproj_project_batched")
    return outs, [inf.as_dict() for inf in infos]


def project_tiny_batched(As, outs=None, stream=None):
    """psdproj_project_tiny_batched: exact projections of many tiny blocks (n <= 112) in one launch.
    Returns (outs, npos list)."""
    L = _lib.load()
    k = len(As)
    outs = outs if outs is not None else [torch.empty_like(a) for a in As]
    ns = (ctypes.c_int * k)(*[a.shape[0] for a in As])
    Ap = (ctypes.c_void_p * k)(*[a.data_ptr() for a in As])
    Op = (ctypes.c_void_p * k)(*[o.data_ptr() for o in outs])
    la = (ctypes.c_int * k)(*[_ld_sym(a) for a in As])
    lo = (ctypes.c_int * k)(*[_ld_sym(o) for o in outs])
    npos = (ctypes.c_int * k)()
    check(L.psdproj_project_tiny_batched(k, ns, Ap, la, Op, lo, npos, _stream_ptr(stream)),
          "psdproj_project_tiny_batched")
    return outs, list(npos)


class TinyLobpcgBatch:
    """f4: many tiny blocks (n <= 112) each projected by a one-CTA warm LOBPCG in one launch
    (psdproj_project_tiny_lobpcg). Holds the per-block warm blocks (device, n x 8) and widths."""

    def __init__(self, sizes, device="cuda", guard=1, m0=2, seed=0x5eed1912, max_iter=500):
        L = _lib.load()
        self.sizes = [int(n) for n in sizes]
        self.count = len(self.sizes)
        self.guard, self.m0, self.seed, self.max_iter = guard, m0, seed, max_iter
        self.Xw = [torch.zeros(8, n, dtype=torch.float64, device=device).T for n in self.sizes]  # n x 8, ld n
        self.m_state = (ctypes.c_int * self.count)()
        nb = int(L.psdproj_tiny_lobpcg_ws_bytes(self.count))
        self.ws = torch.empty(nb + 256, dtype=torch.uint8, device=device)
        self.calls = 0

    def project(self, As, tol, outs=None, stream=None):
        """Returns (outs, dict of per-block status / iters / npos / bound lists)."""
        L = _lib.load()
        k = self.count
        outs = outs if outs is not None else [torch.empty_like(a) for a in As]
        ns = (ctypes.c_int * k)(*self.sizes)
        Ap = (ctypes.c_void_p * k)(*[a.data_ptr() for a in As])
        Op = (ctypes.c_void_p * k)(*[o.data_ptr() for o in outs])
        Xp = (ctypes.c_void_p * k)(*[x.data_ptr() for x in self.Xw])
        la = (ctypes.c_int * k)(*[_ld_sym(a) for a in As])
        lo = (ctypes.c_int * k)(*[_ld_sym(o) for o in outs])
        st, it, npos = (ctypes.c_int * k)(), (ctypes.c_int * k)(), (ctypes.c_int * k)()
        bd = (ctypes.c_double * k)()
        base = self.ws.data_ptr()
        off = (-base) % 256
        check(L.psdproj_project_tiny_lobpcg(k, ns, Ap, la, Op, lo, Xp, self.m_state, float(tol), self.max_iter,
                                            self.guard, self.m0, self.seed, self.calls, ctypes.c_void_p(base + off),
                                            self.ws.numel() - off, st, it, npos, bd, _stream_ptr(stream)),
              "psdproj_project_tiny_lobpcg")
        self.calls += 1
        return outs, {"status": list(st), "iters": list(it), "npos": list(npos), "bound": list(bd)}


def dgemm(opA, opB, alpha, A, B, beta, C, ws=None, stream=None):
    """C = alpha op(A) op(B) + beta C on column-major device tensors (psdproj_dgemm)."""
    L = _lib.load()
    M, N = C.shape
    K = A.shape[1] if opA == 0 else A.shape[0]
    ws_elems = ws.numel() if ws is not None else 0
    rc = L.psdproj_dgemm(opA, opB, M, N, K, float(alpha), _ptr(A), _ld_colmajor(A), _ptr(B), _ld_colmajor(B),
                         float(beta), _ptr(C), _ld_colmajor(C), _ptr(ws) if ws is not None else None, ws_elems,
                         _stream_ptr(stream))
    check(rc, "psdproj_dgemm")
    return C


def symm_multiply(alpha, A, Z, Y=None, ws=None, stream=None):
    """Y = alpha A Z for a symmetric device matrix A (the path's TMA a3 kernel, psdproj_symm_multiply)."""
    L = _lib.load()
    n, k = Z.shape
    Y = Y if Y is not None else colmajor(n, k, device=Z.device)
    rc = L.psdproj_symm_multiply(n, k, float(alpha), _ptr(A), _ld_sym(A), _ptr(Z), _ld_colmajor(Z), _ptr(Y),
                                 _ld_colmajor(Y), _ptr(ws) if ws is not None else None,
                                 ws.numel() if ws is not None else 0, _stream_ptr(stream))
    check(rc, "psdproj_symm_multiply")
    return Y


def jacobi(A, stream=None):
    """Eigendecomposition by the path's Jacobi kernels: returns (w unsorted, V, sweeps)."""
    L = _lib.load()
    s = A.shape[0]
    w = torch.empty(s, dtype=torch.float64, device=A.device)
    V = colmajor(s, s, device=A.device)
    ws = torch.empty(int(L.psdproj_jacobi_ws_elems(s)), dtype=torch.float64, device=A.device)
    sweeps = check(L.psdproj_jacobi(s, _ptr(A), _ld_sym(A), _ptr(w), _ptr(V), s, _ptr(ws), _stream_ptr(stream)),
                   "psdproj_jacobi")
    return w, V, sweeps


def eigh(A, m=None, stream=None):
    """Top-m eigenpairs (descending) by the path's tridiagonal eigensolver: (w, V, npos)."""
    L = _lib.load()
    s = A.shape[0]
    m = s if m is None else m
    w = torch.empty(max(m, 1), dtype=torch.float64, device=A.device)
    V = colmajor(s, max(m, 1), device=A.device)
    npos = torch.zeros(1, dtype=torch.int32, device=A.device)
    ws = torch.empty(int(L.psdproj_eigh_ws_elems(s, m)), dtype=torch.float64, device=A.device)
    check(L.psdproj_eigh(s, _ptr(A), _ld_sym(A), m, _ptr(w), _ptr(V), s, _ptr(npos), _ptr(ws), _stream_ptr(stream)),
          "psdproj_eigh")
    return w[:m], V[:, :m], int(npos.item())


def cholesky(G, stream=None):
    """In-place Cholesky of the path (a6) on a column-major copy of G: (L, status)."""
    L_ = _lib.load()
    t = G.shape[0]
    M = colmajor(t, t, device=G.device)
    M.copy_(G)
    rc = check(L_.psdproj_cholesky(t, _ptr(M), t, _stream_ptr(stream)), "psdproj_cholesky")
    return M, rc


def philox_raw(count, c1, c2, c3, k0, k1, device="cuda", stream=None):
    L = _lib.load()
    out = torch.empty(4 * count, dtype=torch.int32, device=device)
    check(L.psdproj_philox_raw(count, c1, c2, c3, k0, k1, _ptr(out), _stream_ptr(stream)), "psdproj_philox_raw")
    return out


def philox_gauss(n, q, seed, stream_id, ctx=0, tag=0, device="cuda", stream=None):
    L = _lib.load()
    out = colmajor(n, q, device=device)
    check(L.psdproj_philox_gauss(n, q, _ptr(out), n, seed, stream_id, ctx, tag, _stream_ptr(stream)),
          "psdproj_philox_gauss")
    return out
