"""ctypes declarations of include/psdproj.h (argument marshalling only).

Loads the in-tree libpsdproj.so built by build.py. There is no fallback: if the shared
library is missing or fails to load, import of the API raises.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libpsdproj.so")

OK, NOT_CONVERGED = 0, 1
E_INVALID, E_NONFINITE, E_CUDA, E_DEGENERATE, E_NCCL, E_WORKSPACE, E_CAPACITY = -1, -2, -3, -4, -5, -6, -7
SIDE_AUTO, SIDE_POS, SIDE_NEG, SIDE_DIRECT = 0, 1, -1, 2
LOCK_SOFT, LOCK_HARD = 1, 2

# every symbol include/psdproj.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "psdproj_default_params", "psdproj_workspace_bytes", "psdproj_create", "psdproj_project",
    "psdproj_project_host", "psdproj_project_batched", "psdproj_project_tiny_batched", "psdproj_get_ritz", "psdproj_reset",
    "psdproj_destroy", "psdproj_last_error", "psdproj_dgemm", "psdproj_jacobi_ws_elems",
    "psdproj_jacobi", "psdproj_philox_raw", "psdproj_philox_gauss", "psdproj_eigh_ws_elems",
    "psdproj_eigh", "psdproj_cholesky", "psdproj_get_nccl_uid", "psdproj_workspace_bytes_sharded",
    "psdproj_create_sharded", "psdproj_admm_maxcut_step1", "psdproj_admm_maxcut_step2",
    "psdproj_admm_certificate_terms", "psdproj_symm_multiply", "psdproj_tiny_lobpcg_ws_bytes",
    "psdproj_project_tiny_lobpcg",
]


class Params(ctypes.Structure):
    _fields_ = [
        ("max_iter", ctypes.c_int), ("m0", ctypes.c_int), ("expand_q", ctypes.c_int),
        ("guard", ctypes.c_int), ("side", ctypes.c_int), ("locking", ctypes.c_int),
        ("keep_extra", ctypes.c_int), ("m_max", ctypes.c_int), ("seed", ctypes.c_uint64),
        ("ctx_id", ctypes.c_uint32), ("profile", ctypes.c_int), ("host_io", ctypes.c_int),
        ("perp_steps", ctypes.c_int), ("perp_delta", ctypes.c_double), ("lock_factor", ctypes.c_double),
        ("krylov_depth", ctypes.c_int), ("guard_active", ctypes.c_int),
        ("krylov_max_active", ctypes.c_int),
    ]


class Info(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int), ("side", ctypes.c_int), ("iters", ctypes.c_int), ("m", ctypes.c_int),
        ("npos", ctypes.c_int), ("expansions", ctypes.c_int), ("a_passes", ctypes.c_int),
        ("cold", ctypes.c_int), ("rr_max", ctypes.c_int), ("locked", ctypes.c_int),
        ("a_cols", ctypes.c_longlong), ("err_bound", ctypes.c_double), ("resid_fro", ctypes.c_double),
        ("resid_max", ctypes.c_double), ("lock_defect", ctypes.c_double), ("anorm_f", ctypes.c_double),
        ("flops", ctypes.c_double), ("bytes", ctypes.c_double), ("amul_flops", ctypes.c_double),
        ("amul_bytes", ctypes.c_double), ("amul_ms", ctypes.c_double), ("amul_launches", ctypes.c_int),
        ("last_pos", ctypes.c_int), ("last_neg", ctypes.c_int), ("launches", ctypes.c_int),
        ("dropped", ctypes.c_int), ("phase_ms", ctypes.c_double * 12), ("perp_est", ctypes.c_double),
        ("orth_defect", ctypes.c_double), ("perp_mu", ctypes.c_double), ("tri_ms", ctypes.c_double),
        ("tri_launches", ctypes.c_int), ("tri_flops", ctypes.c_double), ("pi_fro", ctypes.c_double),
    ]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["phase_ms"] = list(self.phase_ms)
        return d


_lib = None


def load(path=SO_PATH):
    """Load libpsdproj.so (raises OSError if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"libpsdproj.so not built at {path}; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    vp, i, d, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
    u32, u64 = ctypes.c_uint32, ctypes.c_uint64
    P = ctypes.POINTER
    L.psdproj_default_params.argtypes = [P(Params)]
    L.psdproj_default_params.restype = None
    L.psdproj_workspace_bytes.argtypes = [i, P(Params)]
    L.psdproj_workspace_bytes.restype = sz
    L.psdproj_create.argtypes = [i, P(Params), vp, sz, P(vp)]
    L.psdproj_project.argtypes = [vp, vp, i, vp, i, d, vp, P(Info)]
    L.psdproj_project_host.argtypes = [vp, vp, i, vp, i, d, vp, P(Info)]
    L.psdproj_project_batched.argtypes = [P(vp), i, P(vp), P(i), P(vp), P(i), P(d), vp, P(Info)]
    L.psdproj_project_tiny_batched.argtypes = [i, P(i), P(vp), P(i), P(vp), P(i), P(i), vp]
    L.psdproj_get_ritz.argtypes = [vp, P(d), i, vp, i]
    L.psdproj_reset.argtypes = [vp]
    L.psdproj_destroy.argtypes = [vp]
    L.psdproj_last_error.argtypes = []
    L.psdproj_last_error.restype = ctypes.c_char_p
    L.psdproj_dgemm.argtypes = [i, i, i, i, i, d, vp, i, vp, i, d, vp, i, vp, sz, vp]
    L.psdproj_tiny_lobpcg_ws_bytes.argtypes = [i]
    L.psdproj_tiny_lobpcg_ws_bytes.restype = sz
    L.psdproj_project_tiny_lobpcg.argtypes = [i, P(i), P(vp), P(i), P(vp), P(i), P(vp), P(i), d, i, i, i, u64, u32,
                                              vp, sz, P(i), P(i), P(i), P(d), vp]
    L.psdproj_symm_multiply.argtypes = [i, i, d, vp, i, vp, i, vp, i, vp, sz, vp]
    L.psdproj_jacobi_ws_elems.argtypes = [i]
    L.psdproj_jacobi_ws_elems.restype = sz
    L.psdproj_jacobi.argtypes = [i, vp, i, vp, vp, i, vp, vp]
    L.psdproj_eigh_ws_elems.argtypes = [i, i]
    L.psdproj_eigh_ws_elems.restype = sz
    L.psdproj_eigh.argtypes = [i, vp, i, i, vp, vp, i, vp, vp, vp]
    L.psdproj_cholesky.argtypes = [i, vp, i, vp]
    L.psdproj_get_nccl_uid.argtypes = [vp]
    L.psdproj_admm_maxcut_step1.argtypes = [i, vp, vp, vp, vp, vp, i, d, d, d, vp, vp, vp, vp, vp, vp]
    L.psdproj_admm_maxcut_step2.argtypes = [i, vp, vp, vp, vp, vp, vp, vp, i, d, P(d), vp, vp, vp]
    L.psdproj_admm_certificate_terms.argtypes = [i, vp, vp, vp, vp, vp, vp, vp, i, vp, vp, vp, vp, vp, sz, P(d), vp]
    L.psdproj_workspace_bytes_sharded.argtypes = [i, i, i, P(Params)]
    L.psdproj_workspace_bytes_sharded.restype = sz
    L.psdproj_create_sharded.argtypes = [i, i, i, vp, i, i, P(Params), vp, sz, P(vp)]
    L.psdproj_philox_raw.argtypes = [i, u32, u32, u32, u32, u32, vp, vp]
    L.psdproj_philox_gauss.argtypes = [i, i, vp, i, u64, u32, u32, u32, vp]
    special = ("psdproj_default_params", "psdproj_workspace_bytes", "psdproj_last_error", "psdproj_tiny_lobpcg_ws_bytes",
               "psdproj_jacobi_ws_elems", "psdproj_eigh_ws_elems", "psdproj_workspace_bytes_sharded")
    for name in EXPORTS:
        if name not in special:
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def last_error():
    return load().psdproj_last_error().decode()


class PsdprojError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where} failed with code {code}: {last_error()}")
        self.code = code


def check(rc, where):
    if rc < 0:
        raise PsdprojError(rc, where)
    return rc
