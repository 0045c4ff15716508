"""paper_1912_02767_b200 -- B200-native warm-started LOBPCG projection onto the PSD cone
(arXiv:1912.02767). The product path is libpsdproj.so (sm_100a kernels + C ABI,
include/psdproj.h); this package holds its sources (csrc/), the nvcc build (build.py) and a
thin ctypes binding (api.py). Importing the API loads the shared library and raises if it is
missing -- there is no CPU fallback.
"""
from . import _lib  # noqa: F401


def build(force=False):
    from .build import build as _build
    return _build(force=force)
