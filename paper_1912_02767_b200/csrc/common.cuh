// common.cuh -- shared helpers for the psdproj CUDA path (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "psdproj is built for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

#define PSD_U 1.1102230246251565e-16  // unit roundoff 2^-53

namespace psd {

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Column-major element access.
#define IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))

// GvL Alg. 8.5.2 (sym.schur2) with the exact-annihilation update (see oracle/jacobi.c for
// the CPU restatement; the two are written independently).
__device__ __forceinline__ void schur2(double app, double apq, double aqq, double& c, double& s,
                                       double& t) {
  // tau = (aqq - app) / (2 apq), t = sign(tau) / (|tau| + sqrt(1 + tau^2)) rewritten with
  // d = aqq - app, e = 2 apq as t = sgn(d) e / (|d| + hypot(d, e)) (one division, one sqrt)
  double d = aqq - app, e = 2.0 * apq;
  double h = sqrt(fma(d, d, e * e));
  t = (d >= 0.0 ? e : -e) / (fabs(d) + h);
  c = rsqrt(fma(t, t, 1.0));
  s = t * c;
}

}  // namespace psd
