// tridiag.cuh -- dense symmetric eigensolver for the Rayleigh-Ritz step (a7) and the DIRECT path
// (a13): Householder tridiagonalisation (one CTA) -> parallel multisection bisection for the
// wanted eigenvalues (one warp each) -> inverse iteration (one thread per vector) with
// modified Gram-Schmidt inside clusters -> back-transformation by the reflectors (one CTA per
// column group).
//
// Why not Jacobi on the GPU: every Jacobi round is a barrier-separated step and a solve needs
// ~10 s rounds; tridiagonalisation needs s steps, and the remaining stages are embarrassingly
// parallel over eigenpairs (measured in DESIGN.md §6).
//
// References: GvL 4th ed. Alg. 8.3.1 (Householder tridiagonalisation), §8.4.1 (Sturm/bisection),
// §8.4.2-8.4.3 (inverse iteration), LAPACK dstein's clustering rule (ORTOL = 1e-3 ||T||).
#pragma once
#include "common.cuh"

namespace psd {

constexpr int TRI_SMEM_MAX = 160;  // 160 x 161 doubles = 206 KB of shared memory

template <int NT>
__device__ __forceinline__ double tri_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < NT / 32) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

// Householder tridiagonalisation of the symmetric s x s matrix A (lda).
// Outputs: d[s], e[s-1] (sub-diagonal), tau[s-2], reflectors Vh (s x s, ldv): column j holds
// v_j with v_j[j+1] = 1 and v_j[i] = 0 for i <= j. Works in shared memory when s <= TRI_SMEM_MAX,
// otherwise in the global scratch G (s x s, ldg) -- A is never modified.
template <int NT>
__global__ void __launch_bounds__(NT) tridiag_kernel(int s, const double* __restrict__ A, int lda,
                                                     double* __restrict__ d, double* __restrict__ e,
                                                     double* __restrict__ tau, double* __restrict__ Vh, int ldv,
                                                     double* __restrict__ G, int ldg) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[33];
  __shared__ double sh_scale, sh_tau;
  const bool in_smem = s <= TRI_SMEM_MAX;
  const int L = in_smem ? (s + 1) : ldg;
  double* M = in_smem ? sm : G;
  double* sv = in_smem ? sm + (size_t)s * (s + 1) : sm;  // dynamic: [M (smem mode)] sv[s] sp[s + 8 s]
  double* sp = sv + s;
  for (int e2 = threadIdx.x; e2 < s * s; e2 += NT) {
    int i = e2 % s, j = e2 / s;
    M[i + (size_t)j * L] = 0.5 * (A[IDX(i, j, lda)] + A[IDX(j, i, lda)]);
  }
  for (int e2 = threadIdx.x; e2 < s * s; e2 += NT) {
    int i = e2 % s, j = e2 / s;
    Vh[IDX(i, j, ldv)] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j + 2 < s; ++j) {
    const int t = s - j - 1;  // trailing size
    double* col = M + (j + 1) + (size_t)j * L;
    // sigma = ||x(1:)||^2 of the column below the sub-diagonal
    double acc = 0.0;
    for (int i = 1 + threadIdx.x; i < t; i += NT) acc += col[i] * col[i];
    double sigma = tri_block_sum<NT>(acc, red);
    if (threadIdx.x == 0) {
      double alpha = col[0];
      double tj, beta, scale;
      if (sigma == 0.0) {
        tj = 0.0;
        beta = alpha;
        scale = 0.0;
      } else {
        double mu = sqrt(alpha * alpha + sigma);
        beta = (alpha <= 0.0) ? mu : -mu;
        double v0 = alpha - beta;
        tj = (beta - alpha) / beta;
        scale = 1.0 / v0;
      }
      d[j] = M[j + (size_t)j * L];
      e[j] = beta;
      tau[j] = tj;
      sh_scale = scale;
      sh_tau = tj;
    }
    __syncthreads();
    const double tj = sh_tau;
    if (tj == 0.0) {  // nothing to annihilate: H_j = I
      for (int i = threadIdx.x; i < t; i += NT) Vh[IDX(j + 1 + i, j, ldv)] = (i == 0) ? 1.0 : 0.0;
      __syncthreads();
      continue;
    }
    const double scale = sh_scale;
    for (int i = threadIdx.x; i < t; i += NT) {
      double v = (i == 0) ? 1.0 : col[i] * scale;
      sv[i] = v;
      Vh[IDX(j + 1 + i, j, ldv)] = v;
    }
    __syncthreads();
    // p = tau * A22 v: warp (rb, cc) sums rows [32 rb, 32 rb + 32) over column chunk cc;
    // lanes are consecutive rows (conflict-free column reads), sv[c] is a broadcast.
    double* A22 = M + (j + 1) + (size_t)(j + 1) * L;
    {
      const int nrb = (t + 31) / 32;
      const int nwarps = NT / 32;
      const int ncc = max(1, min(min(nwarps / nrb, 8), (t + 15) / 16));
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int task = warp; task < nrb * ncc; task += nwarps) {
        const int rb = task % nrb, cc = task / nrb;
        const int r = rb * 32 + lane;
        const int c0 = (int)((long)t * cc / ncc), c1 = (int)((long)t * (cc + 1) / ncc);
        double a2 = 0.0;
        if (r < t)
          for (int c = c0; c < c1; ++c) a2 += A22[r + (size_t)c * L] * sv[c];
        if (r < t) sp[t + cc * t + r] = a2;  // partials after sp[0..t)
      }
      __syncthreads();
      for (int r = threadIdx.x; r < t; r += NT) {
        double a2 = 0.0;
        for (int cc = 0; cc < ncc; ++cc) a2 += sp[t + cc * t + r];
        sp[r] = tj * a2;
      }
    }
    __syncthreads();
    acc = 0.0;
    for (int i = threadIdx.x; i < t; i += NT) acc += sp[i] * sv[i];
    double ptv = tri_block_sum<NT>(acc, red);
    const double K = 0.5 * tj * ptv;
    for (int i = threadIdx.x; i < t; i += NT) sp[i] -= K * sv[i];  // w = p - K v
    __syncthreads();
    // A22 -= v w^T + w v^T: lanes = rows, each warp walks a set of columns
    {
      const int nrb = (t + 31) / 32;
      const int nwarps = NT / 32;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int task = warp; task < nrb * t; task += nwarps) {
        const int rb = task % nrb, c = task / nrb;
        const int r = rb * 32 + lane;
        if (r < t) {
          double vr = sv[r], wr = sp[r];
          A22[r + (size_t)c * L] -= vr * sp[c] + wr * sv[c];
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (s >= 2) {
      d[s - 2] = M[(s - 2) + (size_t)(s - 2) * L];
      d[s - 1] = M[(s - 1) + (size_t)(s - 1) * L];
      e[s - 2] = M[(s - 1) + (size_t)(s - 2) * L];
    } else {
      d[0] = M[0];
    }
  }
}

// 1/x from the hardware approximation (rcp.approx.ftz.f64) plus two Newton steps: within an ulp
// or two of the IEEE quotient, several times cheaper than the division (latency-bound recurrences).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Sturm count: number of eigenvalues of T (d, e2 = e^2) strictly below x (GvL §8.4.1).
__device__ __forceinline__ int sturm_count(int s, const double* __restrict__ d, const double* __restrict__ e2,
                                           double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < s; ++i) {
    q = (d[i] - x) - e2[i - 1] * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// e2[i] = e[i]^2, bounds[0..1] = Gershgorin interval, bounds[2] = pivmin (one CTA)
__global__ void tri_prep_kernel(int s, const double* __restrict__ d, const double* __restrict__ e,
                                double* __restrict__ e2, double* __restrict__ bounds) {
  __shared__ double lo[32], hi[32], mx[32];
  double l = 1e300, h = -1e300, m = 0.0;
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < s ? fabs(e[i]) : 0.0);
    l = fmin(l, d[i] - r);
    h = fmax(h, d[i] + r);
    if (i + 1 < s) {
      double q = e[i] * e[i];
      e2[i] = q;
      m = fmax(m, q);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    l = fmin(l, __shfl_xor_sync(0xffffffffu, l, o));
    h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { lo[w] = l; hi[w] = h; mx[w] = m; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) { l = fmin(l, lo[i]); h = fmax(h, hi[i]); m = fmax(m, mx[i]); }
    l = fmin(l, lo[0]); h = fmax(h, hi[0]); m = fmax(m, mx[0]);
    double span = fmax(h - l, fmax(fabs(l), fabs(h)));
    double pad = 2.0 * PSD_U * span * s + 1e-300;
    bounds[0] = l - pad;
    bounds[1] = h + pad;
    bounds[2] = 2.2250738585072014e-308 * fmax(1.0, m) * 4.0;
  }
}

// One warp per wanted eigenvalue: ks-th largest, ks = blockIdx.x * warps + warp (ks < m),
// 32-way multisection. out[ks] = eigenvalue (descending). Warp id == m computes npos =
// #eigenvalues > 0 (s - count(0)).
__global__ void tri_bisect_kernel(int s, int m, const double* __restrict__ dg, const double* __restrict__ e2g,
                                  const double* __restrict__ bounds, double* __restrict__ out,
                                  int* __restrict__ npos) {
  extern __shared__ __align__(16) double bsm[];
  double* d = bsm;
  double* e2 = bsm + s;
  for (int k = threadIdx.x; k < s; k += blockDim.x) {
    d[k] = dg[k];
    if (k + 1 < s) e2[k] = e2g[k];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int ks = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (ks > m) return;
  const double pivmin = bounds[2];
  if (ks == m) {
    if (lane == 0) *npos = s - sturm_count(s, d, e2, 0.0, pivmin);
    return;
  }
  const int k = s - 1 - ks;  // ascending index: count(lo) <= k < count(hi)
  double lo = bounds[0], hi = bounds[1];
  // absolute accuracy u ||T|| suffices: the Rayleigh-Ritz values enter absolute residual tests, and
  // bisection to a relative tolerance near zero would add rounds for no gain (dstebz's ABSTOL)
  const double atol = 4.0 * PSD_U * fmax(fabs(lo), fabs(hi));
  for (int it = 0; it < 64; ++it) {
    double w = hi - lo;
    if (w <= fmax(2.0 * PSD_U * fmax(fabs(lo), fabs(hi)), atol) + 4.0 * pivmin) break;
    double x = lo + w * (double)(lane + 1) / 33.0;
    int c = sturm_count(s, d, e2, x, pivmin);
    unsigned below = __ballot_sync(0xffffffffu, c <= k);  // x still at or below the target
    // the first lane with count > k bounds the target from above
    int first_above = __ffs(~below) - 1;  // -1 if all lanes are below
    double nlo = lo, nhi = hi;
    if (first_above < 0) {
      nlo = lo + w * 32.0 / 33.0;
    } else {
      nhi = lo + w * (double)(first_above + 1) / 33.0;
      if (first_above > 0) nlo = lo + w * (double)first_above / 33.0;
    }
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) out[ks] = 0.5 * (lo + hi);
}

// Inverse iteration (GvL §8.4.2): one thread per eigenvector i < m (eigenvalue lam[i]):
// LU with partial pivoting of T - lam I (LAPACK dgttrf), `iters` solves (dgttrs), each
// normalised. y (s x m, ldy) holds the start vectors when `use_start`, else a fixed
// pseudo-random start. scratch: 5 s doubles per vector.
// Per-vector arrays live in shared memory when they fit (smem_ok), else in `scratch`.
__global__ void tri_inviter_kernel(int s, int m, const double* __restrict__ d, const double* __restrict__ e,
                                   const double* __restrict__ lam, const double* __restrict__ bounds,
                                   double* __restrict__ y, int ldy, double* __restrict__ scratch, int iters,
                                   int use_start, int smem_ok) {
  extern __shared__ __align__(16) double ism[];
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  // interleaved layout in smem: element k of thread t at [k * blockDim + t] (conflict-free)
  const int stride = smem_ok ? blockDim.x : 1;
  double* base = smem_ok ? ism + threadIdx.x : scratch + (size_t)i * 6 * s;
  double* dd = base;
  double* du = base + (size_t)s * stride;
  double* du2 = base + (size_t)2 * s * stride;
  double* dl = base + (size_t)3 * s * stride;
  double* pv = base + (size_t)4 * s * stride;  // pivots stored as doubles (0/1)
  double* yy = base + (size_t)5 * s * stride;  // working vector
  double* yi = y + (size_t)i * ldy;
#define DD(k) dd[(size_t)(k) * stride]
#define DU(k) du[(size_t)(k) * stride]
#define DU2(k) du2[(size_t)(k) * stride]
#define DL(k) dl[(size_t)(k) * stride]
#define PV(k) pv[(size_t)(k) * stride]
#define YY(k) yy[(size_t)(k) * stride]
  const double span = fmax(fabs(bounds[0]), fabs(bounds[1]));
  const double eps_piv = PSD_U * span + 1e-300;
  const double lm = lam[i];
  for (int k = 0; k < s; ++k) {
    DD(k) = d[k] - lm;
    if (k + 1 < s) { DU(k) = e[k]; DL(k) = e[k]; }
    DU2(k) = 0.0;
  }
  for (int k = 0; k + 1 < s; ++k) {  // dgttrf
    double dk = DD(k), lk = DL(k);
    if (fabs(dk) >= fabs(lk)) {
      if (dk == 0.0) dk = eps_piv;
      double fact = lk * fast_rcp(dk);
      DD(k) = dk;
      DL(k) = fact;
      DD(k + 1) -= fact * DU(k);
      DU2(k) = 0.0;
      PV(k) = 0.0;
    } else {
      double fact = dk * fast_rcp(lk);
      DD(k) = lk;
      DL(k) = fact;
      double tmp = DU(k);
      double dk1 = DD(k + 1);
      DU(k) = dk1;
      DD(k + 1) = tmp - fact * dk1;
      if (k + 2 < s) {
        double u1 = DU(k + 1);
        DU2(k) = u1;
        DU(k + 1) = -fact * u1;
      } else {
        DU2(k) = 0.0;
      }
      PV(k) = 1.0;
    }
  }
  for (int k = 0; k < s; ++k) {  // DD <- 1 / pivot (the solves multiply)
    double p = DD(k);
    if (fabs(p) < eps_piv) p = (p < 0.0) ? -eps_piv : eps_piv;
    DD(k) = fast_rcp(p);
  }
  if (!use_start) {
    uint32_t h = 0x9E3779B9u * (uint32_t)(i + 1) + 0x7F4A7C15u;
    for (int k = 0; k < s; ++k) {
      h ^= h << 13; h ^= h >> 17; h ^= h << 5;
      YY(k) = 0.5 + (double)(h & 0xffffff) / 16777216.0;
    }
  } else {
    for (int k = 0; k < s; ++k) YY(k) = yi[k];
  }
  // iterations without separate scaling passes: the previous iteration's 1/max scale is applied as
  // the forward sweep reads each entry, and the last backward sweep accumulates ||y||^2
  double sc = 1.0, n2 = 0.0;
  for (int it = 0; it < iters; ++it) {
    const bool last = it + 1 == iters;
    double y0 = YY(0) * sc;
    for (int k = 0; k + 1 < s; ++k) {  // dgttrs forward (L with interchanges)
      const double y1 = YY(k + 1) * sc;
      if (PV(k) == 0.0) {
        YY(k) = y0;
        y0 = y1 - DL(k) * y0;
      } else {
        YY(k) = y1;
        y0 = y0 - DL(k) * y1;
      }
    }
    YY(s - 1) = y0;
    double nrm = 0.0;
    double b1 = 0.0, b2 = 0.0;  // YY(k + 1), YY(k + 2) of the back substitution
    for (int k = s - 1; k >= 0; --k) {  // back substitution with U
      double v = YY(k);
      if (k + 1 < s) v -= DU(k) * b1;
      if (k + 2 < s) v -= DU2(k) * b2;
      v *= DD(k);
      YY(k) = v;
      b2 = b1;
      b1 = v;
      if (last)
        n2 = fma(v, v, n2);
      else
        nrm = fmax(nrm, fabs(v));
    }
    sc = (nrm > 0.0) ? 1.0 / nrm : 1.0;
  }
  double inv = (n2 > 0.0) ? rsqrt(n2) : 0.0;
  for (int k = 0; k < s; ++k) yi[k] = YY(k) * inv;
#undef DD
#undef DU
#undef DU2
#undef DL
#undef PV
#undef YY
}

// Modified Gram-Schmidt inside clusters (dstein: |lam_i - lam_{i-1}| <= 1e-3 ||T||), one CTA,
// vectors in descending eigenvalue order.
template <int NT>
__global__ void __launch_bounds__(NT) tri_cluster_mgs_kernel(int s, int m, const double* __restrict__ lam,
                                                             const double* __restrict__ bounds,
                                                             double* __restrict__ y, int ldy) {
  __shared__ double red[33];
  const double ortol = 1e-3 * fmax(fabs(bounds[0]), fabs(bounds[1]));
  int cstart = 0;
  for (int i = 0; i < m; ++i) {
    if (i == 0 || fabs(lam[i - 1] - lam[i]) > ortol) {
      cstart = i;
      continue;
    }
    double* yi = y + (size_t)i * ldy;
    for (int jv = cstart; jv < i; ++jv) {
      const double* yj = y + (size_t)jv * ldy;
      double acc = 0.0;
      for (int k = threadIdx.x; k < s; k += NT) acc += yi[k] * yj[k];
      double dot = tri_block_sum<NT>(acc, red);
      for (int k = threadIdx.x; k < s; k += NT) yi[k] -= dot * yj[k];
      __syncthreads();
    }
    double acc = 0.0;
    for (int k = threadIdx.x; k < s; k += NT) acc += yi[k] * yi[k];
    double nn = tri_block_sum<NT>(acc, red);
    double inv = (nn > 0.0) ? rsqrt(nn) : 0.0;
    for (int k = threadIdx.x; k < s; k += NT) yi[k] *= inv;
    __syncthreads();
  }
}

// Back-transformation Y <- Q Y, Q = H_0 H_1 ... H_{s-3}: apply H_{s-3} first. One warp per
// column, the column held in registers (s <= 32 * TRI_BT_PER_LANE), reflectors read through L1.
constexpr int TRI_BT_PER_LANE = 40;
__global__ void __launch_bounds__(256) tri_backtransform_kernel(int s, int m, const double* __restrict__ Vh, int ldv,
                                                                const double* __restrict__ tau,
                                                                double* __restrict__ y, int ldy) {
  const int lane = threadIdx.x & 31;
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (col >= m) return;
  double* yc = y + (size_t)col * ldy;
  double r[TRI_BT_PER_LANE];
#pragma unroll
  for (int q = 0; q < TRI_BT_PER_LANE; ++q) {
    int k = lane + 32 * q;
    r[q] = (k < s) ? yc[k] : 0.0;
  }
  for (int j = s - 3; j >= 0; --j) {
    const double tj = __ldg(tau + j);
    if (tj == 0.0) continue;
    const double* v = Vh + (size_t)j * ldv;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < TRI_BT_PER_LANE; ++q) {
      int k = lane + 32 * q;
      if (k > j && k < s) acc += __ldg(v + k) * r[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    acc *= tj;
#pragma unroll
    for (int q = 0; q < TRI_BT_PER_LANE; ++q) {
      int k = lane + 32 * q;
      if (k > j && k < s) r[q] -= acc * __ldg(v + k);
    }
  }
#pragma unroll
  for (int q = 0; q < TRI_BT_PER_LANE; ++q) {
    int k = lane + 32 * q;
    if (k < s) yc[k] = r[q];
  }
}

}  // namespace psd
