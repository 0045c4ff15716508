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

// Sturm count by the leading principal minors of T - x I (three-term recurrence
// P_i = (d_i - x) P_{i-1} - e_{i-1}^2 P_{i-2}, GvL §8.4.1): the number of eigenvalues below x is the
// number of sign changes in P_0 = 1, P_1, ..., P_s. Unlike the ratio form q_i = P_i / P_{i-1} it has
// no division on the dependency chain (one FMA per step: e^2 P_{i-2} is formed a step early).
// T is pre-scaled by a power of two to O(1) entries and the pair (P_i, P_{i-1}) is rescaled by a
// power of two every 8 steps (exact), so the minors neither overflow nor underflow. An exact zero
// minor is replaced by -2^-60 P_{i-1} (the ratio form's q_i = -pivmin).
__device__ __forceinline__ int sturm_count_det(int s, const double* __restrict__ d, const double* __restrict__ e2,
                                               double x) {
  double pm = 1.0, p = d[0] - x;
  if (p == 0.0) p = -0x1p-60;
  int cnt = p < 0.0;
  for (int i = 1; i < s; ++i) {
    const double t = e2[i - 1] * pm;  // off the chain
    double pn = fma(d[i] - x, p, -t);
    if (pn == 0.0) pn = -0x1p-60 * p;
    cnt += (pn < 0.0) != (p < 0.0);
    pm = p;
    p = pn;
    if ((i & 7) == 0) {
      const double mx = fmax(fabs(p), fabs(pm));
      const int ex = (int)((__double_as_longlong(mx) >> 52) & 0x7ff);
      if (ex > 0 && ex < 2047) {
        const double sc = __longlong_as_double((long long)(2046 - ex) << 52);  // 2^(1023 - (ex - 1023))
        p *= sc;
        pm *= sc;
      }
    }
  }
  return cnt;
}

// Multisection bisection (dstebz-like). One warp per wanted eigenvalue: ks-th largest,
// ks = blockIdx.x * warps + warp (ks < m), 32-way multisection. out[ks] = eigenvalue (descending).
// Warp id == m computes npos = #eigenvalues > 0 (s - count(0)).
__global__ void tri_bisect_kernel(int s, int m, const double* __restrict__ dg, const double* __restrict__ e2g,
                                  const double* __restrict__ bounds, double* __restrict__ out,
                                  int* __restrict__ npos) {
  extern __shared__ __align__(16) double bsm[];
  double* d = bsm;
  double* e2 = bsm + s;
  // power-of-two scale to O(1): 1 / 2^ceil(log2 max(|lo|, |hi|))
  const double span = fmax(fmax(fabs(bounds[0]), fabs(bounds[1])), 1e-300);
  const int sex = (int)((__double_as_longlong(span) >> 52) & 0x7ff) - 1022;  // span < 2^sex
  const double inv = ldexp(1.0, -sex);  // <= 2^997: inv^2 would overflow for tiny spans
  for (int k = threadIdx.x; k < s; k += blockDim.x) {
    d[k] = dg[k] * inv;
    if (k + 1 < s) e2[k] = (e2g[k] * inv) * inv;  // e^2 <= span^2: no intermediate overflow
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int ks = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (ks > m) return;
  if (ks == m) {
    if (lane == 0) *npos = s - sturm_count_det(s, d, e2, 0.0);
    return;
  }
  const int k = s - 1 - ks;  // ascending index: count(lo) <= k < count(hi)
  double lo = bounds[0], hi = bounds[1];
  const double pivmin = bounds[2];
  // absolute accuracy u ||T|| suffices: the Rayleigh-Ritz values enter absolute residual tests, and
  // bisection to a relative tolerance near zero would add rounds for no gain (dstebz's ABSTOL)
  const double atol = 4.0 * PSD_U * fmax(fabs(lo), fabs(hi));
  for (int it = 0; it < 64; ++it) {
    double w = hi - lo;
    if (w <= fmax(2.0 * PSD_U * fmax(fabs(lo), fabs(hi)), atol) + 4.0 * pivmin) break;
    double x = lo + w * (double)(lane + 1) / 33.0;
    int c = sturm_count_det(s, d, e2, x * inv);
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
  // a final bracket around 0 cannot tell the sign: report the eigenvalue as 0 (non-positive, as the
  // Sturm count at 0 does)
  if (lane == 0) out[ks] = (lo <= 0.0 && hi >= 0.0) ? 0.0 : 0.5 * (lo + hi);
}

// Multisection with G = blockDim.x (a multiple of 32, <= 1024) points per round: one CTA per wanted
// eigenvalue (ks = blockIdx.x < m, ks-th largest), the CTA's G threads evaluate the Sturm count at
// the G interior points of a (G + 1)-section of [lo, hi]; block m computes npos. Each round narrows
// the bracket by G + 1 (log2(G + 1) bits) for one Sturm chain of latency: a 128-point round gains 7
// bits where one warp gains 5, and the threads are free (m is ~100 CTAs on 148 SMs).
// The per-warp "count <= k" ballots go through shared memory (double-buffered by round parity: one
// barrier per round); every thread derives the same new bracket.
__global__ void tri_bisect_ms_kernel(int s, int m, const double* __restrict__ dg, const double* __restrict__ e2g,
                                     const double* __restrict__ bounds, double* __restrict__ out,
                                     int* __restrict__ npos) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  extern __shared__ __align__(16) double bsm[];
  __shared__ unsigned masks[2][32];
  double* d = bsm;
  double* e2 = bsm + s;
  const double span = fmax(fmax(fabs(bounds[0]), fabs(bounds[1])), 1e-300);
  const int sex = (int)((__double_as_longlong(span) >> 52) & 0x7ff) - 1022;  // span < 2^sex
  const double inv = ldexp(1.0, -sex);
  for (int k = threadIdx.x; k < s; k += blockDim.x) {
    d[k] = dg[k] * inv;
    if (k + 1 < s) e2[k] = (e2g[k] * inv) * inv;
  }
  __syncthreads();
  const int ks = blockIdx.x;
  if (ks >= m) {
    if (threadIdx.x == 0) *npos = s - sturm_count_det(s, d, e2, 0.0);
    return;
  }
  const int G = blockDim.x, nw = G >> 5, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int k = s - 1 - ks;  // ascending index: count(lo) <= k < count(hi)
  double lo = bounds[0], hi = bounds[1];
  const double pivmin = bounds[2];
  const double atol = 4.0 * PSD_U * fmax(fabs(lo), fabs(hi));
  const double rg = 1.0 / (double)(G + 1);
  for (int it = 0; it < 64; ++it) {
    const double w = hi - lo;
    if (w <= fmax(2.0 * PSD_U * fmax(fabs(lo), fabs(hi)), atol) + 4.0 * pivmin) break;
    const double x = lo + w * (double)(t + 1) * rg;
    const int c = sturm_count_det(s, d, e2, x * inv);
    const unsigned below = __ballot_sync(0xffffffffu, c <= k);
    if (lane == 0) masks[it & 1][warp] = below;
    __syncthreads();
    // first point (in order) with count > k bounds the target from above
    int first_above = -1;
    for (int q = 0; q < nw; ++q) {
      const unsigned b = masks[it & 1][q];
      if (b != 0xffffffffu) {
        first_above = q * 32 + __ffs(~b) - 1;
        break;
      }
    }
    double nlo = lo, nhi = hi;
    if (first_above < 0) {
      nlo = lo + w * (double)G * rg;
    } else {
      nhi = lo + w * (double)(first_above + 1) * rg;
      if (first_above > 0) nlo = lo + w * (double)first_above * rg;
    }
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  if (t == 0) out[ks] = (lo <= 0.0 && hi >= 0.0) ? 0.0 : 0.5 * (lo + hi);  // as tri_bisect_kernel
}

// Inverse iteration (GvL §8.4.2): one thread per eigenvector i < m (eigenvalue lam[i]):
// LU with partial pivoting of T - lam I (LAPACK dgttrf), `iters` solves (dgttrs), each
// normalised. y (s x m, ldy) holds the start vectors when `use_start`, else a fixed
// pseudo-random start. The recurrences are sequential in k, so the kernel is latency-bound per
// vector: d, e are staged once per CTA in shared memory (broadcast reads), the factorisation
// carries the running pivot and super-diagonal in registers (one reciprocal per step on the
// dependency chain), the random start is drawn inside the factorisation sweep, and the stored
// pivots are reciprocals (the solves multiply).
// Shared memory: 2 s doubles (d, e) + per thread 5 s doubles (1/pivot, L, U, U2, y) + s bytes
// (interchanges), interleaved [k * blockDim + t] (conflict-free). smem_ok = 0: the per-thread
// arrays live in `scratch` (5 s doubles + s bytes per vector) instead.
__host__ __device__ inline size_t tri_inviter_smem_bytes(int s, int vpb) {
  return (size_t)2 * s * sizeof(double) + (size_t)vpb * s * (5 * sizeof(double) + 1);
}
__global__ void tri_inviter_kernel(int s, int m, const double* __restrict__ d, const double* __restrict__ e,
                                   const double* __restrict__ lam, const double* __restrict__ bounds,
                                   double* __restrict__ y, int ldy, double* __restrict__ scratch, int iters,
                                   int use_start, int smem_ok) {
  extern __shared__ __align__(16) double ism[];
  double* sd = ism;
  double* se = ism + s;
  for (int k = threadIdx.x; k < s; k += blockDim.x) {
    sd[k] = d[k];
    se[k] = (k + 1 < s) ? e[k] : 0.0;
  }
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int stride = smem_ok ? blockDim.x : 1;
  double* base = smem_ok ? ism + 2 * (size_t)s + threadIdx.x : scratch + (size_t)i * 6 * s;
  double* rd = base;                           // 1 / pivot
  double* dl = base + (size_t)s * stride;      // L multipliers
  double* du = base + (size_t)2 * s * stride;  // U super-diagonal
  double* du2 = base + (size_t)3 * s * stride; // U second super-diagonal (interchanges)
  double* yy = base + (size_t)4 * s * stride;  // working vector
  unsigned char* pv = smem_ok ? reinterpret_cast<unsigned char*>(ism + 2 * (size_t)s + (size_t)5 * s * blockDim.x) + threadIdx.x
                              : reinterpret_cast<unsigned char*>(scratch + (size_t)i * 6 * s + (size_t)5 * s);
#define RD(k) rd[(size_t)(k) * stride]
#define DL(k) dl[(size_t)(k) * stride]
#define DU(k) du[(size_t)(k) * stride]
#define DU2(k) du2[(size_t)(k) * stride]
#define YY(k) yy[(size_t)(k) * stride]
#define PV(k) pv[(size_t)(k) * stride]
  double* yi = y + (size_t)i * ldy;
  const double span = fmax(fabs(bounds[0]), fabs(bounds[1]));
  const double eps_piv = PSD_U * span + 1e-300;
  const double lm = lam[i];
  auto guarded_rcp = [&](double p, double r) {  // 1 / max(|p|, eps) with the sign of p (r = 1/p)
    return (fabs(p) < eps_piv) ? ((p < 0.0) ? -1.0 / eps_piv : 1.0 / eps_piv) : r;
  };
  // dgttrf with the running pivot dk and super-diagonal uk in registers
  uint32_t h = 0x9E3779B9u * (uint32_t)(i + 1) + 0x7F4A7C15u;
  double dk = sd[0] - lm, uk = se[0];
  for (int k = 0; k + 1 < s; ++k) {
    const double lk = se[k], d1 = sd[k + 1] - lm, e1 = se[k + 1];  // se[s-1] = 0
    if (fabs(dk) >= fabs(lk)) {
      if (dk == 0.0) dk = eps_piv;
      const double r = fast_rcp(dk);
      const double f = lk * r;
      RD(k) = guarded_rcp(dk, r);
      DL(k) = f;
      DU(k) = uk;
      DU2(k) = 0.0;
      PV(k) = 0;
      dk = fma(-f, uk, d1);
      uk = e1;
    } else {
      const double r = fast_rcp(lk);
      const double f = dk * r;
      RD(k) = guarded_rcp(lk, r);
      DL(k) = f;
      DU(k) = d1;
      DU2(k) = e1;
      PV(k) = 1;
      dk = fma(-f, d1, uk);
      uk = -f * e1;
    }
    if (!use_start) {
      h ^= h << 13; h ^= h >> 17; h ^= h << 5;
      YY(k) = 0.5 + (double)(h & 0xffffff) / 16777216.0;
    }
  }
  RD(s - 1) = guarded_rcp(dk, fast_rcp(dk == 0.0 ? eps_piv : dk));
  if (!use_start) {
    h ^= h << 13; h ^= h >> 17; h ^= h << 5;
    YY(s - 1) = 0.5 + (double)(h & 0xffffff) / 16777216.0;
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
      const double lk = DL(k);
      if (PV(k) == 0) {
        YY(k) = y0;
        y0 = fma(-lk, y0, y1);
      } else {
        YY(k) = y1;
        y0 = fma(-lk, y1, y0);
      }
    }
    YY(s - 1) = y0;
    double nrm = 0.0;
    double b1 = 0.0, b2 = 0.0;  // YY(k + 1), YY(k + 2) of the back substitution
    for (int k = s - 1; k >= 0; --k) {  // back substitution with U
      double v = YY(k);
      if (k + 1 < s) v = fma(-DU(k), b1, v);
      if (k + 2 < s) v = fma(-DU2(k), b2, v);
      v *= RD(k);
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
#undef RD
#undef DU
#undef DU2
#undef DL
#undef PV
#undef YY
}

// Eigenvectors by the twisted factorisation (Parlett & Dhillon; LAPACK dlar1v), one warp per
// eigenvalue: T - lam I = L D+ L^T (top-down pivots D+) = U D- U^T (bottom-up pivots D-), twist
// index r = argmin |gamma_k|, gamma_k = D+_k + D-_k - (d_k - lam), and z_r = 1,
// z_i = -(e_i / D+_i) z_{i+1} (i < r), z_{i+1} = -(e_i / D-_{i+1}) z_i (i >= r), normalised.
// The pivots are ratios of leading / trailing principal minors, P_i = (d_i - lam) P_{i-1} -
// e_{i-1}^2 P_{i-2}: one FMA per step on the dependency chain (the division D_i = P_i / P_{i-1}
// is off it), the pair (P_i, P_{i-1}) rescaled by a power of two every 8 steps; an exact zero
// minor becomes -2^-60 P_{i-1} (dlar1v's zero-pivot replacement). Lane 0 runs the top chain,
// lane 1 the bottom chain, in lockstep; the two z products likewise.
// Shared memory per CTA (one warp): d, e, e^2 (staged), D+, l = e/D+, D-, u = e/D- (7 s + 2 doubles).
__global__ void __launch_bounds__(32) tri_twisted_kernel(int s, int m, const double* __restrict__ d,
                                                         const double* __restrict__ e,
                                                         const double* __restrict__ lam, double* __restrict__ y,
                                                         int ldy) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  extern __shared__ __align__(16) double tsm[];
  // ec[k] = e_{k-1} (coupling of rows k-1, k; ec[0] = ec[s] = 0), e2[k] = ec[k]^2
  double* sd = tsm;
  double* ec = tsm + s;                   // s + 1
  double* e2 = tsm + 2 * (size_t)s + 1;   // s + 1
  double* Dp = tsm + 3 * (size_t)s + 2;
  double* Lp = tsm + 4 * (size_t)s + 2;
  double* Dm = tsm + 5 * (size_t)s + 2;
  double* Um = tsm + 6 * (size_t)s + 2;
  const int lane = threadIdx.x, iv = blockIdx.x;
  if (iv >= m) return;
  for (int k = lane; k <= s; k += 32) {
    if (k < s) sd[k] = d[k];
    const double c = (k > 0 && k < s) ? e[k - 1] : 0.0;
    ec[k] = c;
    e2[k] = c * c;
  }
  __syncwarp();
  const double lm = lam[iv];
  if (lane < 2) {
    // lane 0: rows 0, 1, ..., s-1 (previous coupling ec[i], next ec[i+1]);
    // lane 1: rows s-1, ..., 0 (previous coupling ec[i+1], next ec[i])
    const bool top = lane == 0;
    const int dir = top ? 1 : -1, op = top ? 0 : 1, on = top ? 1 : 0;
    double* D = top ? Dp : Dm;
    double* M = top ? Lp : Um;
    double pm = 0.0, p = 1.0, rp = 1.0;  // P_{i-2}, P_{i-1}, 1 / P_{i-1}
    int i = top ? 0 : s - 1;
    auto step = [&]() {
      const double a = sd[i] - lm;
      double pn = fma(a, p, -e2[i + op] * pm);
      if (pn == 0.0) pn = -0x1p-60 * p;
      const double rn = fast_rcp(pn);  // off the P chain
      D[i] = pn * rp;                  // D_i = P_i / P_{i-1}
      M[i] = ec[i + on] * p * rn;      // e / D_i
      pm = p;
      p = pn;
      rp = rn;
      i += dir;
    };
    int st = 0;
    for (; st + 8 <= s; st += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) step();
      const double mx = fmax(fabs(p), fabs(pm));
      const int ex = (int)((__double_as_longlong(mx) >> 52) & 0x7ff);
      if (ex > 0 && ex < 2047) {
        const double sc = __longlong_as_double((long long)(2046 - ex) << 52);
        const double isc = __longlong_as_double((long long)(ex) << 52);  // 1 / sc
        p *= sc;
        pm *= sc;
        rp *= isc;
      }
    }
    for (; st < s; ++st) step();
  }
  __syncwarp();
  // twist index: argmin |gamma_k| (ties: the smallest k)
  double best = INFINITY;
  int bk = 0;
  for (int k = lane; k < s; k += 32) {
    const double g = fabs(Dp[k] + Dm[k] - (sd[k] - lm));
    if (g < best) {
      best = g;
      bk = k;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int okk = __shfl_xor_sync(0xffffffffu, bk, o);
    if (ob < best || (ob == best && okk < bk)) {
      best = ob;
      bk = okk;
    }
  }
  const int r = bk;
  // z (unnormalised) into Dp (free now): lane 0 upwards from r, lane 1 downwards
  double* z = Dp;
  if (lane == 0) {
    double zz = 1.0;
    z[r] = 1.0;
    for (int k = r - 1; k >= 0; --k) {
      zz = -Lp[k] * zz;
      z[k] = zz;
    }
  } else if (lane == 1) {
    double zz = 1.0;
    for (int k = r + 1; k < s; ++k) {
      zz = -Um[k] * zz;
      z[k] = zz;
    }
  }
  __syncwarp();
  double n2 = 0.0;
  for (int k = lane; k < s; k += 32) n2 = fma(z[k], z[k], n2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
  const double inv = (n2 > 0.0) ? rsqrt(n2) : 0.0;
  double* yv = y + (size_t)iv * ldy;
  for (int k = lane; k < s; k += 32) yv[k] = z[k] * inv;
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
