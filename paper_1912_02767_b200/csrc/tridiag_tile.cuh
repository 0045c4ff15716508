// tridiag_tile.cuh -- one-CTA Householder tridiagonalisation for the Rayleigh-Ritz matrices of the
// LOBPCG iteration (a7, s <= 256): the symmetric matrix lives in 32 x 32 tiles of its lower block
// triangle, one tile per warp in REGISTERS (the 16 longest-lived tiles) and the rest in shared memory,
// and every Householder step is ONE fused pass over the trailing tiles: the previous step's rank-2
// update A -= v w^T + w v^T is applied and the next matrix-vector product p = A v accumulated in the
// same read (GvL 4th ed. Alg. 8.3.1, the update deferred by one step as in LAPACK dsytd2's
// two-sided form). No thread-block cluster, no DSMEM hops: four CTA barriers per column.
//
// Tile layout (skewed): lane l of the owning warp holds, at slot q, the element
//     (row 32 I + l, column 32 K + ((l + q) mod 32))
// so that the 32 lanes of a step touch 32 distinct rows AND 32 distinct columns: the row sums of
// A v accumulate per lane and the column sums (the symmetric half, off-diagonal tiles) travel around
// the warp with one shuffle per step; shared-memory tiles are read conflict-free (slot-major).
// Diagonal tiles are stored full (both triangles) and contribute row sums only.
//
// Outputs exactly as tridiag_kernel (tridiag.cuh): d[s], e[s-1], tau[s-2], reflectors Vh (s x s,
// ldv) with column j = v_j, v_j[j+1] = 1, v_j[i] = 0 for i <= j; Q^T A Q = T with Q = H_0 ... H_{s-3}.
#pragma once
#include "common.cuh"

namespace psd {

constexpr int TT_NW = 16;                       // warps per CTA
constexpr int TT_NT = 32 * TT_NW;               // 512 threads
constexpr int TT_NBMAX = 8;                     // 8 x 32 = 256
constexpr int TT_SMAX = 32 * TT_NBMAX;
constexpr int TT_TMAX = TT_NBMAX * (TT_NBMAX + 1) / 2;  // 36 tiles

__host__ __device__ constexpr int tt_tiles(int nb) { return nb * (nb + 1) / 2; }
// dynamic shared memory (doubles): smem tiles, colbuf / v (s rounded to 32 each), the pending pair
// (vp, wp) interleaved, row and column partials (one 32-vector per tile each), scalars
__host__ __device__ inline size_t tri_tile_smem_doubles(int s) {
  const int nb = (s + 31) / 32, T = tt_tiles(nb);
  const int nsm = T > TT_NW ? T - TT_NW : 0;
  return (size_t)nsm * 1024 + 4 * (size_t)nb * 32 + 2 * (size_t)T * 32 + 64;
}

// (I, K) of the o-th tile in the assignment order: by block column K descending (a tile stays active
// while the Householder column index is below 32 K + 32), then I descending; tile o goes to warp
// o mod 16, the first 16 into registers.
__device__ __forceinline__ void tt_tile_of(int o, int nb, int& I, int& K) {
  int c = 0;
  for (int k = nb - 1; k >= 0; --k)
    for (int i = nb - 1; i >= k; --i) {
      if (c == o) {
        I = i;
        K = k;
        return;
      }
      ++c;
    }
  I = K = -1;
}

__device__ __forceinline__ int tt_cid(int I, int K) { return I * (I + 1) / 2 + K; }  // canonical tile id

// element q of a tile held in registers, q known only at run time
__device__ __forceinline__ double tt_reg_get(const double (&rt)[32], int q) {
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k == q) a = rt[k];
  return a;
}

// One fused pass over a tile: pending update A -= vp wp^T + wp vp^T, then row (and, off the diagonal,
// column) partial sums of A v. vb: the current Householder vector; vw: interleaved (vp, wp).
template <bool REG, bool OFF>
__device__ __forceinline__ void tt_pass(double (&rt)[32], double* __restrict__ st, int I, int K, int lane,
                                        const double* __restrict__ vb, const double2* __restrict__ vw,
                                        double& yrow, double& ycol) {
  const int r = 32 * I + lane;
  const double vr = vb[r];
  const double2 pr = vw[r];
  const double* vbc = vb + 32 * K;
  const double2* vwc = vw + 32 * K;
  // column sums: NA interleaved accumulators; acc[X] serves the steps q = NA t + X and, on lane l at
  // round t, holds the partial sum of local column (l + NA t + X) mod 32 (shifted NA lanes per round)
  constexpr int NA = 4;
  double yr0 = 0.0, yr1 = 0.0, acc[NA];
#pragma unroll
  for (int x = 0; x < NA; ++x) acc[x] = 0.0;
#pragma unroll
  for (int t = 0; t < 32 / NA; ++t) {
#pragma unroll
    for (int x = 0; x < NA; ++x) {
      const int q = NA * t + x;
      const int cl = (lane + q) & 31;
      const double vc = vbc[cl];
      const double2 pc = vwc[cl];
      double a = REG ? rt[q] : st[q * 32 + lane];
      a = fma(-pr.x, pc.y, a);
      a = fma(-pr.y, pc.x, a);
      if (REG)
        rt[q] = a;
      else
        st[q * 32 + lane] = a;
      if (x & 1)
        yr1 = fma(a, vc, yr1);
      else
        yr0 = fma(a, vc, yr0);
      if (OFF) acc[x] = fma(a, vr, acc[x]);
    }
    if (OFF) {
#pragma unroll
      for (int x = 0; x < NA; ++x) acc[x] = __shfl_sync(0xffffffffu, acc[x], (lane + NA) & 31);
    }
  }
  double yc = 0.0;
  if (OFF) {
    // after the last round acc[x] on lane l is the sum of local column (l + x) mod 32: gather column l
    yc = acc[0];
#pragma unroll
    for (int x = 1; x < NA; ++x) yc += __shfl_sync(0xffffffffu, acc[x], (lane - x) & 31);
  }
  yrow = yr0 + yr1;
  ycol = yc;
}

__global__ void __launch_bounds__(TT_NT, 1) tridiag_tile_kernel(int s, const double* __restrict__ A, int lda,
                                                                double* __restrict__ d, double* __restrict__ e,
                                                                double* __restrict__ tau, double* __restrict__ Vh,
                                                                int ldv) {
  extern __shared__ __align__(16) double sm[];
  const int nb = (s + 31) / 32, T = tt_tiles(nb), S32 = nb * 32;
  const int nsm = T > TT_NW ? T - TT_NW : 0;
  double* stiles = sm;
  double2* vw = reinterpret_cast<double2*>(stiles + (size_t)nsm * 1024);  // (vp, wp) pending pair
  double* colbuf = reinterpret_cast<double*>(vw + S32);
  double* vb = colbuf + S32;     // current Householder vector (0 above j + 1)
  double* prow = vb + S32;       // [T][32] row partials by canonical tile id
  double* pcol = prow + T * 32;  // [T][32] column partials
  double* red = pcol + T * 32;   // 64: warp partials, scalars
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // this warp's tiles: o = warp (register tile), warp + 16, warp + 32 (shared memory)
  int tI[3] = {-1, -1, -1}, tK[3] = {-1, -1, -1};
  int ntile = 0;
  for (int o = warp, k = 0; o < T && k < 3; o += TT_NW, ++k) {
    tt_tile_of(o, nb, tI[k], tK[k]);
    ntile = k + 1;
  }
  double rt[32];
  // load (symmetrised: 0.5 (A + A^T), zero padding beyond s)
  for (int k = 0; k < ntile; ++k) {
    const int r = 32 * tI[k] + lane;
    double* st = k == 0 ? nullptr : stiles + (size_t)(warp + (k - 1) * TT_NW) * 1024;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int c = 32 * tK[k] + ((lane + q) & 31);
      const double a = (r < s && c < s) ? 0.5 * (A[IDX(r, c, lda)] + A[IDX(c, r, lda)]) : 0.0;
      if (k == 0)
        rt[q] = a;
      else
        st[q * 32 + lane] = a;
    }
  }
  for (int i = threadIdx.x; i < S32; i += TT_NT) {
    vw[i] = make_double2(0.0, 0.0);
    colbuf[i] = 0.0;  // the padding rows [s, 32 nb) are never written by a column extraction
    vb[i] = 0.0;
  }
  // reflector columns s-2, s-1 (and all columns when s <= 2) are zero
  for (int jj = max(s - 2, 0); jj < s; ++jj)
    for (int i = threadIdx.x; i < s; i += TT_NT) Vh[IDX(i, jj, ldv)] = 0.0;
  __syncthreads();

  for (int j = 0; j + 2 < s; ++j) {
    const int jb = j >> 5, j1 = j + 1, kb0 = j1 >> 5;
    // (1) column j with the pending update applied (rows >= j) -> colbuf
    {
      const double2 pj = vw[j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (k >= ntile || tK[k] != jb) continue;
        const int r = 32 * tI[k] + lane;
        const int q = (j - 32 * jb - lane) & 31;
        const double a = k == 0 ? tt_reg_get(rt, q) : stiles[(size_t)(warp + (k - 1) * TT_NW) * 1024 + q * 32 + lane];
        const double2 pr = vw[r];
        if (r >= j && r < s) colbuf[r] = a - (pr.x * pj.y + pr.y * pj.x);
      }
    }
    __syncthreads();
    // (2) warp 0: Householder vector of column j -> vb, scalars -> red[32..33], outputs d, e, tau, Vh
    if (warp == 0) {
      double sig = 0.0;
      for (int i = j + 2 + lane; i < s; i += 32) sig = fma(colbuf[i], colbuf[i], sig);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sig += __shfl_xor_sync(0xffffffffu, sig, o);
      const double alpha = colbuf[j1];
      double tj, beta, scale;
      if (sig == 0.0) {
        tj = 0.0;
        beta = alpha;
        scale = 0.0;
      } else {
        const double mu = sqrt(fma(alpha, alpha, sig));
        beta = (alpha <= 0.0) ? mu : -mu;
        tj = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int i = lane; i < S32; i += 32) {
        const double v = i > j1 ? colbuf[i] * scale : (i == j1 ? 1.0 : 0.0);
        vb[i] = v;
        if (i < s) Vh[IDX(i, j, ldv)] = v;
      }
      if (lane == 0) {
        d[j] = colbuf[j];
        e[j] = beta;
        tau[j] = tj;
        red[32] = tj;
      }
    }
    __syncthreads();
    const double tj = red[32];
    // (3) fused pass: pending update + partial sums of A v over the active tiles (block column >= kb0)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k >= ntile || tK[k] < kb0) continue;
      double* st = k == 0 ? nullptr : stiles + (size_t)(warp + (k - 1) * TT_NW) * 1024;
      double yr, yc = 0.0;
      if (tI[k] != tK[k]) {
        if (k == 0)
          tt_pass<true, true>(rt, st, tI[k], tK[k], lane, vb, vw, yr, yc);
        else
          tt_pass<false, true>(rt, st, tI[k], tK[k], lane, vb, vw, yr, yc);
      } else {
        if (k == 0)
          tt_pass<true, false>(rt, st, tI[k], tK[k], lane, vb, vw, yr, yc);
        else
          tt_pass<false, false>(rt, st, tI[k], tK[k], lane, vb, vw, yr, yc);
      }
      const int cid = tt_cid(tI[k], tK[k]);
      prow[cid * 32 + lane] = yr;
      pcol[cid * 32 + lane] = yc;
    }
    __syncthreads();
    // (4) p = tau A v, w = p - (tau/2)(p^T v) v: the next pending update
    double pi = 0.0, vi = 0.0;
    const int i = threadIdx.x;
    if (i >= j1 && i < s) {
      const int bi = i >> 5, li = i & 31;
      double y = 0.0;
      for (int K = kb0; K <= bi; ++K) y += prow[tt_cid(bi, K) * 32 + li];
      for (int I = bi + 1; I < nb; ++I) y += pcol[tt_cid(I, bi) * 32 + li];
      pi = tj * y;
      vi = vb[i];
    }
    double dp = pi * vi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
    if (lane == 0) red[warp] = dp;
    __syncthreads();
    double ptv = 0.0;
#pragma unroll
    for (int w = 0; w < TT_NW; ++w) ptv += red[w];
    const double Kc = 0.5 * tj * ptv;
    if (i < S32) vw[i] = make_double2(vi, fma(-Kc, vi, pi));
    __syncthreads();
  }
  // trailing 2 x 2 block (or the whole matrix when s <= 2), with the last pending update
  if (threadIdx.x == 0) red[32] = red[33] = red[34] = 0.0;
  __syncthreads();
  for (int k = 0; k < ntile; ++k) {
    const int r = 32 * tI[k] + lane;
    for (int cc = max(s - 2, 0); cc < s; ++cc) {
      if (cc < 32 * tK[k] || cc >= 32 * tK[k] + 32 || r < cc || r >= s) continue;
      const int q = (cc - 32 * tK[k] - lane) & 31;
      const double a = k == 0 ? tt_reg_get(rt, q) : stiles[(size_t)(warp + (k - 1) * TT_NW) * 1024 + q * 32 + lane];
      const double2 pr = vw[r], pc = vw[cc];
      const double u = a - (pr.x * pc.y + pr.y * pc.x);
      // slots: 32 = (s-2, s-2) or (0, 0), 33 = (s-1, s-2), 34 = (s-1, s-1)
      const int slot = (r == cc) ? (r == s - 1 && s >= 2 ? 34 : 32) : 33;
      red[slot] = u;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s >= 2) {
      d[s - 2] = red[32];
      d[s - 1] = red[34];
      e[s - 2] = red[33];
    } else {
      d[0] = red[32];
    }
  }
}

}  // namespace psd
