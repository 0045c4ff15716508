// tridiag_warp.cuh -- one-CTA Householder tridiagonalisation for the small Rayleigh-Ritz matrices of
// the converging LOBPCG iterations (a7, s <= 128; GvL 4th ed. Alg. 8.3.1 with the update deferred by
// one step as in LAPACK dsytd2's two-sided form: A <- A - v w^T - w v^T, p = tau A v,
// w = p - (tau / 2)(p^T v) v).
//
// Layout: the whole symmetric matrix (both triangles) in REGISTERS of one 512-thread CTA. Column c is
// owned by warp c mod 16 (local index c / 16), and lane l of that warp holds rows l + 32 i (i < R):
// a[i][cc] = A(l + 32 i, warp + 16 cc). Per Householder column j there are exactly TWO CTA barriers
// and no thread-block cluster / DSMEM hop:
//   A  every warp applies the pending update of step j - 1 to its own columns; the owner of column j
//      does that column first and then its Householder step (one warp reduction, sqrt, division),
//      writes v_j and tau_j to shared memory (and the reflector store / d, e, tau outputs), then
//      updates its other columns
//   -- barrier 1 --
//   B  every warp: p_c = tau_j sum_r a[r][c] v_j[r] for its own columns c > j (an in-register
//      column dot + a transpose reduction over the lanes), p_c to shared memory, its part of p^T v
//   -- barrier 2 --
// and the next step's K = tau_j / 2 sum(parts) is formed redundantly by every warp in fixed order
// (deterministic, identical in every thread). v / p / parts are double-buffered by the step parity.
// Outputs exactly as tridiag_kernel (tridiag.cuh): d[s], e[s-1], tau[s-2], reflectors Vh (s x s,
// ldv) with column j = v_j, v_j[j+1] = 1, v_j[i] = 0 for i <= j; Q^T A Q = T, Q = H_0 ... H_{s-3}.
#pragma once
#include "common.cuh"

namespace psd {

constexpr int TW_NW = 16;           // warps per CTA
constexpr int TW_NT = 32 * TW_NW;   // 512 threads

template <int R, int C>
__global__ void __launch_bounds__(TW_NT, 1) tridiag_warp_kernel(int s, const double* __restrict__ A, int lda,
                                                                double* __restrict__ d, double* __restrict__ e,
                                                                double* __restrict__ tau, double* __restrict__ Vh,
                                                                int ldv) {
  static_assert(C == 1 || C == 2 || C == 4 || C == 8, "columns per warp: a power of two <= 8");
  static_assert(TW_NW * C <= 32 * R, "every column index is a row of the shared vectors");
  constexpr int NR = 32 * R;  // padded row count
  __shared__ double vb[2][NR];
  __shared__ double pb[2][NR];
  __shared__ double part[2][TW_NW];
  __shared__ double tb[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  double a[R][C];
#pragma unroll
  for (int cc = 0; cc < C; ++cc) {
    const int c = warp + TW_NW * cc;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      a[i][cc] = (r < s && c < s) ? 0.5 * (A[IDX(r, c, lda)] + A[IDX(c, r, lda)]) : 0.0;
    }
  }
  for (int q = threadIdx.x; q < 2 * NR; q += TW_NT) {
    (&vb[0][0])[q] = 0.0;
    (&pb[0][0])[q] = 0.0;
  }
  if (threadIdx.x < 2 * TW_NW) (&part[0][0])[threadIdx.x] = 0.0;
  if (threadIdx.x < 2) tb[threadIdx.x] = 0.0;
  // reflector columns s-2, s-1 (and all columns when s <= 2) are zero
  for (int jj = max(s - 2, 0); jj < s; ++jj)
    for (int i = threadIdx.x; i < s; i += TW_NT) Vh[IDX(i, jj, ldv)] = 0.0;
  __syncthreads();

  // the pending update of the step whose buffers are `pp` (v, p), K = tau/2 p^T v of that step, applied
  // to local column `only` (only < 0: every own column except `skip`)
  // (v and w vanish above row j: on finished columns the update is a no-op; measured cheaper than
  // warp-uniform branches around them)
  auto pending = [&](int pp, double K, int only, int skip, int j) {
    double vr[R], wr[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double v = vb[pp][lane + 32 * i];
      vr[i] = v;
      wr[i] = fma(-K, v, pb[pp][lane + 32 * i]);
    }
#pragma unroll
    for (int cc = 0; cc < C; ++cc) {
      if ((only >= 0 && cc != only) || cc == skip) continue;
      const int c = warp + TW_NW * cc;
      const double vc = vb[pp][c], wc = fma(-K, vc, pb[pp][c]);
#pragma unroll
      for (int i = 0; i < R; ++i) a[i][cc] = fma(-vr[i], wc, fma(-wr[i], vc, a[i][cc]));
    }
  };
  // K = tau/2 p^T v of the step with buffers pp (the 16 warp parts in fixed order, in every thread)
  auto kprev = [&](int pp) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < TW_NW; ++w) sum += part[pp][w];
    return 0.5 * tb[pp] * sum;
  };

  for (int j = 0; j + 2 < s; ++j) {
    const int par = j & 1, pp = par ^ 1;
    const double K = kprev(pp);  // step j - 1 (zero buffers at j = 0)
    const int o = j % TW_NW, jc = j / TW_NW;
    if (warp == o) {
      pending(pp, K, jc, -1, j);  // column j first: it is on the critical path
      // Householder step of column j (rows j+1 ..): sigma = ||a[j+2:, j]||^2, alpha = a[j+1, j]
      double sg = 0.0, xa = 0.0, xd = 0.0;
#pragma unroll
      for (int cc = 0; cc < C; ++cc) {
        if (cc != jc) continue;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int r = lane + 32 * i;
          const double x = a[i][cc];
          if (r >= j + 2) sg = fma(x, x, sg);
          if (r == j + 1) xa = x;
          if (r == j) xd = x;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        sg += __shfl_xor_sync(0xffffffffu, sg, off);
        xa += __shfl_xor_sync(0xffffffffu, xa, off);  // one lane holds it, the others add zero
        xd += __shfl_xor_sync(0xffffffffu, xd, off);
      }
      double tj, beta, scale;
      if (sg == 0.0) {
        tj = 0.0;
        beta = xa;
        scale = 0.0;
      } else {
        const double mu = sqrt(fma(xa, xa, sg));
        beta = (xa <= 0.0) ? mu : -mu;
        tj = (beta - xa) / beta;
        scale = 1.0 / (xa - beta);
      }
#pragma unroll
      for (int cc = 0; cc < C; ++cc) {
        if (cc != jc) continue;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int r = lane + 32 * i;
          const double v = r > j + 1 ? a[i][cc] * scale : (r == j + 1 ? 1.0 : 0.0);
          vb[par][r] = v;
          if (r < s) Vh[IDX(r, j, ldv)] = v;
        }
      }
      if (lane == 0) {
        tb[par] = tj;
        d[j] = xd;
        e[j] = beta;
        tau[j] = tj;
      }
      pending(pp, K, -1, jc, j);  // the owner's other columns
    } else {
      pending(pp, K, -1, -1, j);
    }
    __syncthreads();  // barrier 1: v_j, tau_j published; every pending update of step j - 1 applied
    // p_c = tau_j (A v_j)_c for own columns c > j; p^T v partial of this warp
    {
      const double tj = tb[par];
      double vr[R];
#pragma unroll
      for (int i = 0; i < R; ++i) vr[i] = vb[par][lane + 32 * i];
      double acc[C];
#pragma unroll
      for (int cc = 0; cc < C; ++cc) {
        double t = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) t = fma(a[i][cc], vr[i], t);
        acc[cc] = t;
      }
      // transpose reduction: lane ends with the full sum of local column xc (C lanes per column
      // group of 32 / C lanes hold the same value)
#pragma unroll
      for (int h = C / 2, off = 16; h >= 1; h >>= 1, off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int q = 0; q < h; ++q) {
          const double send = up ? acc[q] : acc[q + h];
          const double keep = up ? acc[q + h] : acc[q];
          acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      double tot = acc[0];
#pragma unroll
      for (int off = 16 / C; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
      int xc = 0;
#pragma unroll
      for (int h = C / 2, off = 16; h >= 1; h >>= 1, off >>= 1)
        if (lane & off) xc += h;
      const int c = warp + TW_NW * xc;
      const double pc = c > j ? tj * tot : 0.0;
      const bool rep = (lane & (16 / C * 2 - 1)) == 0;  // one lane per local column
      if (rep) pb[par][c] = pc;
      double pv = rep ? pc * vb[par][c] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, off);
      if (lane == 0) part[par][warp] = pv;
    }
    __syncthreads();  // barrier 2: p_j and the p^T v parts published
  }
  // the last pending update on the trailing 2 x 2 block (or the whole matrix when s <= 2)
  const int last = s - 3;  // the step whose update is pending (none when s <= 2)
  const int pp = last >= 0 ? (last & 1) : 0;
  const double K = last >= 0 ? kprev(pp) : 0.0;
  if (last >= 0) pending(pp, K, -1, -1, last + 1);
#pragma unroll
  for (int cc = 0; cc < C; ++cc) {
    const int c = warp + TW_NW * cc;
    if (c >= s || c < s - 2) continue;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = lane + 32 * i;
      if (r == c) d[c] = a[i][cc];
      if (r == c + 1 && r < s) e[c] = a[i][cc];
    }
  }
}

}  // namespace psd
