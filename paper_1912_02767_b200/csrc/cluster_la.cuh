// cluster_la.cuh -- latency-bound small dense linear algebra of the Rayleigh-Ritz step (a6, a7)
// on one thread-block cluster (up to 16 CTAs on 16 SMs), the matrix distributed column-cyclically
// over the CTAs' shared memory and exchanged through distributed shared memory (DSMEM).
//
//   cholesky_cluster_kernel  G = L L^T of the direction-block Gram (a6, implicit Cholesky-QR,
//                            PAPER.md:395-397); one cluster barrier per column.
//   tridiag_cluster_kernel   Householder tridiagonalisation Q^T H Q = T of the Rayleigh-Ritz
//                            matrix (a7, the eigensolve of Alg. 2); two cluster
//                            barriers per column.
//
// Why a cluster: both factorizations are s sequential column steps. One CTA streams the whole
// trailing matrix through one SM's shared memory per step (s = 400: 1.3 MB does not fit); a
// grid-wide barrier costs microseconds. A 16-CTA cluster holds s <= 640 in 16 x 227 KB of shared
// memory, its barrier costs ~0.2 us (B300_MICROARCH.md: cluster.sync ~380 cycles) and every CTA
// only touches its own s/16 columns per step.
//
// Column g lives in CTA (g % CS) at local column g / CS (leading dimension = matrix order).
// Conventions match tridiag.cuh (LAPACK dsytd2, lower): reflector j has v[j+1] = 1, stored in
// column j of Vh for the back-transformation kernel there.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemm.cuh"  // cp.async helpers

namespace psd {

namespace cg = cooperative_groups;

constexpr int CLA_NT = 512;
constexpr int CLA_MAX = 640;  // largest order held in a 16-CTA cluster's shared memory
constexpr int CLA_SMEM_BYTES = 226 * 1024;  // dynamic smem cap (227 KB minus the static arrays)

__device__ __forceinline__ void cla_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cla_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
template <typename T>
__device__ __forceinline__ T* cla_remote(T* p, unsigned rank) {
  return cg::this_cluster().map_shared_rank(p, rank);
}

__device__ __forceinline__ double cla_block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // red may still be read by a previous call
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

// ------------------------------------------------------------------ Cholesky (a6)
// Blocked right-looking Cholesky on a cluster. Column blocks of CHOL_NB columns are dealt
// block-cyclically (block b -> CTA b % CS, full column storage, ld = t). Per block: the owner
// factors its panel with CTA barriers only, one cluster barrier publishes it, every CTA copies the
// panel (DSMEM) and applies the rank-CHOL_NB update to its own later columns. t/CHOL_NB cluster
// barriers instead of t.
// In place on G (t x t, ld): lower triangle <- L, upper <- 0. status = j + 1 when pivot j is
// <= fail_rel * max diag(G) (R20), else 0.
constexpr int CHOL_NB = 8;
__host__ __device__ inline int chol_local_cols(int t, int CS) { return cdiv(cdiv(t, CHOL_NB), CS) * CHOL_NB; }
__host__ __device__ inline size_t chol_smem_doubles(int t, int CS) {
  return (size_t)chol_local_cols(t, CS) * t + (size_t)CHOL_NB * t + 16;
}

// Blocked Cholesky: panel b = [D; B] (rows j0.., CHOL_NB columns) is factored by its owner as
// L_bb = chol(D) (every thread computes the 8 x 8 factor redundantly in registers) and
// L_B = B L_bb^-T (row-parallel), so a panel costs one CTA barrier; one cluster barrier publishes
// it; every CTA copies it (DSMEM) and applies the rank-CHOL_NB update to its own later columns.
// GA = true (t too large for shared memory): the own columns live in the L2-resident global scratch
// gA (CS * chol_local_cols(t, CS) * t doubles); panels are still exchanged through DSMEM.
__host__ __device__ inline size_t chol_smem_doubles_ga(int t, int CS) { return (size_t)CHOL_NB * t + 16; }
// INV = true (shared-memory variant only): the triangular inverse X = L^-1 is formed alongside
// (right-looking forward substitution on the identity: X_b <- L_bb^-1 X_b, X_{>b} -= L_{>b,b} X_b,
// each CTA on its own columns with the panel it already holds) and written to Linv (ldi).
__host__ __device__ inline size_t chol_inv_smem_doubles(int t, int CS) {
  return 2 * (size_t)chol_local_cols(t, CS) * t + (size_t)CHOL_NB * t + 16;
}
template <bool GA = false, bool INV = false>
__global__ void __launch_bounds__(CLA_NT) cholesky_cluster_kernel(int t, double* __restrict__ G, int ld,
                                                                   double fail_rel, int* __restrict__ status,
                                                                   double* __restrict__ gA,
                                                                   double* __restrict__ Linv, int ldi,
                                                                   int* __restrict__ started = nullptr, int seq = 0) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[33];
  __shared__ double xchs[4];
  const int CS = (int)gridDim.x;
  const unsigned rank = cla_rank();
  // residency signal for a stream that holds back its own work until this cluster is on the SMs
  if (started && rank == 0 && threadIdx.x == 0)
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(started), "r"(seq) : "memory");
  const int ncl = chol_local_cols(t, CS);
  double* Al = GA ? gA + (size_t)rank * ncl * t : sm;  // ncl x t: local column lc = lb * NB + c <-> global (lb * CS + rank) * NB + c
  double* Xl = (INV && !GA) ? sm + (size_t)ncl * t : nullptr;  // ncl x t: own columns of L^-1
  double* pl = GA ? sm : sm + (size_t)(INV ? 2 : 1) * ncl * t;   // NB x t: local copy of the current panel
  double* xch = xchs;                      // [0] max diag part, [1..2] status of panel by parity
  const int tid = threadIdx.x, NT = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = NT >> 5;
  auto gcol = [&](int lc) { return ((lc / CHOL_NB) * CS + (int)rank) * CHOL_NB + (lc % CHOL_NB); };
  for (int e = tid; e < ncl * t; e += NT) {
    int lc = e / t, i = e - lc * t, g = gcol(lc);
    Al[e] = (g < t) ? G[IDX(i, g, ld)] : 0.0;
    if (INV) Xl[e] = (i == g) ? 1.0 : 0.0;
  }
  __syncthreads();
  double mx = 0.0;
  for (int lc = tid; lc < ncl; lc += NT) {
    int g = gcol(lc);
    if (g < t) mx = fmax(mx, Al[(size_t)lc * t + g]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < nw; ++w) m = fmax(m, red[w]);
    xch[0] = m;
    xch[1] = xch[2] = 0.0;
  }
  cla_cluster_sync();
  if (tid < 32) {
    double m = (tid < CS) ? *cla_remote(xch, (unsigned)tid) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tid == 0) red[32] = m;
  }
  __syncthreads();
  const double floor_ = fail_rel * red[32];
  const int nblk = cdiv(t, CHOL_NB);
  int fail = 0;
  for (int b = 0; b < nblk; ++b) {
    const int owner = b % CS, par = b & 1, j0 = b * CHOL_NB, jb = min(CHOL_NB, t - j0);
    const int jn = j0 + jb;  // first column after the panel
    if ((int)rank == owner) {
      double* P = Al + (size_t)(b / CS) * CHOL_NB * t;
      // redundant 8 x 8 Cholesky of the diagonal block in registers
      double Lb[CHOL_NB][CHOL_NB];
#pragma unroll
      for (int c = 0; c < CHOL_NB; ++c)
#pragma unroll
        for (int r = 0; r < CHOL_NB; ++r) Lb[r][c] = (r >= c && c < jb && r < jb) ? P[(size_t)c * t + j0 + r] : 0.0;
      int f = 0;
      double dinv[CHOL_NB];
#pragma unroll
      for (int c = 0; c < CHOL_NB; ++c) {
        dinv[c] = 0.0;
        if (c < jb && !f) {
          double dcc = Lb[c][c];
#pragma unroll
          for (int k = 0; k < c; ++k) dcc = fma(-Lb[c][k], Lb[c][k], dcc);
          if (!(dcc > floor_)) {
            f = j0 + c + 1;
          } else {
            const double lcc = sqrt(dcc), inv = 1.0 / lcc;
            Lb[c][c] = lcc;
            dinv[c] = inv;
#pragma unroll
            for (int r = c + 1; r < CHOL_NB; ++r) {
              if (r < jb) {
                double v = Lb[r][c];
#pragma unroll
                for (int k = 0; k < c; ++k) v = fma(-Lb[r][k], Lb[c][k], v);
                Lb[r][c] = v * inv;
              }
            }
          }
        }
      }
      __syncthreads();  // every thread has read the diagonal block
      if (!f) {
        // diagonal block <- L_bb (lower), rows below <- B L_bb^-T (row-parallel forward substitution)
        if (tid < CHOL_NB * CHOL_NB) {
          const int r = tid % CHOL_NB, c = tid / CHOL_NB;
          if (r < jb && c < jb && r >= c) {
            double v = 0.0;
#pragma unroll
            for (int rr = 0; rr < CHOL_NB; ++rr)
#pragma unroll
              for (int cc = 0; cc < CHOL_NB; ++cc)
                if (rr == r && cc == c) v = Lb[rr][cc];
            P[(size_t)c * t + j0 + r] = v;
          }
        }
        for (int i = jn + tid; i < t; i += NT) {
          double x[CHOL_NB];
#pragma unroll
          for (int c = 0; c < CHOL_NB; ++c) x[c] = (c < jb) ? P[(size_t)c * t + i] : 0.0;
#pragma unroll
          for (int c = 0; c < CHOL_NB; ++c) {
            double v = x[c];
#pragma unroll
            for (int k = 0; k < c; ++k) v = fma(-x[k], Lb[c][k], v);
            x[c] = v * dinv[c];
          }
#pragma unroll
          for (int c = 0; c < CHOL_NB; ++c)
            if (c < jb) P[(size_t)c * t + i] = x[c];
        }
      }
      if (tid == 0) xch[1 + par] = (double)f;
    }
    cla_cluster_sync();  // panel b factored and visible
    {
      const double f = *cla_remote(xch + 1 + par, (unsigned)owner);
      if (f != 0.0) {
        fail = (int)f;
        break;
      }
    }
    if (jn >= t && !INV) break;
    const int cr0 = INV ? j0 : jn;  // first panel row copied (the diagonal block too when forming L^-1)
    {
      const double* P = GA ? gA + ((size_t)owner * ncl + (size_t)(b / CS) * CHOL_NB) * t
                           : cla_remote(Al + (size_t)(b / CS) * CHOL_NB * t, (unsigned)owner);
      const int len = t - cr0, tot = jb * len;
      int e = tid;
      for (; e + 3 * NT < tot; e += 4 * NT) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int ee = e + u * NT, c = ee / len, i = cr0 + (ee - c * len);
          v[u] = P[(size_t)c * t + i];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int ee = e + u * NT, c = ee / len, i = cr0 + (ee - c * len);
          pl[(size_t)c * t + i] = v[u];
        }
      }
      for (; e < tot; e += NT) {
        int c = e / len, i = cr0 + (e - c * len);
        pl[(size_t)c * t + i] = P[(size_t)c * t + i];
      }
    }
    __syncthreads();
    if (INV) {
      // own columns g < jn of X: X[j0:jn, g] <- L_bb^-1 X[j0:jn, g]; X[jn:, g] -= L[jn:, j0:jn] X[j0:jn, g]
      for (int lc = warp; lc < ncl; lc += nw) {
        const int g = gcol(lc);
        if (g >= jn || g >= t) continue;
        double* xc = Xl + (size_t)lc * t;
        double xb[CHOL_NB];
#pragma unroll
        for (int c = 0; c < CHOL_NB; ++c) xb[c] = (c < jb) ? xc[j0 + c] : 0.0;
#pragma unroll
        for (int c = 0; c < CHOL_NB; ++c) {
          if (c < jb) {
            double v = xb[c];
#pragma unroll
            for (int k = 0; k < c; ++k) v = fma(-pl[(size_t)k * t + j0 + c], xb[k], v);
            xb[c] = v / pl[(size_t)c * t + j0 + c];
          }
        }
        __syncwarp();
        if (lane < jb) {
          double v = 0.0;
#pragma unroll
          for (int c = 0; c < CHOL_NB; ++c)
            if (c == lane) v = xb[c];
          xc[j0 + lane] = v;
        }
        for (int i = jn + lane; i < t; i += 32) {
          double a = xc[i];
#pragma unroll
          for (int c = 0; c < CHOL_NB; ++c)
            if (c < jb) a = fma(-pl[(size_t)c * t + i], xb[c], a);
          xc[i] = a;
        }
      }
      if (jn >= t) break;
    }
    // own columns g >= jn: G[i][g] -= sum_c L[i][j0+c] L[g][j0+c], i >= g (warp per column)
    for (int lc = warp; lc < ncl; lc += nw) {
      const int g = gcol(lc);
      if (g < jn || g >= t) continue;
      double lgc[CHOL_NB];
#pragma unroll
      for (int c = 0; c < CHOL_NB; ++c) lgc[c] = (c < jb) ? pl[(size_t)c * t + g] : 0.0;
      double* col = Al + (size_t)lc * t;
      int i = g + lane;
      for (; i + 32 < t; i += 64) {
        double a0 = col[i], a1 = col[i + 32];
#pragma unroll
        for (int c = 0; c < CHOL_NB; ++c) {
          a0 = fma(-pl[(size_t)c * t + i], lgc[c], a0);
          a1 = fma(-pl[(size_t)c * t + i + 32], lgc[c], a1);
        }
        col[i] = a0;
        col[i + 32] = a1;
      }
      if (i < t) {
        double a0 = col[i];
#pragma unroll
        for (int c = 0; c < CHOL_NB; ++c) a0 = fma(-pl[(size_t)c * t + i], lgc[c], a0);
        col[i] = a0;
      }
    }
    __syncthreads();
  }
  if (rank == 0 && tid == 0) *status = fail;
  if (!fail) {
    __syncthreads();
    for (int e = tid; e < ncl * t; e += NT) {
      int lc = e / t, i = e - lc * t, g = gcol(lc);
      if (g < t) {
        G[IDX(i, g, ld)] = (i >= g) ? Al[e] : 0.0;
        if (INV) Linv[IDX(i, g, ldi)] = (i >= g) ? Xl[e] : 0.0;
      }
    }
  }
  cla_cluster_sync();  // no CTA leaves while its shared memory may still be read
}

// ------------------------------------------------------------------ tridiagonalisation (a7)
// A (s x s, lda) symmetric (symmetrised on load, never modified). Outputs d[s], e[s-1], tau[s-2]
// and the reflectors in Vh (s x s, ldv: column j rows j+1..s-1).
// Column g lives in CTA g % CS (local column g / CS, ld = s). The rank-2 update of step j-1 is
// applied lazily, fused with the matrix-vector product of step j (one pass over the own columns
// per step), except for column j, which the owner's warp 0 updates eagerly before forming the
// Householder vector of step j. Step j:
//   owner(j), warp 0: column j <- step j-1 update; Householder v_j, tau_j; v_j[i] is stored into
//                     CTA (i % CS)'s vloc (DSMEM stores), tau_j into every CTA's vloc[j]
//   B1 (cluster barrier)
//   all:  v_j <- gather of the interleaved pieces (DSMEM), so no CTA's port serves the broadcast
//         rows split over the threads: for own columns g > j, A[r, g] -= v'_r a'_g + p'_r v'_g
//         (step j-1, a' = p'_g - 2 K' v'_g) and partial dots A[r, g] v_j[r]; column sums -> p_g
//   B2
//   all:  p_j <- gather (DSMEM); K_j = tau_j / 2 * sum of the CTAs' partials of p.v_j
// (Column sums are reduced in a fixed order: results are deterministic.)
constexpr int TRI_CB = 8;  // own columns processed per batch (independent reduction chains)
__host__ __device__ inline size_t tri_smem_doubles(int s, int CS) {
  return (size_t)cdiv(s, CS) * s + 5 * (size_t)s + 3 * (size_t)cdiv(s, CS) + 16 * (size_t)(cdiv(s, CS) + TRI_CB) + 2 * 32 +
         16;
}
// GA = true (s too large for the cluster's shared memory): the own columns live in the global
// scratch gA (L2-resident; CS * cdiv(s, CS) * s doubles), everything else as above.
__host__ __device__ inline size_t tri_smem_doubles_ga(int s, int CS) {
  return 5 * (size_t)s + 3 * (size_t)cdiv(s, CS) + 16 * (size_t)(cdiv(s, CS) + TRI_CB) + 2 * 32 + 16 + 1300;
}

// Householder vector of step j by the owner's warp 0 (rows i = j + lane + 32 q, q < Q): eager
// update of column j with step j-1, sigma, (tau, beta), v_j pushed to its interleaved holders
// (DSMEM stores; tau_j to every CTA) and kept in column j as reflector storage. No global stores:
// a release barrier would wait for them to reach L2.
template <int Q>
__device__ __forceinline__ void tri_house(int j, int s, int CS, double* __restrict__ col,
                                          const double* __restrict__ vp, const double* __restrict__ pq, double Kq,
                                          bool pend, double* __restrict__ vb, double* __restrict__ dj_out,
                                          double* __restrict__ e_out, double* __restrict__ t_out,
                                          double* __restrict__ vout) {
  const int lane = threadIdx.x & 31;
  double ag = 0.0, bg = 0.0;
  if (pend) {
    bg = vp[j];
    ag = pq[j] - 2.0 * Kq * bg;
  }
  double x[Q];
  const double* cp = col + j + lane;
#pragma unroll
  for (int q = 0; q < Q; ++q) x[q] = cp[32 * q];
  if (pend) {
#pragma unroll
    for (int q = 0; q < Q; ++q) x[q] = fma(-vp[j + lane + 32 * q], ag, fma(-pq[j + lane + 32 * q], bg, x[q]));
  }
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = j + lane + 32 * q;
    const double xs = (i >= j + 2 && i < s) ? x[q] : 0.0;
    acc = fma(xs, xs, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const double sigma = acc;
  const double alpha = __shfl_sync(0xffffffffu, x[0], 1);  // row j + 1 sits in lane 1, slot 0
  const double dj = __shfl_sync(0xffffffffu, x[0], 0);
  double tj, beta, scale;
  if (sigma == 0.0) {
    tj = 0.0;
    beta = alpha;
    scale = 0.0;
  } else {
    const double mu = sqrt(fma(alpha, alpha, sigma));
    beta = (alpha <= 0.0) ? mu : -mu;
    tj = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
  if (lane == 0) {
    *dj_out = dj;
    *e_out = beta;
    *t_out = tj;
  }
  if (lane < CS) *cla_remote(vb + j, (unsigned)lane) = tj;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = j + lane + 32 * q;
    if (i > j && i < s) {
      const double v = (i == j + 1) ? 1.0 : x[q] * scale;
      *cla_remote(vb + i, (unsigned)(i & (CS - 1))) = v;
      vout[i] = v;
    }
  }
}

// Fused loop of one tridiagonalisation step on the CTA's own columns g > j (column per warp, rows
// i = j + 1 + lane + 32 q for q < Q; rows >= s read finite padding, masked by v_j = 0 and by the
// store predicate). Q <= 20: v', p', v_j in registers; larger Q re-reads v', p' per column.
template <int Q>
__device__ __forceinline__ double tri_fused_cols(int j, int s, int CS, unsigned rank, int ncl, int warp, int nw,
                                                 int lane, bool pend, double Kp, double tj, double* __restrict__ Al,
                                                 const double* __restrict__ vprow, const double* __restrict__ pprow,
                                                 const double* __restrict__ vj, double* __restrict__ pbuf, int dbg) {
  constexpr bool REG = Q <= 20;
  const int i0 = j + 1 + lane;
  double rj[Q], rv[REG ? Q : 1], rp[REG ? Q : 1];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const bool ok = i0 + 32 * q < s;
    rj[q] = ok ? vj[i0 + 32 * q] : 0.0;
    if (REG) {
      rv[REG ? q : 0] = (ok && pend) ? vprow[i0 + 32 * q] : 0.0;
      rp[REG ? q : 0] = (ok && pend) ? pprow[i0 + 32 * q] : 0.0;
    }
  }
  const int lc0 = (j + 1 > (int)rank) ? (j + 1 - (int)rank + CS - 1) / CS : 0;
  double part = 0.0;
  for (int lc = lc0 + warp; lc < ncl && !(dbg & 1); lc += nw) {
    const int g = (int)rank + CS * lc;
    if (g >= s) break;
    double* cp = Al + (size_t)lc * s + i0;
    double a0 = 0.0, a1 = 0.0;
    if (pend) {
      const double bg = vprow[g];
      const double ag = pprow[g] - 2.0 * Kp * bg;
      double x[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const double vq = REG ? rv[REG ? q : 0] : vprow[i0 + 32 * q];
        const double pq = REG ? rp[REG ? q : 0] : pprow[i0 + 32 * q];
        x[q] = fma(-vq, ag, fma(-pq, bg, cp[32 * q]));
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (q & 1)
          a1 = fma(x[q], rj[q], a1);
        else
          a0 = fma(x[q], rj[q], a0);
        if (i0 + 32 * q < s) cp[32 * q] = x[q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (q & 1)
          a1 = fma(cp[32 * q], rj[q], a1);
        else
          a0 = fma(cp[32 * q], rj[q], a0);
      }
    }
    double acc = a0 + a1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    acc *= tj;
    if (lane == 0) pbuf[g] = acc;
    part = fma(acc, vj[g], part);
  }
  return part;
}

template <int PL, int TNT, bool GA = false>
__global__ void __launch_bounds__(TNT) tridiag_cluster_kernel(int s, const double* __restrict__ A, int lda,
                                                                  double* __restrict__ d, double* __restrict__ e,
                                                                  double* __restrict__ tau, double* __restrict__ Vh,
                                                                  int ldv, long long* __restrict__ prof,
                                                                  double* __restrict__ gA, int dbg) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double Kbuf[2];
  long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = 0;
#define TRI_T(k)                  \
  if (prof && threadIdx.x == 0) { \
    long long tn = clock64();     \
    pt[k] += tn - tprev;          \
    tprev = tn;                   \
  }
  const int CS = (int)gridDim.x;
  const unsigned rank = cla_rank();
  const int ncl = cdiv(s, CS);
  double* Al = GA ? gA + (size_t)rank * ncl * s : sm;  // ncl x s, own columns
  double* vloc = GA ? sm : Al + (size_t)ncl * s;        // 2 x s (parity): [tau_j at index j | v_j at j+1..s-1]
  double* ploc = vloc + 2 * (size_t)s;                  // 2 x s (parity): gathered p_j (all rows)
  double* pbuf = ploc + 2 * (size_t)s;                  // own entries of p_j (global column index), read remotely
  double* wpart = pbuf + s;                             // 2 x 32: per-warp partials of p.v (parity)
  double* dl = wpart + 64;                              // d, e, tau of own columns (written out at the end)
  double* el = dl + ncl;
  double* tl = el + ncl;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = NT >> 5;
  if (GA) {
    for (size_t q = tid; q < tri_smem_doubles_ga(s, CS); q += NT) sm[q] = 0.0;
  } else {
    for (size_t q = (size_t)ncl * s + tid; q < tri_smem_doubles(s, CS); q += NT) sm[q] = 0.0;
  }
  for (int q = tid; q < ncl * s; q += NT) {
    int lc = q / s, i = q - lc * s, g = (int)rank + CS * lc;
    Al[q] = (g < s) ? 0.5 * (A[IDX(i, g, lda)] + A[IDX(g, i, lda)]) : 0.0;
  }
  __syncthreads();
  cla_cluster_sync();  // every CTA is running before the first DSMEM store
  if (prof && threadIdx.x == 0) tprev = clock64();
  for (int j = 0; j + 2 < s; ++j) {
    const int owner = j % CS, par = j & 1, pp = par ^ 1;
    const bool pend = j > 0;  // step j-1's update is pending on columns > j
    if ((int)rank == owner && warp == 0) {
      const int nqh = (s - j + 31) >> 5;  // rows j..s-1
      double* col = Al + (size_t)(j / CS) * s;
#define TRI_HOUSE(QQ) tri_house<QQ>(j, s, CS, col, vloc + (size_t)pp * s, ploc + (size_t)pp * s, Kbuf[pp], pend, \
                                    vloc + (size_t)par * s, dl + j / CS, el + j / CS, tl + j / CS, col)
      if (nqh <= 2)
        TRI_HOUSE((PL < 2 ? PL : 2));
      else if (nqh <= 4)
        TRI_HOUSE((PL < 4 ? PL : 4));
      else if (nqh <= 8)
        TRI_HOUSE((PL < 8 ? PL : 8));
      else if (nqh <= 14)
        TRI_HOUSE((PL < 14 ? PL : 14));
      else if (nqh <= 20)
        TRI_HOUSE((PL < 20 ? PL : 20));
      else
        TRI_HOUSE(PL);
#undef TRI_HOUSE
    }
    TRI_T(0);
    cla_cluster_sync();  // B1: v_j pieces and tau_j visible; step j-1 finished everywhere
    TRI_T(1);
    double* vj = vloc + (size_t)par * s;
    {
      int i = j + 1 + tid;
      for (; i + NT < s; i += 2 * NT) {
        const int r0 = i & (CS - 1), r1 = (i + NT) & (CS - 1);
        const double a = (r0 == (int)rank) ? vj[i] : *cla_remote(vj + i, (unsigned)r0);
        const double b = (r1 == (int)rank) ? vj[i + NT] : *cla_remote(vj + i + NT, (unsigned)r1);
        vj[i] = a;
        vj[i + NT] = b;
      }
      if (i < s) {
        const int r0 = i & (CS - 1);
        if (r0 != (int)rank) vj[i] = *cla_remote(vj + i, (unsigned)r0);
      }
    }
    __syncthreads();
    TRI_T(2);
    const double tj = vj[j];
    const double Kp = pend ? Kbuf[pp] : 0.0;
    // fused pending update (step j-1) + p_g = tau_j A[:, g] . v_j over the own columns g > j; the
    // row loop length is dispatched on the trailing size (no work on rows past s)
    const int nq = (s - j - 1 + 31) >> 5;
    const double* vprow = vloc + (size_t)pp * s;
    const double* pprow = ploc + (size_t)pp * s;
    double part;
#define TRI_COLS(QQ) tri_fused_cols<QQ>(j, s, CS, rank, ncl, warp, nw, lane, pend, Kp, tj, Al, vprow, pprow, vj, pbuf, dbg)
    if (nq <= 2)
      part = TRI_COLS((PL < 2 ? PL : 2));
    else if (nq <= 4)
      part = TRI_COLS((PL < 4 ? PL : 4));
    else if (nq <= 8)
      part = TRI_COLS((PL < 8 ? PL : 8));
    else if (nq <= 14)
      part = TRI_COLS((PL < 14 ? PL : 14));
    else if (nq <= 20)
      part = TRI_COLS((PL < 20 ? PL : 20));
    else
      part = TRI_COLS(PL);
#undef TRI_COLS
    if (lane == 0) wpart[par * 32 + warp] = part;
    TRI_T(3);
    cla_cluster_sync();  // B2: p_j entries and partials visible
    TRI_T(4);
    double* pj = ploc + (size_t)par * s;
    {
      int i = j + 1 + tid;
      for (; i + NT < s; i += 2 * NT) {
        const double a = *cla_remote(pbuf + i, (unsigned)(i & (CS - 1)));
        const double b = *cla_remote(pbuf + i + NT, (unsigned)((i + NT) & (CS - 1)));
        pj[i] = a;
        pj[i + NT] = b;
      }
      if (i < s) pj[i] = *cla_remote(pbuf + i, (unsigned)(i & (CS - 1)));
    }
    if (warp == nw - 1) {
      double pv = 0.0;
      for (int q = lane; q < nw * CS; q += 32) pv += *cla_remote(wpart + par * 32 + (q % nw), (unsigned)(q / nw));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
      if (lane == 0) Kbuf[par] = 0.5 * tj * pv;
    }
    TRI_T(5);
    __syncthreads();
    TRI_T(6);
  }
  if (prof && threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) prof[rank * 8 + k] = pt[k];
#undef TRI_T
  // pending update of the last step on columns s-2, s-1 (rows >= s-2), then the trailing 2 x 2
  if (s >= 3) {
    const int jl = s - 3, pl = jl & 1;
    const double* vp = vloc + (size_t)pl * s;
    const double* pq = ploc + (size_t)pl * s;
    const double Kp = Kbuf[pl];
    if (tid < 4) {
      const int g = s - 2 + (tid >> 1), i = s - 2 + (tid & 1);
      if ((int)rank == g % CS) {
        double* col = Al + (size_t)(g / CS) * s;
        const double bg = vp[g], ag = pq[g] - 2.0 * Kp * bg;
        col[i] -= vp[i] * ag + pq[i] * bg;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (s >= 2) {
      int g = s - 2;
      if ((int)rank == g % CS) {
        d[g] = Al[(size_t)(g / CS) * s + g];
        e[g] = Al[(size_t)(g / CS) * s + g + 1];
      }
      g = s - 1;
      if ((int)rank == g % CS) d[g] = Al[(size_t)(g / CS) * s + g];
    } else if (rank == 0) {
      d[0] = Al[0];
    }
  }
  // reflectors (own columns g <= s-3, rows g+1..s-1) and d, e, tau of the own columns
  for (int q = tid; q < ncl * s; q += NT) {
    int lc = q / s, i = q - lc * s, g = (int)rank + CS * lc;
    if (g + 2 < s && i > g) Vh[IDX(i, g, ldv)] = Al[q];
  }
  for (int lc = tid; lc < ncl; lc += NT) {
    int g = (int)rank + CS * lc;
    if (g + 2 < s) {
      d[g] = dl[lc];
      e[g] = el[lc];
      tau[g] = tl[lc];
    }
  }
  cla_cluster_sync();  // no CTA leaves while its shared memory may still be read
}

// ---- push-style DSMEM exchange: st.async into the receiver's shared memory, completing on the
// receiver's mbarrier (one hop, no cluster barrier; tools/micro/push_bench.cu: ~570 cycles for a
// one-double broadcast hop against ~1.6k for barrier.cluster + remote load)
__device__ __forceinline__ uint32_t cla_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cla_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cla_mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cla_smem_u32(b)), "r"(cnt) : "memory");
}
// the local arrival of a phase, announcing the bytes the phase will receive
__device__ __forceinline__ void cla_mbar_arm(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(cla_smem_u32(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void cla_mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nCLA_WAIT_%=: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra CLA_WAIT_%=;\n}\n" ::"r"(cla_smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cla_st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}

// Register-resident, push-exchanged tridiagonalisation (s <= 64 KR, cdiv(s, CS) <= TRI_TCG CR):
// the own columns live in registers, so a step moves no matrix bytes through shared memory, and
// the exchanges of a step are one-way pushes completing on the receiver's mbarrier instead of
// cluster barriers + remote loads (tools/micro/push_bench*.cu: ~0.9k cycles per st.async hop
// against ~1.6k for barrier.cluster + remote load).
// Thread t: column group cg = t / 64 (two warps), rows r = t % 64 + 64 k (k < KR), own local
// columns lc = cg + TRI_TCG c (c < CR). Step j (parity buffers par = j & 1, mbarrier phase j >> 1):
//   U1  owner(j): the threads of column j apply the pending update (step j-1) to it, copy it to
//       colb and reduce sigma = ||A[j+2:, j]||^2; Householder scalars; v_j written to the
//       reflector store (tau_j at row j) and sent by one bulk copy (cp.async.bulk
//       shared::cta -> shared::cluster) per CTA, completing on each CTA's vbar
//   U2  all: the pending update on the other own columns (overlaps the flight of v_j)
//   D   all: wait vbar; acc[c] = sum_r a[r][c] v_j[r] (rows > j); column sums by an in-warp
//       transpose reduction + the group's two warps; p_g = tau_j sum for own g > j st.async'ed to
//       every CTA's ploc[par][g], the CTA's part of p.v_j to wpart[par][rank] (pbar, warp w
//       serving destinations w, w + 8); wait pbar; K_j = tau_j / 2 sum(wpart)
// Two hops per column (the owner's broadcast, the p all-gather): the step is latency-bound.
// Buffer reuse is ordered by the data dependencies: nothing is written into a parity-par buffer
// for step j + 2 before every CTA has pushed p_{j+1}, i.e. finished reading step j's buffers.
// Each CTA re-arms a barrier for step j + 2 right after observing its step-j phase (by then no
// step-(j+2) bytes can have arrived), so no phase ever sees bytes before its expect_tx.
__constant__ int g_tri_bulk_spread = 0;  // set by the host (PSDPROJ_TRI_SPREAD)
constexpr int TRI_TCG = 4;
__host__ __device__ inline size_t tri_reg_smem_doubles(int s, int CS) {
  const size_t sr = (size_t)((s + 1) & ~1);
  return (size_t)cdiv(s, CS) * sr + 4 * sr + 3 * (size_t)cdiv(s, CS) + (s + 256) + 2 * 8 * 32 + 64 + 16;
}
template <int N>
__device__ __forceinline__ double tri_xreduce(double (&v)[N], int lane) {
  // transpose reduction: after log2 N halving levels lane holds column c(lane) summed over the
  // lanes that agree with it in bits 4 .. 5 - log2 N; the remaining levels sum those lanes
#pragma unroll
  for (int h = N / 2, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double r = v[0];
#pragma unroll
  for (int o = 16 / N; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}
template <int N>
__device__ __forceinline__ int tri_xreduce_col(int lane) {
  int c = 0;
#pragma unroll
  for (int h = N / 2, o = 16; h >= 1; h >>= 1, o >>= 1)
    if (lane & o) c += h;
  return c;
}
__host__ __device__ constexpr int tri_pow2_ceil(int n) { return n <= 1 ? 1 : 2 * tri_pow2_ceil((n + 1) / 2); }

template <int KR, int CR>
__global__ void __launch_bounds__(256, 1) tridiag_reg_kernel(int s, const double* __restrict__ A, int lda,
                                                             double* __restrict__ d, double* __restrict__ e,
                                                             double* __restrict__ tau, double* __restrict__ Vh, int ldv,
                                                             long long* __restrict__ prof, int dbg) {
  constexpr int NT = 256, RG = 64, TCG = TRI_TCG, CRP = tri_pow2_ceil(CR);
  static_assert(RG * TCG == NT, "thread layout");
  static_assert(CRP <= 32, "columns per thread");
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t vbar[2], pbar[2];
  __shared__ double hsm[18];
  long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, po[4] = {0, 0, 0, 0};
  long long tprev = 0;
#define TRI_O(k)                                                          \
  if (prof && threadIdx.x == 0) {                                         \
    long long tn;                                                         \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(tn)::"memory");          \
    po[k] += tn - tprev;                                                  \
    tprev = tn;                                                           \
  }
#define TRI_T(k)                                                          \
  if (prof && threadIdx.x == 0) {                                         \
    long long tn;                                                         \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(tn)::"memory");          \
    pt[k] += tn - tprev;                                                  \
    tprev = tn;                                                           \
  }
  const int CS = (int)gridDim.x, lcs = __ffs(CS) - 1;  // CS in {4, 8, 16}
  const unsigned rank = cla_rank();
  const int ncl = cdiv(s, CS);  // <= 32 (one lane per own column in the p push)
  const int sr = (s + 1) & ~1;             // even row stride: 16-byte aligned bulk copies
  double* refl = sm;                       // ncl x sr: reflectors of the own columns (tau_j at row j)
  double* vloc = refl + (size_t)ncl * sr;  // 2 x sr (parity): [tau_j at index j | v_j at j+1..s-1]
  double* ploc = vloc + 2 * (size_t)sr;    // 2 x sr (parity): p_j (pushed by the column owners)
  double* colb = ploc + 2 * (size_t)sr;    // column j for the owner's Householder step (s + 256: tail pad)
  double* wred = colb + s + 256;          // 2 x 8 warps x 32: per-warp column partials (parity)
  double* wpart = wred + 2 * 8 * 32;      // 2 x 32 (parity): every CTA's part of p.v_j, by rank
  double* dl = wpart + 64;
  double* el = dl + ncl;
  double* tl = el + ncl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cg = tid / RG, rg = tid % RG;
  for (size_t q = tid; q < tri_reg_smem_doubles(s, CS); q += NT) sm[q] = 0.0;
  double a[KR][CR];
#pragma unroll
  for (int c = 0; c < CR; ++c) {
    const int g = (int)rank + CS * (cg + TCG * c);
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = rg + RG * k;
      a[k][c] = (g < s && r < s) ? 0.5 * (A[IDX(r, g, lda)] + A[IDX(g, r, lda)]) : 0.0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      cla_mbar_init(&vbar[b], 1);
      cla_mbar_init(&pbar[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int jj = 0; jj < 2 && jj + 2 < s; ++jj) {
      cla_mbar_arm(&vbar[jj], 8u * (uint32_t)(sr - (jj & ~1)));
      cla_mbar_arm(&pbar[jj], 8u * (uint32_t)(s - jj - 1 + CS));
    }
  }
  __syncthreads();
  cla_cluster_sync();  // every CTA's barriers are initialised and armed before the first push
  if (prof && threadIdx.x == 0) tprev = clock64();
  double Kp = 0.0;  // K_{j-1}
  for (int j = 0; j + 2 < s; ++j) {
    const int owner = j & (CS - 1), par = j & 1, pp = par ^ 1;
    const uint32_t ph = (uint32_t)(j >> 1) & 1u;
    const bool pend = j > 0;
    const bool rearm = tid == 0 && j + 4 < s;  // step j + 2 exists
    double* vj = vloc + (size_t)par * sr;
    const double* vp = vloc + (size_t)pp * sr;
    const double* pq = ploc + (size_t)pp * sr;
    // ---- U: the pending update of step j-1 (rows >= j), column j first on its owner
    double rv[KR], rp[KR], ag[CR], bg[CR];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = rg + RG * k;
      const bool ok = pend && r >= j && r < s;
      rv[k] = ok ? vp[r] : 0.0;
      rp[k] = ok ? pq[r] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < CR; ++c) {
      const int g = (int)rank + CS * (cg + TCG * c);
      const bool act = pend && g >= j && g < s;
      const int gi = act ? g : 0;
      bg[c] = act ? vp[gi] : 0.0;
      ag[c] = act ? pq[gi] - 2.0 * Kp * bg[c] : 0.0;
    }
    if ((int)rank == owner) {
      // column j = local column lj: group lj % TCG (two warps), slot lj / TCG. Its threads update
      // it, copy it to colb and form the partial sums of sigma = ||A[j+2:, j]||^2.
      const int lj = j >> lcs, cgj = lj & (TCG - 1), cj = lj >> 2;
      if (cg == cgj) {
        double sg = 0.0;
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          if (c == cj) {
#pragma unroll
            for (int k = 0; k < KR; ++k) {
              const int r = rg + RG * k;
              const double x = fma(-rv[k], ag[c], fma(-rp[k], bg[c], a[k][c]));
              a[k][c] = x;
              if (r >= j && r < s) {
                colb[r] = x;
                if (r >= j + 2) sg = fma(x, x, sg);
                if (r == j) hsm[16] = x;
                if (r == j + 1) hsm[17] = x;
              }
            }
            ag[c] = 0.0;  // done: the U2 pass below must not apply it again
            bg[c] = 0.0;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
        if (lane == 0) hsm[warp & 1] = sg;
      }
      TRI_O(0);
      __syncthreads();
      TRI_O(1);
      // Householder vector (LAPACK dlarfg, beta = -sign(alpha) ||(alpha, x)||): 1/mu from rsqrt,
      // 1/(alpha - beta) from a refined reciprocal (the owner's critical path)
      const double sigma = hsm[0] + hsm[1];
      const double dj = hsm[16], alpha = hsm[17];
      double tj, beta, scale;
      if (sigma == 0.0) {
        tj = 0.0;
        beta = alpha;
        scale = 0.0;
      } else {
        const double ss = fma(alpha, alpha, sigma);
        const double rr = rsqrt(ss);
        const double mu = ss * rr;
        beta = (alpha <= 0.0) ? mu : -mu;
        tj = fma(alpha, (alpha <= 0.0) ? -rr : rr, 1.0);  // (beta - alpha) / beta
        const double dd = alpha - beta;
        double rc;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(dd));
        double ee = fma(-dd, rc, 1.0);
        rc = fma(rc, ee, rc);
        ee = fma(-dd, rc, 1.0);
        scale = fma(rc, ee, rc);
      }
      TRI_O(2);
      if (tid == 0) {
        dl[lj] = dj;
        el[lj] = beta;
        tl[lj] = tj;
      }
      // v_j (rows > j) into the reflector store with tau_j at row j, then one bulk copy per CTA of
      // rows [j & ~1, sr) (row j - 1, when copied, is dead at the receivers) completing on its vbar
      double* vout = refl + (size_t)lj * sr;
      for (int i = j + 1 + tid; i < s; i += NT) vout[i] = (i == j + 1) ? 1.0 : colb[i] * scale;
      if (tid == 0) vout[j] = tj;
      __syncthreads();
      // one bulk copy per destination CTA, issued by lanes 0-1 of every warp (g_tri_bulk_spread) or by
      // lanes 0..CS-1 of warp 0: a warp's bulk-copy lanes are issued one after another
      const int bdst = g_tri_bulk_spread ? (((tid & 31) < 2) ? 2 * warp + (tid & 31) : CS) : tid;
      if (bdst < CS) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int i0 = j & ~1;
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                cla_mapa(cla_smem_u32(vj + i0), (uint32_t)bdst)),
            "r"(cla_smem_u32(vout + i0)), "r"(8u * (uint32_t)(sr - i0)), "r"(cla_mapa(cla_smem_u32(&vbar[par]), (uint32_t)bdst))
            : "memory");
      }
      if (prof && tid == 0) pt[7] += 1;
    }
    TRI_T(0);
    // U2: the other own columns (overlaps the flight of v_j)
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      if (pend && RG * k < s && RG * k + RG - 1 >= j) {
#pragma unroll
        for (int c = 0; c < CR; ++c) a[k][c] = fma(-rv[k], ag[c], fma(-rp[k], bg[c], a[k][c]));
      }
    }
    TRI_T(5);
    cla_mbar_wait(&vbar[par], ph);  // tau_j and all rows of v_j
    if (rearm) cla_mbar_arm(&vbar[par], 8u * (uint32_t)(sr - ((j + 2) & ~1)));
    TRI_T(1);
    TRI_T(2);
    // ---- D: column sums of A[:, g] v_j (rows > j) for the own columns
    const double tj = vj[j];
    double rj[KR], acc[CRP];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = rg + RG * k;
      rj[k] = (r > j && r < s) ? vj[r] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < CRP; ++c) acc[c] = 0.0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      if (RG * k < s && RG * k + RG - 1 > j) {
#pragma unroll
        for (int c = 0; c < CR; ++c) acc[c] = fma(a[k][c], rj[k], acc[c]);
      }
    }
    if constexpr (CRP > CR) {
      // the thread's part of p.v_j / tau_j rides in the reduction's spare slot CR (no separate
      // warp reduction before the push)
      double q = 0.0;
#pragma unroll
      for (int c = 0; c < CR; ++c) {
        const int g = (int)rank + CS * (cg + TCG * c);
        if (g > j && g < s) q = fma(acc[c], vj[g], q);
      }
      acc[CR] = q;
    }
    double* wr = wred + par * 256;
    {
      const double w = tri_xreduce<CRP>(acc, lane);
      if ((lane & (32 / CRP - 1)) == 0) wr[warp * 32 + tri_xreduce_col<CRP>(lane)] = w;
    }
    TRI_T(6);
    __syncthreads();
    {
      // p_g of the own columns (lane = local column), pushed by every warp to destinations
      // warp, warp + 8
      double part = 0.0, pg = 0.0;
      const int lc = lane, g = (int)rank + CS * lc;
      const bool act = lc < ncl && g > j && g < s;
      if (act) {
        const int cgl = lc % TCG, c = lc / TCG;
        pg = tj * (wr[(2 * cgl) * 32 + c] + wr[(2 * cgl + 1) * 32 + c]);
      }
      if constexpr (CRP > CR) {
        double q = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) q += wr[w * 32 + CR];  // fixed order: identical in every warp
        part = tj * q;
      } else {
        if (act) part = pg * vj[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      }
      const uint32_t b0 = cla_smem_u32(&pbar[par]);
      const uint32_t p0 = cla_smem_u32(ploc + (size_t)par * sr + g);
      const uint32_t w0 = cla_smem_u32(wpart + par * 32 + rank);
      for (int dst = warp; dst < CS; dst += 8) {
        if (act) cla_st_async(cla_mapa(p0, (uint32_t)dst), pg, cla_mapa(b0, (uint32_t)dst));
        if (lane == 0) cla_st_async(cla_mapa(w0, (uint32_t)dst), part, cla_mapa(b0, (uint32_t)dst));
      }
    }
    TRI_T(3);
    cla_mbar_wait(&pbar[par], ph);  // p_j and the CTAs' parts of p.v_j
    if (rearm) cla_mbar_arm(&pbar[par], 8u * (uint32_t)(s - j - 3 + CS));
    {
      double k0 = 0.0, k1 = 0.0;
      for (int q = 0; q < CS; q += 2) {
        k0 += wpart[par * 32 + q];
        k1 += wpart[par * 32 + q + 1];
      }
      Kp = 0.5 * tj * (k0 + k1);
    }
    TRI_T(4);
  }
  if (prof && threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) prof[rank * 8 + k] = pt[k];
  if (prof && threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) prof[128 + rank * 4 + k] = po[k];
#undef TRI_T
#undef TRI_O
  // the last pending update (step s-3) on the trailing 2 x 2, then d, e of the last two columns
  if (s >= 3) {
    const int pl = (s - 3) & 1;
    const double* vp = vloc + (size_t)pl * sr;
    const double* pq = ploc + (size_t)pl * sr;
#pragma unroll
    for (int c = 0; c < CR; ++c) {
      const int g = (int)rank + CS * (cg + TCG * c);
      if (g >= s - 2 && g < s) {
        const double bg = vp[g], ag = pq[g] - 2.0 * Kp * bg;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const int r = rg + RG * k;
          if (r >= g && r < s) {
            const double x = a[k][c] - (vp[r] * ag + pq[r] * bg);
            if (r == g)
              d[g] = x;
            else
              e[g] = x;  // (s-1, s-2)
          }
        }
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < ncl * s; q += NT) {
    int lc = q / s, i = q - lc * s, g = (int)rank + CS * lc;
    if (g + 2 < s && i > g) Vh[IDX(i, g, ldv)] = refl[(size_t)lc * sr + i];
  }
  for (int lc = tid; lc < ncl; lc += NT) {
    int g = (int)rank + CS * lc;
    if (g + 2 < s) {
      d[g] = dl[lc];
      e[g] = el[lc];
      tau[g] = tl[lc];
    }
  }
  cla_cluster_sync();  // no CTA leaves while a push to it may be in flight
}

// Back-transformation Y <- Q Y, Q = H_0 H_1 ... H_{s-3} (apply H_{s-3} first): one warp per
// column (held in registers), reflectors staged through shared memory in panels of BT_PB
// (coalesced loads shared by the CTA's warps instead of per-warp L2 round trips).
constexpr int BT_PB = 16;
constexpr int BT_PER_LANE = 40;  // s <= 1280
template <int PL>
__global__ void __launch_bounds__(256) backtransform_panel_kernel(int s, int m, const double* __restrict__ Vh, int ldv,
                                                                  const double* __restrict__ tau,
                                                                  double* __restrict__ y, int ldy, int PB) {
  // two panel buffers (PB <= BT_PB reflectors x s each): panel k+1 streams in with cp.async while
  // panel k is applied
  extern __shared__ __align__(16) double pv[];
  __shared__ double ptau[2][BT_PB];
  const int lane = threadIdx.x & 31;
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool active = col < m;
  double* yc = y + (size_t)(active ? col : 0) * ldy;
  double r[PL];
#pragma unroll
  for (int q = 0; q < PL; ++q) {
    int k = lane + 32 * q;
    r[q] = (active && k < s) ? yc[k] : 0.0;
  }
  const int nref = s - 2;  // reflectors 0 .. s-3, applied from the last one down
  const int npan = cdiv(max(nref, 0), PB);
  auto issue = [&](int pnl, int buf) {
    const int hi = nref - 1 - pnl * PB, lo = max(0, hi - PB + 1);
    double* dst = pv + (size_t)buf * PB * s;
    for (int c = 0; c <= hi - lo; ++c) {
      const int j = lo + c;
      for (int i = threadIdx.x; i < s; i += blockDim.x)
        cp_async_8(dst + (size_t)c * s + i, Vh + IDX(i, j, ldv), (i > j) ? 8 : 0);  // zero-fill rows <= j
    }
    if (threadIdx.x <= hi - lo) ptau[buf][threadIdx.x] = __ldg(tau + lo + threadIdx.x);
    cp_async_commit();
  };
  if (npan > 0) issue(0, 0);
  for (int pnl = 0; pnl < npan; ++pnl) {
    const int buf = pnl & 1;
    if (pnl + 1 < npan) {
      issue(pnl + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int hi = nref - 1 - pnl * PB, lo = max(0, hi - PB + 1);
    if (active) {
      for (int j = hi; j >= lo; --j) {
        const double tj = ptau[buf][j - lo];
        if (tj == 0.0) continue;
        const double* v = pv + (size_t)buf * PB * s + (size_t)(j - lo) * s;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int q = 0; q < PL; ++q) {
          int k = lane + 32 * q;
          if (k < s) {
            if (q & 1)
              a1 = fma(v[k], r[q], a1);
            else
              a0 = fma(v[k], r[q], a0);
          }
        }
        double acc = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        acc *= tj;
#pragma unroll
        for (int q = 0; q < PL; ++q) {
          int k = lane + 32 * q;
          if (k < s) r[q] = fma(-acc, v[k], r[q]);
        }
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next issue
  }
  if (!active) return;
#pragma unroll
  for (int q = 0; q < PL; ++q) {
    int k = lane + 32 * q;
    if (k < s) yc[k] = r[q];
  }
}

// ------------------------------------------------------------------ helpers for the RR step
// Li = L^-1 (t x t lower, ldl -> ldi): one warp per column j of the inverse (x = L^-1 e_j held in
// registers, rows lane + 32 q), columns of L streamed through shared memory in panels of TI_KB
// shared by the CTA's 8 warps: x_k /= L_kk; x_{k+1:} -= x_k L_{k+1:,k}.
constexpr int TI_KB = 16;
template <int PL>
__global__ void __launch_bounds__(256) trinv_panel_kernel(int t, const double* __restrict__ L, int ldl,
                                                          double* __restrict__ Li, int ldi) {
  extern __shared__ __align__(16) double lp[];  // TI_KB x t
  __shared__ double dinv[TI_KB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int jbase = blockIdx.x * 8;
  const int j = jbase + w;
  double x[PL];
#pragma unroll
  for (int q = 0; q < PL; ++q) x[q] = (lane + 32 * q == j) ? 1.0 : 0.0;
  for (int k0 = jbase; k0 < t; k0 += TI_KB) {
    const int kb = min(TI_KB, t - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kb * t; e += blockDim.x) {
      const int c = e / t, i = e - c * t;
      lp[(size_t)c * t + i] = (i > k0 + c) ? __ldg(L + IDX(i, k0 + c, ldl)) : 0.0;
    }
    if (threadIdx.x < kb) dinv[threadIdx.x] = 1.0 / __ldg(L + IDX(k0 + threadIdx.x, k0 + threadIdx.x, ldl));
    __syncthreads();
    if (j >= t) continue;
    for (int c = 0; c < kb; ++c) {
      const int k = k0 + c;
      if (k < j) continue;
      const int kq = k >> 5, kl = k & 31;
      double xv = 0.0;
#pragma unroll
      for (int q = 0; q < PL; ++q)
        if (q == kq) xv = x[q];
      const double xk = __shfl_sync(0xffffffffu, xv, kl) * dinv[c];
#pragma unroll
      for (int q = 0; q < PL; ++q)
        if (q == kq && lane == kl) x[q] = xk;
      const double* lc = lp + (size_t)c * t;  // zero at rows <= k
#pragma unroll
      for (int q = 0; q < PL; ++q) {
        const int i = lane + 32 * q;
        if (i < t) x[q] = fma(-xk, lc[i], x[q]);
      }
    }
  }
  if (j >= t) return;
#pragma unroll
  for (int q = 0; q < PL; ++q) {
    const int i = lane + 32 * q;
    if (i < t) Li[IDX(i, j, ldi)] = x[q];
  }
}

// Blocked back-transformation with the compact WY form (LAPACK dlarft/dlarfb): the reflectors of
// panel p (columns lo..hi, hi - lo + 1 <= WY_PB) satisfy H_lo ... H_hi = I - V T V^T with T upper
// triangular. larft_kernel builds every panel's T in parallel (one CTA per panel); the apply kernel
// walks the panels from the last to the first, Y <- (I - V T V^T) Y: per panel and column, WY_PB
// independent dot products (one interleaved warp reduction) instead of WY_PB dependent ones.
constexpr int WY_PB = 16;
__global__ void __launch_bounds__(256) larft_kernel(int s, const double* __restrict__ Vh, int ldv,
                                                    const double* __restrict__ tau, double* __restrict__ Tb) {
  __shared__ double G[WY_PB][WY_PB + 1];
  __shared__ double T[WY_PB][WY_PB + 1];
  const int nref = s - 2;
  const int p = blockIdx.x;
  const int lo = p * WY_PB, kb = min(WY_PB, nref - lo);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // Gram of the panel columns (upper triangle incl. diagonal), v_c zero at rows <= lo + c
  for (int pr = warp; pr < kb * kb; pr += nw) {
    const int a = pr % kb, b = pr / kb;
    if (a > b) continue;
    const int j0 = lo + b;  // column b is nonzero from row j0 + 1
    double acc = 0.0;
    for (int i = j0 + 1 + lane; i < s; i += 32) acc = fma(__ldg(Vh + IDX(i, lo + a, ldv)), __ldg(Vh + IDX(i, j0, ldv)), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) G[a][b] = acc;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // T(0:i-1, i) = T(0:i-1, 0:i-1) (-tau_i G(0:i-1, i)), one lane per row
    const int r = lane;
    for (int i = 0; i < kb; ++i) {
      const double ti = __ldg(tau + lo + i);
      T[r < WY_PB ? r : 0][i] = 0.0;
      __syncwarp();
      // w_r <- sum_{c = r..i-1} T[r][c] (-tau_i G[c][i])
      double acc = 0.0;
      for (int c = r; c < i; ++c) acc = fma(T[r][c], -ti * G[c][i], acc);
      __syncwarp();
      if (r < i) T[r][i] = acc;
      if (r == i) T[r][i] = ti;
      __syncwarp();
    }
    for (int e = lane; e < WY_PB * WY_PB; e += 32) {
      const int a = e % WY_PB, b = e / WY_PB;
      Tb[(size_t)p * WY_PB * WY_PB + e] = (a < kb && b < kb && a <= b) ? T[a][b] : 0.0;
    }
  }
}

// CPB warps per CTA, one column each (CPB = 4: m = 130 columns -> 33 CTAs instead of 17 with 8):
// per panel the 16 dot products of a column are reduced across the warp by one transposed
// shuffle reduction (tri_xreduce) instead of 16 x 32 sequential shared-memory sums.
__host__ __device__ inline size_t bt_wy_smem_doubles(int PL, int CPB) {
  return (size_t)2 * WY_PB * 32 * PL + 2 * WY_PB * WY_PB + (size_t)CPB * 2 * WY_PB;
}
template <int PL, int CPB>
__global__ void __launch_bounds__(32 * CPB) backtransform_wy_kernel(int s, int m, const double* __restrict__ Vh, int ldv,
                                                                    const double* __restrict__ Tb,
                                                                    double* __restrict__ y, int ldy) {
  // two panel buffers (WY_PB x 32 PL each, rows >= s zero) + T, streamed with cp.async
  extern __shared__ __align__(16) double pv[];
  const int LDP = 32 * PL;
  double* Ts = pv + (size_t)2 * WY_PB * LDP;  // 2 x WY_PB x WY_PB
  double* wsm = Ts + 2 * WY_PB * WY_PB;       // per warp: w (WY_PB), z (WY_PB)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = blockIdx.x * CPB + warp;
  const bool active = col < m;
  double* yc = y + (size_t)(active ? col : 0) * ldy;
  double r[PL];
#pragma unroll
  for (int q = 0; q < PL; ++q) {
    const int k = lane + 32 * q;
    r[q] = (active && k < s) ? yc[k] : 0.0;
  }
  const int nref = s - 2;
  const int npan = cdiv(max(nref, 0), WY_PB);
  auto issue = [&](int pnl, int buf) {
    const int lo = pnl * WY_PB, kb = min(WY_PB, nref - lo);
    double* dst = pv + (size_t)buf * WY_PB * LDP;
    // row pairs: one 16-byte copy (or zero fill) when both rows agree and the source is aligned
    for (int e = threadIdx.x; e < WY_PB * (LDP / 2); e += blockDim.x) {
      const int c = e / (LDP / 2), i = 2 * (e - c * (LDP / 2)), j = lo + c;
      const bool ok0 = c < kb && i > j && i < s, ok1 = c < kb && i + 1 > j && i + 1 < s;
      const double* src = Vh + IDX(i, (c < kb ? j : 0), ldv);
      double* d0 = dst + (size_t)c * LDP + i;
      if (ok0 == ok1 && (!ok0 || ((reinterpret_cast<uintptr_t>(src) & 15) == 0))) {
        cp_async_16(d0, ok0 ? src : Vh, ok0 ? 16 : 0);
      } else {
        cp_async_8(d0, ok0 ? src : Vh, ok0 ? 8 : 0);
        cp_async_8(d0 + 1, ok1 ? src + 1 : Vh, ok1 ? 8 : 0);
      }
    }
    for (int e = threadIdx.x; e < WY_PB * WY_PB; e += blockDim.x)
      cp_async_8(Ts + (size_t)buf * WY_PB * WY_PB + e, Tb + (size_t)pnl * WY_PB * WY_PB + e, 8);
    cp_async_commit();
  };
  if (npan > 0) issue(npan - 1, (npan - 1) & 1);
  double* wz = wsm + (size_t)warp * 2 * WY_PB;
  for (int pnl = npan - 1; pnl >= 0; --pnl) {
    const int buf = pnl & 1;
    if (pnl > 0) {
      issue(pnl - 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const double* V = pv + (size_t)buf * WY_PB * LDP;
      const double* T = Ts + (size_t)buf * WY_PB * WY_PB;
      // lane partials of w_c = v_c . y for all c (16 independent chains), then one transposed
      // reduction: lane l ends with w_{c(l)} (lanes l, l ^ 1 agree)
      double a[WY_PB];
#pragma unroll
      for (int c = 0; c < WY_PB; ++c) a[c] = 0.0;
#pragma unroll
      for (int q = 0; q < PL; ++q) {
#pragma unroll
        for (int c = 0; c < WY_PB; ++c) a[c] = fma(V[(size_t)c * LDP + lane + 32 * q], r[q], a[c]);
      }
      const double wl = tri_xreduce<WY_PB>(a, lane);
      if ((lane & 1) == 0) wz[tri_xreduce_col<WY_PB>(lane)] = wl;
      __syncwarp();
      if (lane < WY_PB) {  // z = T w (T upper triangular, column-major)
        double acc = 0.0;
        for (int bcol = lane; bcol < WY_PB; ++bcol) acc = fma(T[lane + bcol * WY_PB], wz[bcol], acc);
        wz[WY_PB + lane] = acc;
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < WY_PB; ++c) {
        const double zc = wz[WY_PB + c];
#pragma unroll
        for (int q = 0; q < PL; ++q) r[q] = fma(-V[(size_t)c * LDP + lane + 32 * q], zc, r[q]);
      }
      __syncwarp();
    }
    __syncthreads();  // buffer `buf` is refilled by the next issue
  }
  if (!active) return;
#pragma unroll
  for (int q = 0; q < PL; ++q) {
    const int k = lane + 32 * q;
    if (k < s) yc[k] = r[q];
  }
}

// One column per 256-thread CTA (m ~ 100 CTAs on 148 SMs): the rows of the column are split over
// the CTA (thread t owns rows t + 256 q, q < PLW), so per panel every warp does PLW x 16 FMAs for
// the dot products and as many for the update instead of a whole column's worth (the one-warp-per-
// column kernel above is bound by its own instruction stream: ~3 cycles per issued instruction).
// Per panel: lane partials of w = V^T y, a transposed warp reduction, the 8 warp sums added in
// fixed order while z = T w is formed by 256 threads (one product T(r, b) w_b each, reduced over
// the 16 lanes of b), then y -= V z.
__host__ __device__ inline size_t bt_col_smem_doubles(int s) {
  return (size_t)2 * WY_PB * ((s + 2) & ~1) + 2 * WY_PB * WY_PB + 8 * WY_PB + WY_PB;
}
template <int PLW>
__global__ void __launch_bounds__(256) backtransform_wy_col_kernel(int s, int m, const double* __restrict__ Vh,
                                                                   int ldv, const double* __restrict__ Tb,
                                                                   double* __restrict__ y, int ldy) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  extern __shared__ __align__(16) double pv[];
  const int LDP = (s + 2) & ~1;                // panel column pitch: row s exists and is zero-filled
  double* Ts = pv + (size_t)2 * WY_PB * LDP;   // 2 x WY_PB x WY_PB
  double* wp = Ts + 2 * WY_PB * WY_PB;         // 8 warps x WY_PB partial dot products
  double* zs = wp + 8 * WY_PB;                 // z = T w
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double* yc = y + (size_t)blockIdx.x * ldy;
  double r[PLW];
  int kk[PLW];  // panel row of y row k; rows >= s read the zero row s (their r stays 0)
#pragma unroll
  for (int q = 0; q < PLW; ++q) {
    const int k = t + 256 * q;
    r[q] = k < s ? yc[k] : 0.0;
    kk[q] = min(k, s);
  }
  const int nref = s - 2;
  const int npan = cdiv(max(nref, 0), WY_PB);
  auto issue = [&](int pnl, int buf) {
    const int lo = pnl * WY_PB, kb = min(WY_PB, nref - lo);
    double* dst = pv + (size_t)buf * WY_PB * LDP;
    for (int e = t; e < WY_PB * (LDP / 2); e += 256) {
      const int c = e / (LDP / 2), i = 2 * (e - c * (LDP / 2)), j = lo + c;
      const bool ok0 = c < kb && i > j && i < s, ok1 = c < kb && i + 1 > j && i + 1 < s;
      const double* src = Vh + IDX(i, (c < kb ? j : 0), ldv);
      double* d0 = dst + (size_t)c * LDP + i;
      if (ok0 == ok1 && (!ok0 || ((reinterpret_cast<uintptr_t>(src) & 15) == 0))) {
        cp_async_16(d0, ok0 ? src : Vh, ok0 ? 16 : 0);
      } else {
        cp_async_8(d0, ok0 ? src : Vh, ok0 ? 8 : 0);
        cp_async_8(d0 + 1, ok1 ? src + 1 : Vh, ok1 ? 8 : 0);
      }
    }
    for (int e = t; e < WY_PB * WY_PB; e += 256)
      cp_async_8(Ts + (size_t)buf * WY_PB * WY_PB + e, Tb + (size_t)pnl * WY_PB * WY_PB + e, 8);
    cp_async_commit();
  };
  if (npan > 0) issue(npan - 1, (npan - 1) & 1);
  for (int pnl = npan - 1; pnl >= 0; --pnl) {
    const int buf = pnl & 1;
    if (pnl > 0) {
      issue(pnl - 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* V = pv + (size_t)buf * WY_PB * LDP;
    const double* T = Ts + (size_t)buf * WY_PB * WY_PB;
    {
      double a[WY_PB];
#pragma unroll
      for (int c = 0; c < WY_PB; ++c) a[c] = 0.0;
#pragma unroll
      for (int q = 0; q < PLW; ++q) {
#pragma unroll
        for (int c = 0; c < WY_PB; ++c) a[c] = fma(V[(size_t)c * LDP + kk[q]], r[q], a[c]);
      }
      const double wl = tri_xreduce<WY_PB>(a, lane);
      if ((lane & 1) == 0) wp[warp * WY_PB + tri_xreduce_col<WY_PB>(lane)] = wl;
    }
    __syncthreads();
    {
      const int rr = t >> 4, b = t & 15;
      double wb = 0.0;
#pragma unroll
      for (int wi = 0; wi < 8; ++wi) wb += wp[wi * WY_PB + b];
      double pr = (b >= rr) ? T[rr + b * WY_PB] * wb : 0.0;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) pr += __shfl_xor_sync(0xffffffffu, pr, o);
      if (b == 0) zs[rr] = pr;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < WY_PB; ++c) {
      const double zc = zs[c];
#pragma unroll
      for (int q = 0; q < PLW; ++q) r[q] = fma(-V[(size_t)c * LDP + kk[q]], zc, r[q]);
    }
    __syncthreads();  // buffer `buf` is refilled by the next issue
  }
#pragma unroll
  for (int q = 0; q < PLW; ++q) {
    const int k = t + 256 * q;
    if (k < s) yc[k] = r[q];
  }
}

// Newton-Schulz step towards the polar factor: Z = 1.5 I - 0.5 M for M = Y^T Y (m x m), and
// dev = max |M - I| accumulated into *dev (as a non-negative double's bit pattern, atomicMax).
__global__ void ns_coeff_kernel(int m, const double* __restrict__ M, int ldm, double* __restrict__ Z, int ldz,
                                unsigned long long* __restrict__ dev) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  double mx = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)m * m;
       q += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(q % m), k = (int)(q / m);
    double mik = M[IDX(i, k, ldm)], id = (i == k) ? 1.0 : 0.0;
    Z[IDX(i, k, ldz)] = 1.5 * id - 0.5 * mik;
    mx = fmax(mx, fabs(mik - id));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(dev, (unsigned long long)__double_as_longlong(mx));
}

}  // namespace psd
