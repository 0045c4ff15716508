// sbr.cuh -- two-stage tridiagonalisation of the Rayleigh-Ritz matrix (a7, the eigensolve of Alg. 2,
// PAPER.md:337, 404-405): dense -> band (stage 1, a thread-block cluster) -> tridiagonal (stage 2,
// bulge chasing in one CTA), and the back-transformation of the tridiagonal eigenvectors through both.
//
// Why two stages. The one-stage Householder reduction (cluster_la.cuh: tridiag_reg_kernel) is bound by
// two cluster-wide hops per column (the reflector broadcast, the matrix-vector all-gather): ~4k cycles
// per column whatever the arithmetic. Stage 1 reduces a panel of SB columns per step with two hops (the
// panel all-gather, the all-gather of Y = A V T), the panel's QR redundantly in every CTA's shared
// memory; stage 2 chases the bulges of the band inside one CTA (no cluster hop at all), several sweeps
// in flight on different warps.
//
// Stage 1 (sb1_kernel, CS CTAs of one cluster, column g in CTA g % CS at local column g / CS, full
// column storage): for panel p (columns j0 = p SB .. j0 + SB - 1, rows r0 = j0 + SB .. s - 1 below the
// band) Q_p = I - V T V^T from the Householder QR of A[r0:, j0:j0+SB] (LAPACK dgeqr2 + dlarft forward
// column-wise), then the two-sided update of the trailing matrix in the dsytrd/dsyr2k form
//     A22 <- A22 - V Y^T - Y V^T + V M V^T,   Y = A22 V T,   M = T^T V^T Y  (= T^T V^T A22 V T),
// rows of Y computed by the owners of the matching columns (A22 symmetric) and all-gathered.
// Output: the lower band (bandwidth SB) in SB_LDW-wide storage Bg[c * SB_LDW + (r - c)] (zeros beyond
// distance SB), the panel reflectors V_p (column j0 + i of Vq holds reflector i: 1 at row r0 + i) and
// T_p (Tq + p SB^2, column-major).
//
// Stage 2 (sb2_kernel, one CTA): sweep j annihilates column j below the subdiagonal with a Householder
// reflector of rows [j+1, j+1+SB) and chases the bulge it creates down the band: task (j, k) acts on rows
// [a, a+L), a = j + 1 + k SB (left block: columns [a-SB+1, a) of those rows; the symmetric diagonal block;
// right block: rows [a+L, a+L+SB) of columns [a, a+L)), and the next task annihilates the first column of
// that right block (only the first column of each bulge; the rest is swept by later sweeps). Entries stay
// within distance 2 SB - 1 of the diagonal (SB_LDW = 2 SB storage). Task (j, k) may start once task
// (j-1, k+2) is complete (the footprints of (j, k) and (j-1, k+2) meet in one row; (j-1, k+3) is
// disjoint): every sweep runs on its own warp, ordered by per-sweep progress counters in shared memory.
// Reflector (j, k) is stored at Vr + 17 (off(j) + k) (v_0..v_15 with v_0 = 1, tau at 16).
//
// Back-transformation (sbr_bt_kernel): eigenvectors of A = Q1 Q2 y, Q2 = prod over sweeps (j ascending;
// the reflectors of one sweep act on disjoint rows, and every reflector of a later sweep that overlaps an
// earlier one was applied after it), Q1 = Q_0 Q_1 ... Q_{P-1}: y <- Q2 y sweep by sweep from the last,
// then y <- Q_p y from the last panel.
#pragma once
#include "cluster_la.cuh"

namespace psd {

constexpr int SB = 16;          // band width of stage 1
constexpr int SB_LDW = 2 * SB;  // band storage width (distances 0 .. 2 SB - 1): stride 31 across columns
constexpr int SB1_NT = 256;
constexpr int SB2_NW = 16;      // stage-2 warps (sweeps in flight)
constexpr int SB_MAX = 768;     // SB2_NW warps keep every sweep on a distinct warp up to 3 SB SB2_NW

__host__ __device__ inline int sb_npanels(int s) { return s - 1 - SB > 0 ? cdiv(s - 1 - SB, SB) : 0; }
__host__ __device__ inline int sb_nsweeps(int s) { return s > 2 ? s - 2 : 0; }
__host__ __device__ inline int sb_ktasks(int s, int j) { return cdiv(s - 1 - j, SB); }
// sum_{u = 0}^{N - 1} floor(u / SB)
__host__ __device__ inline long long sb_fsum(long long N) {
  const long long q = N / SB, r = N % SB;
  return SB * q * (q - 1) / 2 + q * r;
}
// reflector offset of sweep j: sum_{j' < j} K_{j'}, K_{j'} = floor((s - 2 - j') / SB) + 1
__host__ __device__ inline long long sb_refl_off(int s, int j) {
  return (long long)j + sb_fsum(s - 1) - sb_fsum(s - 1 - j);
}
__host__ __device__ inline size_t sb_refl_doubles(int s) { return 17 * (size_t)(sb_refl_off(s, sb_nsweeps(s)) + 1); }

__host__ __device__ inline size_t sb1_smem_doubles(int s, int CS) {
  const size_t sr = (size_t)((s + 1) & ~1), ncl = (size_t)cdiv(s, CS);
  return ncl * sr + 2 * (size_t)SB * sr + (size_t)CS * ncl * SB + 2 * SB + 3 * SB * SB + 8 * 2 * SB + 64;
}

__device__ __forceinline__ void sb_bulk_s2c(uint32_t dst_cluster, const double* src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(cla_smem_u32(src)), "r"(bytes), "r"(bar_cluster)
               : "memory");
}

// ------------------------------------------------------------------ stage 1: dense -> band (cluster)
__global__ void __launch_bounds__(SB1_NT, 1) sb1_kernel(int s, const double* __restrict__ A, int lda,
                                                        double* __restrict__ Bg, double* __restrict__ Vq, int ldq,
                                                        double* __restrict__ Tq) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t pbar[2], ybar;
  const int CS = (int)gridDim.x;
  const int rank = (int)cla_rank();
  const int ncl = cdiv(s, CS), sr = (s + 1) & ~1;
  double* Aloc = sm;                               // ncl x sr: own columns (full)
  double* PB = Aloc + (size_t)ncl * sr;            // 2 x SB x sr: the panel (parity), absolute rows
  double* Yf = PB + 2 * (size_t)SB * sr;           // CS x ncl x SB: rows of Y by (owner, local column)
  double* tau = Yf + (size_t)CS * ncl * SB;        // SB
  double* Rd = tau + SB;                           // SB: R diagonal (beta)
  double* T = Rd + SB;                             // SB x SB, T[k + l SB]
  double* Nm = T + SB * SB;                        // SB x SB: z = V^T V (strict upper), then N = V^T Y
  double* Mm = Nm + SB * SB;                       // SB x SB: M = T^T N
  double* Zw = Mm + SB * SB;                       // 8 warps x (Z_c | V_c)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int npan = sb_npanels(s);

  for (size_t q = tid; q < (size_t)ncl * sr; q += SB1_NT) {
    const int lc = (int)(q / sr), r = (int)(q - (size_t)lc * sr), g = rank + CS * lc;
    Aloc[q] = (g < s && r < s) ? 0.5 * (A[IDX(r, g, lda)] + A[IDX(g, r, lda)]) : 0.0;
  }
  // band storage of the own columns: zero (entries are written as they become final)
  for (int q = tid; q < ncl * SB_LDW; q += SB1_NT) {
    const int lc = q / SB_LDW, g = rank + CS * lc;
    if (g < s) Bg[(size_t)g * SB_LDW + (q - lc * SB_LDW)] = 0.0;
  }
  // trailing own columns of panel p (rows of Y this CTA produces): local columns [lo, hi)
  auto trail = [&](int r0, int& lo, int& hi) {
    lo = r0 <= rank ? 0 : cdiv(r0 - rank, CS);
    hi = s <= rank ? 0 : cdiv(s - rank, CS);
    if (hi < lo) hi = lo;
  };
  auto ybytes = [&](int p) -> uint32_t {  // Y bytes this CTA receives for panel p (all rows but its own)
    const int r0 = (p + 1) * SB;
    int lo, hi;
    trail(r0, lo, hi);
    return 8u * SB * (uint32_t)((s - r0) - (hi - lo));
  };
  auto pbytes = [&](int p) -> uint32_t { return 8u * SB * (uint32_t)(sr - (p + 1) * SB); };
  __syncthreads();
  if (tid == 0) {
    cla_mbar_init(&pbar[0], 1);
    cla_mbar_init(&pbar[1], 1);
    cla_mbar_init(&ybar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (npan > 0) {
      cla_mbar_arm(&pbar[0], pbytes(0));
      cla_mbar_arm(&ybar, ybytes(0));
    }
    if (npan > 1) cla_mbar_arm(&pbar[1], pbytes(1));
  }
  __syncthreads();
  cla_cluster_sync();  // every CTA's barriers are initialised and armed before the first push

  // push the own columns of panel q (rows [r0, sr)) into every CTA's PB[q & 1]
  auto push_panel = [&](int q) {
    const int j0 = q * SB, r0 = j0 + SB;
    const int nown = SB / CS > 0 ? SB / CS : 1;  // own columns per panel (CS divides SB or SB divides CS)
    if (tid < nown * CS) {
      const int which = tid / CS, dst = tid - which * CS;
      // the which-th own column in [j0, j0 + SB)
      const int g0 = j0 + ((rank - j0) % CS + CS) % CS;
      const int g = g0 + which * CS;
      if (g < j0 + SB) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const double* src = Aloc + (size_t)(g / CS) * sr + r0;
        double* dstp = PB + (size_t)(q & 1) * SB * sr + (size_t)(g - j0) * sr + r0;
        sb_bulk_s2c(cla_mapa(cla_smem_u32(dstp), (uint32_t)dst), src, 8u * (uint32_t)(sr - r0),
                    cla_mapa(cla_smem_u32(&pbar[q & 1]), (uint32_t)dst));
      }
    }
  };
  if (npan > 0) push_panel(0);

  for (int p = 0; p < npan; ++p) {
    const int par = p & 1, j0 = p * SB, r0 = j0 + SB;
    double* P = PB + (size_t)par * SB * sr;
    cla_mbar_wait(&pbar[par], (uint32_t)(p >> 1) & 1u);
    if (tid == 0 && p + 2 < npan) cla_mbar_arm(&pbar[par], pbytes(p + 2));
    // band: the diagonal block of the panel's own columns (final)
    for (int q = tid; q < SB * SB; q += SB1_NT) {
      const int i = q / SB, rr = q - i * SB;  // column j0 + i, row j0 + rr
      const int g = j0 + i, r = j0 + rr;
      if (g % CS == rank && r >= g) Bg[(size_t)g * SB_LDW + (r - g)] = Aloc[(size_t)(g / CS) * sr + r];
    }
    // ---- Householder QR of the panel P[:, r0:s] (every CTA, redundantly). Column i on warp i % 8.
    for (int i = 0; i < SB; ++i) {
      const int ri = r0 + i;
      if (warp == (i & 7)) {
        double* col = P + (size_t)i * sr;
        double sg = 0.0;
        for (int r = ri + 1 + lane; r < s; r += 32) sg = fma(col[r], col[r], sg);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
        const double alpha = ri < s ? col[ri] : 0.0;
        double tj = 0.0, beta = alpha, scale = 0.0;
        if (sg != 0.0) {
          const double mu = sqrt(fma(alpha, alpha, sg));
          beta = alpha <= 0.0 ? mu : -mu;
          tj = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        for (int r = ri + 1 + lane; r < s; r += 32) col[r] *= scale;
        if (lane == 0) {
          tau[i] = tj;
          Rd[i] = beta;
        }
      }
      __syncthreads();
      const double tj = tau[i];
      if (tj != 0.0) {
        const double* v = P + (size_t)i * sr;
        for (int k = warp; k < SB; k += 8) {
          if (k <= i) continue;
          double* ck = P + (size_t)k * sr;
          double w = 0.0;
          for (int r = ri + 1 + lane; r < s; r += 32) w = fma(v[r], ck[r], w);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
          w += ck[ri];
          const double f = tj * w;
          __syncwarp();
          if (lane == 0) ck[ri] -= f;
          for (int r = ri + 1 + lane; r < s; r += 32) ck[r] = fma(-f, v[r], ck[r]);
        }
      }
    }
    __syncthreads();
    // band: R (rows r0 .. r0 + i of column j0 + i); Q1 output (CTA 0): V_p, then V canonical in P
    // (1 on the diagonal, 0 above) so that V_k(r) = P[k][r] for every r >= r0
    for (int q = tid; q < SB * SB; q += SB1_NT) {
      const int i = q / SB, l = q - i * SB, g = j0 + i, r = r0 + l;
      if (g % CS == rank && l <= i && r < s)
        Bg[(size_t)g * SB_LDW + (r - g)] = (l == i) ? Rd[i] : P[(size_t)i * sr + r];
    }
    __syncthreads();
    for (int q = tid; q < SB * SB; q += SB1_NT) {
      const int i = q / SB, l = q - i * SB, r = r0 + l;
      if (l <= i && r < s) P[(size_t)i * sr + r] = (l == i) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (rank == 0) {
      for (int i = 0; i < SB; ++i)
        for (int r = r0 + tid; r < s; r += SB1_NT) Vq[IDX(r, j0 + i, ldq)] = P[(size_t)i * sr + r];
    }
    // ---- T (dlarft, forward, column-wise): z = V^T V (pairs k < i over two threads), then the recurrence
    {
      const int pair = tid >> 1, half = tid & 1;
      const bool ok = pair < SB * (SB - 1) / 2;
      int i = 1, base = 0;
      while (ok && base + i <= pair) {
        base += i;
        ++i;
      }
      const int k = ok ? pair - base : 0;  // k < i
      double z = 0.0;
      if (ok) {
        const double* vk = P + (size_t)k * sr;
        const double* vi = P + (size_t)i * sr;
        for (int r = r0 + i + half; r < s; r += 2) z = fma(vk[r], vi[r], z);
      }
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      if (ok && half == 0) Nm[k + i * SB] = z;
    }
    __syncthreads();
    if (warp == 0) {
      // T[k][i] = -tau_i sum_{l = k}^{i-1} T[k][l] z[l][i] (lane k < i), one column per step
      if (lane < SB) {
        for (int q = 0; q < SB; ++q) T[lane + q * SB] = 0.0;
        T[lane + lane * SB] = tau[lane];
      }
      __syncwarp();
      for (int i = 1; i < SB; ++i) {
        double t = 0.0;
        if (lane < i) {
          for (int l = lane; l < i; ++l) t = fma(T[lane + l * SB], Nm[l + i * SB], t);
          t *= -tau[i];
        }
        __syncwarp();
        if (lane < i) T[lane + i * SB] = t;
        __syncwarp();
      }
    }
    // before the Y rows are rewritten: this CTA's previous Y pushes have finished reading Yf
    if (tid < CS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
    // ---- Y rows of the own trailing columns: u = A[r0:, g]^T V, Y[g, :] = u T
    int lo, hi;
    trail(r0, lo, hi);
    for (int lc = lo + warp; lc < hi; lc += 8) {
      const double* ac = Aloc + (size_t)lc * sr;
      double acc[SB];
#pragma unroll
      for (int k = 0; k < SB; ++k) acc[k] = 0.0;
      for (int r = r0 + lane; r < s; r += 32) {
        const double x = ac[r];
#pragma unroll
        for (int k = 0; k < SB; ++k) acc[k] = fma(x, P[(size_t)k * sr + r], acc[k]);
      }
      const double u = tri_xreduce<SB>(acc, lane);  // lane holds u[c(lane)]
      const int cu = tri_xreduce_col<SB>(lane);
      // Y[l] = sum_{k <= l} u[k] T[k][l]; lane l < SB gathers u[k] from a lane holding it
      double y = 0.0;
#pragma unroll
      for (int k = 0; k < SB; ++k) {
        // the lane with column k: tri_xreduce_col is a bit-reversal-like map; find it by search-free
        // broadcast: every lane holding column k has the same value
        const int src = __ffs(__ballot_sync(0xffffffffu, cu == k)) - 1;
        const double uk = __shfl_sync(0xffffffffu, u, src);
        if (lane < SB && k <= lane) y = fma(uk, T[k + lane * SB], y);
      }
      if (lane < SB) Yf[((size_t)rank * ncl + lc) * SB + lane] = y;
    }
    __syncthreads();
    if (tid < CS && tid != rank && hi > lo) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const double* src = Yf + ((size_t)rank * ncl + lo) * SB;
      sb_bulk_s2c(cla_mapa(cla_smem_u32(src), (uint32_t)tid), src, 8u * SB * (uint32_t)(hi - lo),
                  cla_mapa(cla_smem_u32(&ybar), (uint32_t)tid));
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (rank == 0)
      for (int q = tid; q < SB * SB; q += SB1_NT) Tq[(size_t)p * SB * SB + q] = T[q];
    cla_mbar_wait(&ybar, (uint32_t)p & 1u);
    if (tid == 0 && p + 1 < npan) cla_mbar_arm(&ybar, ybytes(p + 1));
    // ---- N = V^T Y (thread (k, l)), M = T^T N
    auto yrow = [&](int r) -> const double* { return Yf + ((size_t)(r % CS) * ncl + r / CS) * SB; };
    {
      const int k = tid >> 4, l = tid & 15;
      const double* vk = P + (size_t)k * sr;
      double n0 = 0.0, n1 = 0.0;
      int r = r0 + k;
      for (; r + 1 < s; r += 2) {
        n0 = fma(vk[r], yrow(r)[l], n0);
        n1 = fma(vk[r + 1], yrow(r + 1)[l], n1);
      }
      if (r < s) n0 = fma(vk[r], yrow(r)[l], n0);
      Nm[k + l * SB] = n0 + n1;
    }
    __syncthreads();
    {
      const int k = tid >> 4, l = tid & 15;
      double m = 0.0;
      for (int i = 0; i <= k; ++i) m = fma(T[i + k * SB], Nm[i + l * SB], m);
      Mm[k + l * SB] = m;
    }
    __syncthreads();
    // ---- update of the own trailing columns: A[r, g] -= sum_k V_k(r) Z_g[k] + Y[r][k] V_k(g),
    // Z_g = Y[g, :] - M V(g, :)^T
    for (int lc = lo + warp; lc < hi; lc += 8) {
      const int g = rank + CS * lc;
      double* zw = Zw + warp * 2 * SB;
      if (lane < SB) {
        const double* yg = Yf + ((size_t)rank * ncl + lc) * SB;
        double z = yg[lane];
#pragma unroll
        for (int l = 0; l < SB; ++l) z = fma(-Mm[lane + l * SB], P[(size_t)l * sr + g], z);
        zw[lane] = z;
        zw[SB + lane] = P[(size_t)lane * sr + g];
      }
      __syncwarp();
      double* ac = Aloc + (size_t)lc * sr;
      for (int r = r0 + lane; r < s; r += 32) {
        const double* yr = yrow(r);
        double a = ac[r];
#pragma unroll
        for (int k = 0; k < SB; ++k) a = fma(-P[(size_t)k * sr + r], zw[k], fma(-yr[k], zw[SB + k], a));
        ac[r] = a;
      }
      __syncwarp();
    }
    __syncthreads();
    if (p + 1 < npan) push_panel(p + 1);
  }
  // the trailing block (columns from npan SB on) is final: its band entries
  {
    const int c0 = npan * SB;
    for (int lc = tid; lc < ncl; lc += SB1_NT) {
      const int g = rank + CS * lc;
      if (g >= c0 && g < s)
        for (int d = 0; d <= SB && g + d < s; ++d) Bg[(size_t)g * SB_LDW + d] = Aloc[(size_t)lc * sr + g + d];
    }
  }
  if (tid < CS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncthreads();
  cla_cluster_sync();  // no CTA leaves while a push to it may be in flight
}

// ------------------------------------------------------------------ stage 2: band -> tridiagonal (one CTA)
// Wb[c * SB_LDW + (r - c)] holds A[r, c] for 0 <= r - c < SB_LDW (lower triangle; entries beyond the
// current bulge are zero).
__device__ __forceinline__ double& sb_at(double* Wb, int r, int c) { return Wb[c * SB_LDW + (r - c)]; }

__global__ void __launch_bounds__(SB2_NW * 32, 1) sb2_kernel(int s, const double* __restrict__ Bg, double* __restrict__ d,
                                                            double* __restrict__ e, double* __restrict__ Vr) {
  extern __shared__ __align__(16) double sm2[];
  double* Wb = sm2;                                        // s x SB_LDW
  double* vb = Wb + (size_t)s * SB_LDW;                    // SB2_NW x SB: the warps' reflectors
  volatile int* prog = (volatile int*)(vb + SB2_NW * SB);  // s: completed tasks per sweep
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nsw = sb_nsweeps(s);
  for (int q = tid; q < s * SB_LDW; q += SB2_NW * 32) Wb[q] = Bg[q];
  for (int q = tid; q < s; q += SB2_NW * 32) prog[q] = 0;
  __syncthreads();
  const int i = lane & 15, h = lane >> 4;
  double* v = vb + warp * SB;
  for (int j = warp; j < nsw; j += SB2_NW) {
    const int K = sb_ktasks(s, j);
    const long long roff = sb_refl_off(s, j);
    for (int k = 0; k < K; ++k) {
      // (j, k) after (j - 1, k + 2)
      if (j > 0) {
        const int need = min(k + 3, sb_ktasks(s, j - 1));
        if (lane == 0)
          while (prog[j - 1] < need) __nanosleep(32);
        __syncwarp();
        __threadfence_block();
      }
      const int a = j + 1 + k * SB, L = min(SB, s - a);
      const int c0 = k == 0 ? j : a - SB;  // the column annihilated in rows [a, a + L)
      const double x = i < L ? sb_at(Wb, a + i, c0) : 0.0;
      double sg = (i >= 1) ? x * x : 0.0;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
      const double alpha = __shfl_sync(0xffffffffu, x, 0);
      double tj = 0.0, beta = alpha, scale = 0.0;
      if (sg != 0.0) {
        const double mu = sqrt(fma(alpha, alpha, sg));
        beta = alpha <= 0.0 ? mu : -mu;
        tj = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      const double vi = i == 0 ? 1.0 : (i < L ? x * scale : 0.0);
      double* rf = Vr + 17 * (roff + k);
      if (h == 0) rf[i] = vi;
      if (lane == 0) rf[16] = tj;
      if (tj != 0.0) {
        if (h == 0) v[i] = vi;
        __syncwarp();
        if (h == 0 && i < L) sb_at(Wb, a + i, c0) = i == 0 ? beta : 0.0;
        // left block: rows [a, a + L) x columns [c0 + 1, a) (k >= 1); lane (column c0 + 1 + i, rows 8h..)
        if (k > 0) {
          const bool lc_ok = i < SB - 1;
          const int c = c0 + 1 + (lc_ok ? i : 0);
          double w = 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int l = 8 * h + q;
            if (lc_ok && l < L) w = fma(v[l], sb_at(Wb, a + l, c), w);
          }
          w += __shfl_xor_sync(0xffffffffu, w, 16);
          const double f = tj * w;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int l = 8 * h + q;
            if (lc_ok && l < L) sb_at(Wb, a + l, c) = fma(-f, v[l], sb_at(Wb, a + l, c));
          }
        }
        // diagonal block D = A[a:a+L, a:a+L]: p = D v, w = tau p, K = tau/2 w.v, q = w - K v,
        // D -= v q^T + q v^T
        double pi = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int l = 8 * h + q;
          if (i < L && l < L) pi = fma(i >= l ? sb_at(Wb, a + i, a + l) : sb_at(Wb, a + l, a + i), v[l], pi);
        }
        pi += __shfl_xor_sync(0xffffffffu, pi, 16);
        const double wi = tj * pi;
        double kk = (i < L) ? wi * v[i] : 0.0;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) kk += __shfl_xor_sync(0xffffffffu, kk, o);
        const double qi = fma(-0.5 * tj * kk, v[i], wi);
        // right block rows [a + L, a + L + Lr) x columns [a, a + L): y = R v (lane row i, columns 8h..)
        const int Lr = min(SB, s - a - L);
        double y = 0.0;
        if (i < Lr) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int l = 8 * h + q;
            if (l < L) y = fma(sb_at(Wb, a + L + i, a + l), v[l], y);
          }
        }
        y += __shfl_xor_sync(0xffffffffu, y, 16);
        __syncwarp();
        // D update (lane row i, columns 8h.. <= i) and R update
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int l = 8 * h + q;
          const double ql = __shfl_sync(0xffffffffu, qi, l);
          if (i < L && l <= i) {
            double& dd = sb_at(Wb, a + i, a + l);
            dd = fma(-v[i], ql, fma(-qi, v[l], dd));
          }
        }
        if (i < Lr) {
          const double f = tj * y;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int l = 8 * h + q;
            if (l < L) {
              double& rr = sb_at(Wb, a + L + i, a + l);
              rr = fma(-f, v[l], rr);
            }
          }
        }
      }
      __syncwarp();
      __threadfence_block();
      if (lane == 0) prog[j] = k + 1;
    }
  }
  __syncthreads();
  for (int c = tid; c < s; c += SB2_NW * 32) {
    d[c] = Wb[c * SB_LDW];
    if (c + 1 < s) e[c] = Wb[c * SB_LDW + 1];
  }
}

// ------------------------------------------------------------------ back-transformation y <- Q1 Q2 y
// One CTA per eigenvector column (held in shared memory). Q2: sweeps from the last; the reflectors of a
// sweep act on disjoint rows (a group of 16 threads each). Q1: panels from the last,
// y[r0:] -= V (T (V^T y[r0:])).
constexpr int SBT_NT = 512;
__global__ void __launch_bounds__(SBT_NT) sbr_bt_kernel(int s, int m, const double* __restrict__ Vr,
                                                        const double* __restrict__ Vq, int ldq,
                                                        const double* __restrict__ Tq, double* __restrict__ Y,
                                                        int ldy) {
  extern __shared__ __align__(16) double sy[];  // s (the column), then 2 SB scratch
  const int tid = threadIdx.x, col = blockIdx.x;
  double* ys = sy;
  double* wz = sy + s;
  for (int r = tid; r < s; r += SBT_NT) ys[r] = Y[IDX(r, col, ldy)];
  __syncthreads();
  // Q2: groups of 16 threads, one reflector each (warp-uniform trip counts: both groups of a warp
  // iterate together, an idle one with tau = 0)
  const int grp = tid >> 4, gl = tid & 15, ngrp = SBT_NT / 16;
  for (int j = sb_nsweeps(s) - 1; j >= 0; --j) {
    const int K = sb_ktasks(s, j);
    const long long roff = sb_refl_off(s, j);
    for (int k0 = 0; k0 < K; k0 += ngrp) {
      const int k = k0 + grp;
      const bool ok = k < K;
      const int a = j + 1 + k * SB, L = ok ? min(SB, s - a) : 0;
      const double* rf = Vr + 17 * (roff + (ok ? k : 0));
      const double tj = ok ? rf[16] : 0.0;
      const double vl = gl < L ? rf[gl] : 0.0;
      const double yl = gl < L ? ys[a + gl] : 0.0;
      double w = vl * yl;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      if (gl < L && tj != 0.0) ys[a + gl] = fma(-tj * w, vl, yl);
    }
    __syncthreads();
  }
  // Q1: panels from the last; u = V^T y[r0:] (group k), z = T u, y[r0:] -= V z
  const int npan = sb_npanels(s);
  for (int p = npan - 1; p >= 0; --p) {
    const int r0 = (p + 1) * SB;
    const double* Tp = Tq + (size_t)p * SB * SB;
    if (grp < SB) {
      const int k = grp;
      const double* vk = Vq + IDX(0, r0 - SB + k, ldq);
      double u = 0.0;
      for (int r = r0 + k + gl; r < s; r += 16) u = fma(vk[r], ys[r], u);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
      if (gl == 0) wz[k] = u;
    }
    __syncthreads();
    if (tid < SB) {
      double z = 0.0;
      for (int l = tid; l < SB; ++l) z = fma(Tp[tid + l * SB], wz[l], z);
      wz[SB + tid] = z;
    }
    __syncthreads();
    for (int r = r0 + tid; r < s; r += SBT_NT) {
      double acc = ys[r];
      const int kmax = min(SB - 1, r - r0);
      for (int k = 0; k <= kmax; ++k) acc = fma(-Vq[IDX(r, r0 - SB + k, ldq)], wz[SB + k], acc);
      ys[r] = acc;
    }
    __syncthreads();
  }
  for (int r = tid; r < s; r += SBT_NT) Y[IDX(r, col, ldy)] = ys[r];
}

}  // namespace psd
