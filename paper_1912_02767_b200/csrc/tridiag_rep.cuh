// tridiag_rep.cuh -- Householder tridiagonalisation of the Rayleigh-Ritz matrix (a7, PAPER.md:337,
// 404-405) on a 16-CTA cluster with ONE cluster hop per column.
//
// tridiag_reg_kernel (cluster_la.cuh) needs two hops per column: the owner of column j forms v_j and
// broadcasts it, then the p = A v_j all-gather. Here every CTA holds a replica of column j, pushed by its
// owner one step ahead (during step j - 1, right after the owner has applied the step-(j-2) update to it
// in registers), so after the step-(j-1) all-gather every CTA applies the last pending rank-2 update to
// its replica and forms v_j, tau_j itself -- identical arithmetic in every CTA, so identical bits -- and
// the only hop left on the critical path is the p all-gather. The replica push rides in the shadow of
// the step's matrix-vector product and its all-gather.
//
// Layout and step structure otherwise as tridiag_reg_kernel: thread t holds rows t % 64 + 64 k (k < KR)
// of its own local columns t / 64 + 4 c (c < CR) in registers; column g lives in CTA g % CS. Step j
// (parity par = j & 1):
//   R  wait for the replica of column j (colr[j & 1], mbarrier rbar[j & 1]; column 0 is loaded from A);
//      rows r >= j: x_r = colr[r] - (v_{j-1}[r] a'_j + p'_{j-1}[r] b_j) (the pending update), sigma =
//      ||x[j+2:]||^2 by a CTA reduction, the Householder scalars, v_j into vloc[par]; the owner keeps d_j,
//      beta, tau_j and the reflector for the output
//   U2 the pending update on the own columns; the owner of column j + 1 stages it (rows >= j + 1) and,
//      after the CTA barrier, one bulk copy per destination CTA (lanes 0-1 of every warp) pushes it into
//      colr[(j + 1) & 1] completing on rbar[(j + 1) & 1]
//   D  column sums A[:, g] v_j of the own columns g > j, p_g all-gathered (st.async into every CTA's
//      ploc[par][g], the CTA's part of p.v_j into wpart[par][rank]); wait pbar; K_j
#pragma once
#include "cluster_la.cuh"

namespace psd {

__host__ __device__ inline size_t tri_rep_smem_doubles(int s, int CS) {
  const size_t sr = (size_t)((s + 1) & ~1);
  // refl (ncl x sr) | vloc 2 sr | ploc 2 sr | colr 2 sr | colb sr | wred 2 x 256 | wpart 64 | dl, el, tl
  return (size_t)cdiv(s, CS) * sr + 7 * sr + 2 * 8 * 32 + 64 + 3 * (size_t)cdiv(s, CS) + 16;
}

template <int KR, int CR>
__global__ void __launch_bounds__(256, 1) tridiag_rep_kernel(int s, const double* __restrict__ A, int lda,
                                                             double* __restrict__ d, double* __restrict__ e,
                                                             double* __restrict__ tau, double* __restrict__ Vh, int ldv) {
  constexpr int NT = 256, RG = 64, TCG = TRI_TCG, CRP = tri_pow2_ceil(CR);
  static_assert(RG * TCG == NT, "thread layout");
  static_assert(CRP <= 32, "columns per thread");
  static_assert(2 * NT >= RG * KR, "replica rows per thread (s <= 512)");
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t pbar[2], rbar[2];
  __shared__ double hred[2][10];
  const int CS = (int)gridDim.x;
  const unsigned rank = cla_rank();
  const int ncl = cdiv(s, CS);
  const int sr = (s + 1) & ~1;
  double* refl = sm;                       // ncl x sr: reflectors of the own columns (tau_j at row j)
  double* vloc = refl + (size_t)ncl * sr;  // 2 x sr (parity): [tau_j at j | v_j at j+1..s-1]
  double* ploc = vloc + 2 * (size_t)sr;    // 2 x sr (parity): p_j (pushed by the column owners)
  double* colr = ploc + 2 * (size_t)sr;    // 2 x sr (column parity): replica of the step's column
  double* colb = colr + 2 * (size_t)sr;    // sr: staging of the own column j + 1 for its push
  double* wred = colb + sr;                // 2 x 8 warps x 32: per-warp column partials (parity)
  double* wpart = wred + 2 * 8 * 32;       // 2 x 32 (parity): every CTA's part of p.v_j, by rank
  double* dl = wpart + 64;
  double* el = dl + ncl;
  double* tl = el + ncl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cg = tid / RG, rg = tid % RG;
  for (size_t q = tid; q < tri_rep_smem_doubles(s, CS); q += NT) sm[q] = 0.0;
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
  // the replica of column 0 straight from A (every CTA)
  for (int r = tid; r < s; r += NT) colr[r] = 0.5 * (A[IDX(r, 0, lda)] + A[IDX(0, r, lda)]);
  auto rbytes = [&](int c) -> uint32_t { return 8u * (uint32_t)(sr - (c & ~1)); };
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      cla_mbar_init(&pbar[b], 1);
      cla_mbar_init(&rbar[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int jj = 0; jj < 2 && jj + 2 < s; ++jj) cla_mbar_arm(&pbar[jj], 8u * (uint32_t)(s - jj - 1 + CS));
    // replicas of columns 1 and 2 (pushed during steps 0 and 1)
    for (int c = 1; c <= 2 && c <= s - 3; ++c) cla_mbar_arm(&rbar[c & 1], rbytes(c));
  }
  __syncthreads();
  cla_cluster_sync();  // every CTA's barriers are initialised and armed before the first push
  double Kp = 0.0;     // K_{j-1}
  for (int j = 0; j + 2 < s; ++j) {
    const int owner = j & (CS - 1), par = j & 1, pp = par ^ 1;
    const bool pend = j > 0;
    double* vj = vloc + (size_t)par * sr;
    const double* vp = vloc + (size_t)pp * sr;
    const double* pq = ploc + (size_t)pp * sr;
    const double* cr = colr + (size_t)(j & 1) * sr;
    if (j >= 1) {
      cla_mbar_wait(&rbar[j & 1], (uint32_t)((j - 1) >> 1) & 1u);  // the replica of column j
      if (tid == 0 && j + 2 <= s - 3) cla_mbar_arm(&rbar[j & 1], rbytes(j + 2));
    }
    // ---- R: the pending update on the replica, sigma, Householder scalars, v_j (every CTA)
    const double bj = pend ? vp[j] : 0.0;
    const double aj = pend ? pq[j] - 2.0 * Kp * bj : 0.0;
    double xr[2];
    double sg = 0.0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = j + tid + NT * q;
      double x = 0.0;
      if (r < s) {
        x = cr[r];
        if (pend) x = fma(-vp[r], aj, fma(-pq[r], bj, x));
        if (r >= j + 2) sg = fma(x, x, sg);
      }
      xr[q] = x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
    if (lane == 0) hred[par][warp] = sg;
    if (tid == 0) hred[par][8] = xr[0];  // d_j (row j)
    if (tid == 1) hred[par][9] = xr[0];  // alpha (row j + 1)
    __syncthreads();
    double sigma = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) sigma += hred[par][w];  // fixed order: identical in every CTA
    const double dj = hred[par][8], alpha = hred[par][9];
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
    const bool own_j = (int)rank == owner;
    const int lj = j / CS;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = j + tid + NT * q;
      if (r > j && r < s) {
        const double v = (r == j + 1) ? 1.0 : xr[q] * scale;
        vj[r] = v;
        if (own_j) refl[(size_t)lj * sr + r] = v;
      }
    }
    if (tid == 0) {
      vj[j] = tj;
      if (own_j) {
        refl[(size_t)lj * sr + j] = tj;
        dl[lj] = dj;
        el[lj] = beta;
        tl[lj] = tj;
      }
    }
    // ---- U2: the pending update (step j - 1) on the own columns; column j + 1 staged by its owner
    double rv[KR], rp[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = rg + RG * k;
      const bool ok = pend && r >= j && r < s;
      rv[k] = ok ? vp[r] : 0.0;
      rp[k] = ok ? pq[r] : 0.0;
    }
    const int jn = j + 1;  // the next step's column
    const bool push_next = jn <= s - 3 && (int)rank == (jn & (CS - 1));
    const int ljn = jn / CS, cgn = ljn & (TCG - 1), cn = ljn >> 2;
#pragma unroll
    for (int c = 0; c < CR; ++c) {
      const int g = (int)rank + CS * (cg + TCG * c);
      const bool act = pend && g >= j && g < s;
      const double bg = act ? vp[g] : 0.0;
      const double ag = act ? pq[g] - 2.0 * Kp * bg : 0.0;
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        if (pend && RG * k < s && RG * k + RG - 1 >= j) a[k][c] = fma(-rv[k], ag, fma(-rp[k], bg, a[k][c]));
      }
      if (push_next && cg == cgn && c == cn) {
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const int r = rg + RG * k;
          if (r >= (jn & ~1) && r < sr) colb[r] = r < s ? a[k][c] : 0.0;
        }
      }
    }
    __syncthreads();  // v_j complete; column j + 1 staged
    if (push_next) {
      const int bdst = ((tid & 31) < 2) ? 2 * warp + (tid & 31) : CS;
      if (bdst < CS) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int i0 = jn & ~1;
        double* dstp = colr + (size_t)(jn & 1) * sr + i0;
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                cla_mapa(cla_smem_u32(dstp), (uint32_t)bdst)),
            "r"(cla_smem_u32(colb + i0)), "r"(rbytes(jn)), "r"(cla_mapa(cla_smem_u32(&rbar[jn & 1]), (uint32_t)bdst))
            : "memory");
      }
    }
    // ---- D: column sums of A[:, g] v_j (rows > j) for the own columns, p all-gather
    const double tjv = vj[j];
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
    __syncthreads();
    {
      double part = 0.0, pg = 0.0;
      const int lc = lane, g = (int)rank + CS * lc;
      const bool act = lc < ncl && g > j && g < s;
      if (act) {
        const int cgl = lc % TCG, c = lc / TCG;
        pg = tjv * (wr[(2 * cgl) * 32 + c] + wr[(2 * cgl + 1) * 32 + c]);
      }
      if constexpr (CRP > CR) {
        double q = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) q += wr[w * 32 + CR];
        part = tjv * q;
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
    cla_mbar_wait(&pbar[par], (uint32_t)(j >> 1) & 1u);  // p_j and the CTAs' parts of p.v_j
    if (tid == 0 && j + 4 < s) cla_mbar_arm(&pbar[par], 8u * (uint32_t)(s - j - 3 + CS));
    {
      double k0 = 0.0, k1 = 0.0;
      for (int q = 0; q < CS; q += 2) {
        k0 += wpart[par * 32 + q];
        k1 += wpart[par * 32 + q + 1];
      }
      Kp = 0.5 * tjv * (k0 + k1);
    }
  }
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

}  // namespace psd
