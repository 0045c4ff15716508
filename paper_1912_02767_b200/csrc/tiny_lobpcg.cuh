// tiny_lobpcg.cuh -- f4: many tiny cone blocks of the Bayesian-optimisation kind, whose
// PSD parts have rank one or a few ("rank-one solutions"). ONE CTA runs the whole
// warm-started LOBPCG of one block (Alg. 3, positive side) with the matrix and every
// tall-skinny block in shared memory: block multiply, residuals, Gram / pencil, Cholesky-QR, the small
// Rayleigh-Ritz eigenproblem (one-CTA parallel Jacobi, jacobi_smem_core), rotation, random expansion
// (line 8) and the Theorem-3 certification at exit -- one launch for the whole batch, no host round trip
// per iteration. Readings as the main path (R5-R13, R20, R52, R53); guard g and warm width p + g are this
// path's own (BO blocks have p ~ 1: the main path's 16-wide guard band, R56, would triple their basis).
//
// A block that needs more than TL_MCAP columns, or whose pencil stays singular, or n < 3 (m0 + 1), is
// returned with status TL_NEEDS_EXACT and Pi untouched: the host projects those with the exact one-CTA
// path (psdproj_project_tiny_batched, R50) -- the DIRECT branch of the one-third rule.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace psd {

constexpr int TL_NT = 256;
constexpr int TL_NMAX = 112;
constexpr int TL_MCAP = 8;
constexpr int TL_SMAX = 3 * TL_MCAP + 1;  // [X | W | E | P], one pending expansion column
constexpr int TL_OK = 0, TL_NOT_CONVERGED = 1, TL_NEEDS_EXACT = 2;

struct TinyLobBlock {
  const double* A;
  double* Pi;
  double* Xw;  // warm block (n x TL_MCAP, ld n), caller-owned
  int n, lda, ldpi, pad;
};
struct TinyLobOut {
  double bound;  // Theorem-3 bound (R53 form, perp term 0 as the paper)
  double anorm;
  int status, iters, npos, m;  // m: warm width in / out (0 = cold)
};

__host__ __device__ inline size_t tiny_lob_smem_doubles(int nmax) {
  const size_t n = nmax;
  return n * n + 2 * n * TL_SMAX + 6 * n * TL_MCAP + 5 * (size_t)TL_SMAX * TL_SMAX +
         2 * (size_t)(TL_SMAX + 1) * (TL_SMAX + 2) + 8 * TL_SMAX + 64;
}

// Y[:, j] = A X[:, j], j < cols (A n x n ld n, X / Y ld n), all threads
__device__ __forceinline__ void tl_matmul(int n, const double* __restrict__ A, const double* __restrict__ X, int cols,
                                          double* __restrict__ Y) {
  for (int o = threadIdx.x; o < n * cols; o += TL_NT) {
    const int i = o % n, j = o / n;
    const double* x = X + (size_t)j * n;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(A[i + k * n], x[k], acc);
    Y[i + (size_t)j * n] = acc;
  }
}
// G = S^T T (cs x ct, ld ldg), columns of length n (ld n)
__device__ __forceinline__ void tl_gram(int n, const double* __restrict__ S, int cs, const double* __restrict__ T,
                                        int ct, double* __restrict__ G, int ldg) {
  for (int o = threadIdx.x; o < cs * ct; o += TL_NT) {
    const int i = o % cs, j = o / cs;
    const double* a = S + (size_t)i * n;
    const double* b = T + (size_t)j * n;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc = fma(a[k], b[k], acc);
    G[i + j * ldg] = acc;
  }
}
// Y (n x m) = S (n x s) C (s x m, ld ldc)
__device__ __forceinline__ void tl_rot(int n, const double* __restrict__ S, int s, const double* __restrict__ C,
                                       int ldc, int m, double* __restrict__ Y) {
  for (int o = threadIdx.x; o < n * m; o += TL_NT) {
    const int i = o % n, j = o / n;
    double acc = 0.0;
    for (int k = 0; k < s; ++k) acc = fma(S[i + (size_t)k * n], C[k + j * ldc], acc);
    Y[i + (size_t)j * n] = acc;
  }
}
// column 2-norms of Z (n x cols, ld n) into out[cols]: one warp per column
__device__ __forceinline__ void tl_colnorms(int n, const double* __restrict__ Z, int cols, double* __restrict__ out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int j = w; j < cols; j += TL_NT / 32) {
    double acc = 0.0;
    for (int k = l; k < n; k += 32) acc = fma(Z[k + (size_t)j * n], Z[k + (size_t)j * n], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (l == 0) out[j] = sqrt(acc);
  }
}
// In-place Cholesky of the leading t x t block of G (ld ldg), right-looking, all threads; returns 0 or
// (failing pivot + 1) when a pivot is <= 1e-12 max diag (R20). Upper triangle left untouched.
__device__ int tl_cholesky(int t, double* __restrict__ G, int ldg, int* __restrict__ flag) {
  (void)flag;
  double dmax = 0.0;
  for (int i = 0; i < t; ++i) dmax = fmax(dmax, G[i + i * ldg]);
  __syncthreads();  // every thread has read the diagonal before thread 0 overwrites it
  for (int j = 0; j < t; ++j) {
    int bad = 0;
    if (threadIdx.x == 0) {
      const double d = G[j + j * ldg];
      if (!(d > 1e-12 * dmax))
        bad = 1;
      else
        G[j + j * ldg] = sqrt(d);
    }
    // the failure decision travels with the barrier itself: identical in every thread
    if (__syncthreads_or(bad)) return j + 1;
    const double ljj = G[j + j * ldg];
    for (int i = j + 1 + threadIdx.x; i < t; i += TL_NT) G[i + j * ldg] /= ljj;
    __syncthreads();
    // trailing update of the lower triangle: G[i][k] -= L[i][j] L[k][j], j < k <= i
    const int r = t - j - 1;
    for (int o = threadIdx.x; o < r * r; o += TL_NT) {
      const int i = j + 1 + o % r, k = j + 1 + o / r;
      if (k <= i) G[i + k * ldg] -= G[i + j * ldg] * G[k + j * ldg];
    }
    __syncthreads();
  }
  return 0;
}
// Li = L^-1 (lower, t x t) by forward substitution, one thread per column
__device__ void tl_trinv(int t, const double* __restrict__ L, int ldl, double* __restrict__ Li, int ldi) {
  for (int c = threadIdx.x; c < t; c += TL_NT) {
    for (int i = 0; i < t; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      if (i < c) {
        Li[i + c * ldi] = 0.0;
        continue;
      }
      for (int k = c; k < i; ++k) v -= L[i + k * ldl] * Li[k + c * ldi];
      Li[i + c * ldi] = v / L[i + i * ldl];
    }
  }
}
// N(0,1) column for the expansion / cold start: the Philox stream of R11 keyed by (seed, block, call tag)
__device__ __forceinline__ double tl_gauss(uint64_t seed, uint32_t blk, uint32_t tag, uint32_t l) {
  uint32_t c[4] = {l >> 1, 0x7F4A0000u | (tag & 0xFFFF), blk, 0x71A7u};
  philox10(c, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  const double u1 = u53(c[0], c[1]), u2 = u53(c[2], c[3]);
  const double rad = sqrt(-2.0 * log(u1));
  double sv, cv;
  sincospi(2.0 * u2, &sv, &cv);
  return (l & 1) ? rad * sv : rad * cv;
}

__global__ void __launch_bounds__(TL_NT) tiny_lobpcg_kernel(const TinyLobBlock* __restrict__ blocks,
                                                           TinyLobOut* __restrict__ outs, double tol, int max_iter,
                                                           int guard, int m0, uint64_t seed, uint32_t call) {
  extern __shared__ __align__(16) double sm[];
  const TinyLobBlock bk = blocks[blockIdx.x];
  TinyLobOut* out = outs + blockIdx.x;
  const int n = bk.n;
  const int tid = threadIdx.x;
  // shared layout
  double* A = sm;
  double* S = A + (size_t)n * n;                 // n x SMAX: [X | W | E | P]
  double* BS = S + (size_t)n * TL_SMAX;           // B-images
  double* Pb = BS + (size_t)n * TL_SMAX;          // n x MCAP: P directions
  double* BPb = Pb + (size_t)n * TL_MCAP;
  double* T1 = BPb + (size_t)n * TL_MCAP;
  double* T2 = T1 + (size_t)n * TL_MCAP;
  double* T3 = T2 + (size_t)n * TL_MCAP;
  double* T4 = T3 + (size_t)n * TL_MCAP;
  double* G = T4 + (size_t)n * TL_MCAP;           // SMAX^2 each, ld SMAX
  double* H = G + TL_SMAX * TL_SMAX;
  double* Li = H + TL_SMAX * TL_SMAX;
  double* Hh = Li + TL_SMAX * TL_SMAX;
  double* Cp = Hh + TL_SMAX * TL_SMAX;
  double* jws = Cp + TL_SMAX * TL_SMAX;           // 2 (SMAX + 1) (SMAX + 2)
  double* th = jws + 2 * (TL_SMAX + 1) * (TL_SMAX + 2);  // SMAX each:
  double* rr = th + TL_SMAX;
  double* nrm = rr + TL_SMAX;
  double* lam = nrm + TL_SMAX;
  double* scal = lam + TL_SMAX;                   // 64 scalars
  __shared__ int ord[TL_SMAX], act[TL_MCAP], hasp[TL_MCAP], iflag[4];
  __shared__ int sh_a, sh_ap, sh_qe, sh_state, sh_conv;
  const int nIn = n;
  if (nIn <= 0) return;
  // ---- load A (symmetrised) and its Frobenius norm
  double fro = 0.0;
  for (int e = tid; e < n * n; e += TL_NT) {
    const int i = e % n, j = e / n;
    const double v = 0.5 * (bk.A[IDX(i, j, bk.lda)] + bk.A[IDX(j, i, bk.lda)]);
    A[i + j * n] = v;
    fro += v * v;
  }
  fro = sqrt(block_sum<TL_NT>(fro, scal));
  int m = out->m;
  const bool cold = m <= 0;
  // cold: max(m0, ceil(n/10)) Philox columns (R28's width), within the block capacity and 3 m + 1 <= n
  if (cold) m = min(min(max(m0, (n + 9) / 10), TL_MCAP), max(1, (n - 1) / 3));
  if (tid == 0) {
    out->anorm = fro;
    sh_state = (n < 3 * m + 1 || m > TL_MCAP) ? TL_NEEDS_EXACT : -1;
  }
  __syncthreads();
  if (sh_state == TL_NEEDS_EXACT) {
    if (tid == 0) {
      out->status = TL_NEEDS_EXACT;
      out->iters = 0;
      out->npos = -1;
      out->bound = 0.0;
      out->m = 0;
    }
    return;
  }
  // ---- start block X0 (warm: previous block; cold: Philox) in S[:, 0:m]; orthonormalise (CholQR)
  for (int e = tid; e < n * m; e += TL_NT) {
    const int i = e % n, j = e / n;
    S[i + j * n] = cold ? tl_gauss(seed, blockIdx.x, call, (uint32_t)(i + j * n)) : bk.Xw[i + (size_t)j * n];
  }
  __syncthreads();
  tl_gram(n, S, m, S, m, G, TL_SMAX);
  __syncthreads();
  if (tl_cholesky(m, G, TL_SMAX, iflag)) {
    if (tid == 0) {
      out->status = TL_NEEDS_EXACT;
      out->iters = 0;
      out->npos = -1;
      out->m = 0;
    }
    return;
  }
  tl_trinv(m, G, TL_SMAX, Li, TL_SMAX);
  __syncthreads();
  // X <- X0 L^-T
  for (int o = tid; o < n * m; o += TL_NT) {
    const int i = o % n, j = o / n;
    double acc = 0.0;
    for (int k = 0; k <= j; ++k) acc = fma(S[i + k * n], Li[j + k * TL_SMAX], acc);
    T1[i + j * n] = acc;
  }
  __syncthreads();
  for (int o = tid; o < n * m; o += TL_NT) S[o] = T1[o];
  __syncthreads();
  // initial Rayleigh-Ritz on span(X0) (Alg. 3 line 2)
  tl_matmul(n, A, S, m, BS);
  __syncthreads();
  tl_gram(n, S, m, BS, m, Hh, TL_SMAX);
  __syncthreads();
  for (int o = tid; o < m * m; o += TL_NT) {  // symmetrise
    const int i = o % m, j = o / m;
    if (i < j) {
      const double v = 0.5 * (Hh[i + j * TL_SMAX] + Hh[j + i * TL_SMAX]);
      Hh[i + j * TL_SMAX] = v;
      Hh[j + i * TL_SMAX] = v;
    }
  }
  __syncthreads();
  {
    const int sw = jacobi_smem_core<TL_NT>(m, Hh, TL_SMAX, jws, 40);
    (void)sw;
    const int Nj = m + (m & 1), Lj = Nj + 1;
    if (tid == 0) {
      for (int i = 0; i < m; ++i) ord[i] = i;
      for (int i = 0; i < m; ++i)  // selection sort, descending, ties by index (R21)
        for (int j = i + 1; j < m; ++j)
          if (jws[ord[j] + ord[j] * Lj] > jws[ord[i] + ord[i] * Lj]) {
            const int t = ord[i];
            ord[i] = ord[j];
            ord[j] = t;
          }
      for (int i = 0; i < m; ++i) th[i] = jws[ord[i] + ord[i] * Lj];
    }
    __syncthreads();
    const double* Q = jws + Nj * Lj;
    for (int o = tid; o < m * m; o += TL_NT) {
      const int i = o % m, j = o / m;
      Cp[i + j * TL_SMAX] = Q[i + ord[j] * Lj];
    }
    __syncthreads();
    tl_rot(n, S, m, Cp, TL_SMAX, m, T1);
    tl_rot(n, BS, m, Cp, TL_SMAX, m, T2);
    __syncthreads();
    for (int o = tid; o < n * m; o += TL_NT) {
      S[o] = T1[o];
      BS[o] = T2[o];
    }
    if (tid < TL_MCAP) hasp[tid] = 0;
    if (tid == 0) sh_qe = 0;
    __syncthreads();
  }
  int k = 0, status = TL_NOT_CONVERGED;
  for (;;) {
    // ---- R = B X - X Theta in T1, residual norms
    for (int o = tid; o < n * m; o += TL_NT) {
      const int j = o / n;
      T1[o] = BS[o] - th[j] * S[o];
    }
    __syncthreads();
    tl_colnorms(n, T1, m, rr);
    __syncthreads();
    if (tid == 0 && bk.pad == 1) {  // debugging (PSDPROJ_TINY_DEBUG = block index)
      printf("tiny k=%d m=%d qe=%d:", k, m, sh_qe);
      for (int j = 0; j < m; ++j) printf(" (%.6g, %.3g)", th[j], rr[j]);
      printf("\n");
    }
    if (tid == 0) {
      // stopping rule (R12, R52, R60): positives r <= tol, largest non-positive: theta_g + r_g <= tol, r_g <= max(tol, |theta_g|/2); k >= 1 cold
      int npos = 0, g = -1;
      bool conv = true;
      for (int j = 0; j < m; ++j) {
        if (th[j] > 0.0) {
          ++npos;
          if (!(rr[j] <= tol)) conv = false;
        } else if (g < 0 || th[j] > th[g]) {
          g = j;
        }
      }
      const bool guard_ok =
          (m >= n) || (g >= 0 && th[g] + rr[g] <= tol && rr[g] <= fmax(tol, 0.5 * fabs(th[g])));  // R52, R60
      sh_conv = conv && guard_ok && sh_qe == 0 && !(cold && k == 0);
      (void)npos;
      int a = 0;
      for (int j = 0; j < m; ++j)
        if (rr[j] > tol) act[a++] = j;  // active mask (BLOPEX soft locking)
      sh_a = a;
      int ap = 0;
      for (int jj = 0; jj < a; ++jj) ap += hasp[act[jj]];
      sh_ap = ap;
      // no non-positive column left (npos == m) and no expansion pending: draw one (line 8, R8)
      if (!sh_conv && g < 0 && sh_qe == 0 && m < n) sh_qe = 1;
      sh_state = -1;
      if (m + sh_qe > TL_MCAP || 3 * (m + sh_qe) + 1 > n) sh_state = TL_NEEDS_EXACT;
    }
    __syncthreads();
    if (sh_conv) {
      status = TL_OK;
      break;
    }
    if (sh_state == TL_NEEDS_EXACT) {
      status = TL_NEEDS_EXACT;
      break;
    }
    if (k >= max_iter) break;
    const int a = sh_a, ap = sh_ap, qe = sh_qe;
    // ---- basis S = [X | W | E | P_J]: W = R_J / r_J, E the expansion column (orthogonalised
    // against X, twice), P_J normalised (with its B-image)
    const int offW = m, offE = m + a, offP = m + a + qe;
    int s = offP + ap;
    for (int o = tid; o < n * a; o += TL_NT) {
      const int i = o % n, jj = o / n, j = act[jj];
      S[i + (offW + jj) * n] = T1[i + j * n] / rr[j];
    }
    if (qe) {
      for (int i = tid; i < n; i += TL_NT) S[i + offE * n] = tl_gauss(seed, blockIdx.x, call * 4096u + k + 1, i);
    }
    if (ap) {
      if (tid == 0) {
        int c = 0;
        for (int jj = 0; jj < a; ++jj)
          if (hasp[act[jj]]) ord[c++] = act[jj];
      }
      __syncthreads();
      for (int o = tid; o < n * ap; o += TL_NT) {
        const int i = o % n, c = o / n, j = ord[c];
        S[i + (offP + c) * n] = Pb[i + j * n];
        BS[i + (offP + c) * n] = BPb[i + j * n];
      }
    }
    __syncthreads();
    if (qe) {  // CGS2 of E against X
      for (int pass = 0; pass < 2; ++pass) {
        tl_gram(n, S, m, S + offE * n, 1, nrm, 1);
        __syncthreads();
        for (int i = tid; i < n; i += TL_NT) {
          double v = S[i + offE * n];
          for (int j = 0; j < m; ++j) v -= S[i + j * n] * nrm[j];
          S[i + offE * n] = v;
        }
        __syncthreads();
      }
      tl_colnorms(n, S + offE * n, 1, nrm);
      __syncthreads();
      for (int i = tid; i < n; i += TL_NT) S[i + offE * n] /= nrm[0];
      __syncthreads();
    }
    if (ap) {
      tl_colnorms(n, S + offP * n, ap, nrm);
      __syncthreads();
      for (int o = tid; o < n * ap; o += TL_NT) {
        const int c = o / n;
        S[o + offP * n] /= nrm[c];
        BS[o + offP * n] /= nrm[c];
      }
      __syncthreads();
    }
    // B [W E] (the block multiply, a3)
    tl_matmul(n, A, S + offW * n, a + qe, BS + offW * n);
    __syncthreads();
    // ---- pencil (G, H) with the known X blocks, Cholesky; drop P on failure (R20)
    tl_gram(n, S, s, S, s, G, TL_SMAX);
    tl_gram(n, S, s, BS, s, H, TL_SMAX);
    __syncthreads();
    for (int o = tid; o < s * s; o += TL_NT) {
      const int i = o % s, j = o / s;
      if (i < m && j < m) {
        G[i + j * TL_SMAX] = (i == j) ? 1.0 : 0.0;
        H[i + j * TL_SMAX] = (i == j) ? th[i] : 0.0;
      } else if (i < j) {
        const double g2 = 0.5 * (G[i + j * TL_SMAX] + G[j + i * TL_SMAX]);
        const double h2 = 0.5 * (H[i + j * TL_SMAX] + H[j + i * TL_SMAX]);
        G[i + j * TL_SMAX] = g2;
        G[j + i * TL_SMAX] = g2;
        H[i + j * TL_SMAX] = h2;
        H[j + i * TL_SMAX] = h2;
      }
    }
    __syncthreads();
    // Cholesky on a copy (Li as scratch): G stays for a retry
    for (int o = tid; o < s * s; o += TL_NT) Li[o % s + (o / s) * TL_SMAX] = G[o % s + (o / s) * TL_SMAX];
    __syncthreads();
    int fail = tl_cholesky(s, Li, TL_SMAX, iflag);
    if (fail && ap) {
      s = offP;
      for (int o = tid; o < s * s; o += TL_NT) Li[o % s + (o / s) * TL_SMAX] = G[o % s + (o / s) * TL_SMAX];
      __syncthreads();
      fail = tl_cholesky(s, Li, TL_SMAX, iflag);
    }
    if (fail) {
      status = TL_NEEDS_EXACT;
      break;
    }
    // L^-1 into Hh (scratch), then Hh <- L^-1 H L^-T via Cp
    tl_trinv(s, Li, TL_SMAX, Hh, TL_SMAX);
    __syncthreads();
    for (int o = tid; o < s * s; o += TL_NT) {  // Cp = L^-1 H
      const int i = o % s, j = o / s;
      double acc = 0.0;
      for (int kk = 0; kk <= i; ++kk) acc = fma(Hh[i + kk * TL_SMAX], H[kk + j * TL_SMAX], acc);
      Cp[i + j * TL_SMAX] = acc;
    }
    __syncthreads();
    for (int o = tid; o < s * s; o += TL_NT) {  // G (free now) = Cp L^-T, symmetric part
      const int i = o % s, j = o / s;
      double acc = 0.0;
      for (int kk = 0; kk <= j; ++kk) acc = fma(Cp[i + kk * TL_SMAX], Hh[j + kk * TL_SMAX], acc);
      G[i + j * TL_SMAX] = acc;
    }
    __syncthreads();
    for (int o = tid; o < s * s; o += TL_NT) {
      const int i = o % s, j = o / s;
      if (i < j) {
        const double v = 0.5 * (G[i + j * TL_SMAX] + G[j + i * TL_SMAX]);
        G[i + j * TL_SMAX] = v;
        G[j + i * TL_SMAX] = v;
      }
    }
    __syncthreads();
    // ---- Rayleigh-Ritz eigenproblem (one-CTA Jacobi), top m + qe pairs (R7), C' = L^-T C
    const int sw = jacobi_smem_core<TL_NT>(s, G, TL_SMAX, jws, 40);
    if (sw < 0) {
      status = TL_NEEDS_EXACT;
      break;
    }
    const int Nj = s + (s & 1), Lj = Nj + 1;
    const int mn = min(m + qe, s);
    if (tid == 0) {
      for (int i = 0; i < s; ++i) ord[i] = i;
      for (int i = 0; i < s; ++i)
        for (int j = i + 1; j < s; ++j)
          if (jws[ord[j] + ord[j] * Lj] > jws[ord[i] + ord[i] * Lj]) {
            const int t = ord[i];
            ord[i] = ord[j];
            ord[j] = t;
          }
      for (int i = 0; i < mn; ++i) lam[i] = jws[ord[i] + ord[i] * Lj];
    }
    __syncthreads();
    const double* Q = jws + Nj * Lj;
    for (int o = tid; o < s * mn; o += TL_NT) {  // C' = L^-T Q[:, ord[:mn]]
      const int i = o % s, j = o / s;
      double acc = 0.0;
      for (int kk = i; kk < s; ++kk) acc = fma(Hh[kk + i * TL_SMAX], Q[kk + ord[j] * Lj], acc);
      Cp[i + j * TL_SMAX] = acc;
    }
    __syncthreads();
    // ---- rotation (a8): X = S C', BX = BS C', P = S[:, m:] C'[m:], BP likewise
    tl_rot(n, S, s, Cp, TL_SMAX, mn, T1);
    tl_rot(n, BS, s, Cp, TL_SMAX, mn, T2);
    tl_rot(n, S + (size_t)m * n, s - m, Cp + m, TL_SMAX, mn, T3);
    tl_rot(n, BS + (size_t)m * n, s - m, Cp + m, TL_SMAX, mn, T4);
    __syncthreads();
    for (int o = tid; o < n * mn; o += TL_NT) {
      S[o] = T1[o];
      BS[o] = T2[o];
      Pb[o] = T3[o];
      BPb[o] = T4[o];
    }
    if (tid < mn) {
      th[tid] = lam[tid];
      hasp[tid] = 1;
    }
    if (tid == 0) sh_qe = 0;
    m = mn;
    ++k;
    __syncthreads();
  }
  // ---- exit: certification (R53) with an explicit B V+, Pi = V+ Theta+ V+^T, warm block
  int p = 0;
  for (int j = 0; j < m; ++j) p += th[j] > 0.0;  // th is sorted descending
  if (status == TL_NEEDS_EXACT) {
    if (tid == 0) {
      out->status = TL_NEEDS_EXACT;
      out->iters = k;
      out->npos = -1;
      out->m = 0;
      out->bound = 0.0;
    }
    return;
  }
  if (p > 0) {
    tl_matmul(n, A, S, p, T2);
    __syncthreads();
    for (int o = tid; o < n * p; o += TL_NT) T1[o] = T2[o] - th[o / n] * S[o];
    __syncthreads();
    tl_colnorms(n, T1, p, rr);
    tl_gram(n, S, p, T2, p, G, TL_SMAX);
    tl_gram(n, S, p, S, p, H, TL_SMAX);
    __syncthreads();
    if (tid == 0) {
      double rs = 0.0, d2 = 0.0, e2 = 0.0, thmax = 0.0;
      for (int j = 0; j < p; ++j) {
        rs += rr[j] * rr[j];
        thmax = fmax(thmax, th[j]);
        for (int i = 0; i < p; ++i) {
          const double dv = G[i + j * TL_SMAX] - (i == j ? th[j] : 0.0);
          const double ev = H[i + j * TL_SMAX] - (i == j ? 1.0 : 0.0);
          d2 += dv * dv;
          e2 += ev * ev;
        }
      }
      const double d = sqrt(d2), e = sqrt(e2);
      out->bound = (1.0 + e) * sqrt(2.0 * rs) + (1.0 + sqrt(2.0)) * d + 7.0 * e * thmax + 4.0 * n * PSD_U * fro;
    }
  } else if (tid == 0) {
    out->bound = 4.0 * n * PSD_U * fro;
  }
  // Pi = sum_{theta > 0} theta x x^T, each (i <= j) once and mirrored (exactly symmetric, R24)
  for (int e = tid; e < n * n; e += TL_NT) {
    const int i = e % n, j = e / n;
    if (i > j) continue;
    double acc = 0.0;
    for (int c = 0; c < p; ++c) acc = fma(th[c] * S[i + c * n], S[j + c * n], acc);
    bk.Pi[IDX(i, j, bk.ldpi)] = acc;
    bk.Pi[IDX(j, i, bk.ldpi)] = acc;
  }
  // warm block: positives + max(g, 1) non-positive columns
  const int keep = min(m, p + max(guard, 1));
  for (int o = tid; o < n * keep; o += TL_NT) bk.Xw[o] = S[o];
  if (tid == 0) {
    out->status = status;
    out->iters = k;
    out->npos = p;
    out->m = keep;
  }
}

}  // namespace psd
