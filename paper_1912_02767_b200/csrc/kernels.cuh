// kernels.cuh -- non-GEMM kernels of the psdproj path (sm_100a).
//
//   resid_norm      a4: R = B X - X diag(theta), r_j = ||R_:,j||_2
//   colnorm/scale   unit-column scaling of the residual / direction blocks (R6, §8.c.3 4.4)
//   gather_cols     active-set compaction (BLOPEX active mask)
//   philox_gauss    cold block / random expansion (Alg. 3 line 8; R11)
//   insert_known    known Gram blocks X^T X = I, X^T B X = Theta (a5)
//   cholesky / trinv  implicit Cholesky-QR of the pencil (a6)
//   jacobi_*        Rayleigh-Ritz eigensolve of L^-1 H L^-T (a7, Alg. 2) and the
//                   DIRECT full eigendecomposition (a13)
//   sort_desc       Ritz values in descending order, "the m largest"
//   symmetrize      exact symmetry of Pi (R24)
// Every reduction is a fixed-order tree (deterministic, R25).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace psd {
namespace cg = cooperative_groups;

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < NT / 32) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- a4 residual + norms
// one CTA per column; R may be null (norms only). theta_sign: B = s*A already folded in BX.
template <int NT>
__global__ void __launch_bounds__(NT) resid_norm_kernel(int n, const double* __restrict__ X, int ldx,
                                                        const double* __restrict__ BX, int ldb,
                                                        const double* __restrict__ theta, double* __restrict__ R,
                                                        int ldr, double* __restrict__ rnorm, int squared = 0) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  __shared__ double red[32];
  int j = blockIdx.x;
  double th = theta[j];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) {
    double v = BX[IDX(i, j, ldb)] - th * X[IDX(i, j, ldx)];
    if (R) R[IDX(i, j, ldr)] = v;
    acc += v * v;
  }
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) rnorm[j] = squared ? acc : sqrt(acc);
}

template <int NT>
__global__ void __launch_bounds__(NT) colnorm_kernel(int n, const double* __restrict__ Z, int ld,
                                                     double* __restrict__ out, int squared = 0) {
  __shared__ double red[32];
  int j = blockIdx.x;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) {
    double v = Z[IDX(i, j, ld)];
    acc += v * v;
  }
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) out[j] = squared ? acc : sqrt(acc);
}

// colnorm_kernel + scale_cols_kernel in one pass per column (unsharded): norm[j] = ||Z[:, j]||,
// then Z[:, j] /= norm[j] (Z2 likewise; a zero norm leaves the column unchanged). Same reduction
// and the same per-element arithmetic as the two kernels.
template <int NT>
__global__ void __launch_bounds__(NT) colnorm_scale_kernel(int n, double* __restrict__ Z, int ld,
                                                           double* __restrict__ Z2, int ld2,
                                                           double* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  __shared__ double red[32];
  int j = blockIdx.x;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) {
    double v = Z[IDX(i, j, ld)];
    acc += v * v;
  }
  acc = block_sum<NT>(acc, red);
  const double s = sqrt(acc);
  if (threadIdx.x == 0) out[j] = s;
  if (s > 0.0) {
    const double inv = 1.0 / s;
    for (int i = threadIdx.x; i < n; i += NT) {
      Z[IDX(i, j, ld)] *= inv;
      if (Z2) Z2[IDX(i, j, ld2)] *= inv;
    }
  }
}

__global__ void i2d_kernel(const int* __restrict__ f, double* __restrict__ d) {
  if (threadIdx.x == 0) d[0] = (double)f[0];
}
__global__ void d2i_kernel(const double* __restrict__ d, int* __restrict__ f) {
  if (threadIdx.x == 0) f[0] = d[0] != 0.0 ? 1 : 0;
}

__global__ void sqrt_inplace_kernel(int k, double* __restrict__ v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) v[i] = sqrt(v[i]);
}

// row-sharded mode: Z_full (n x k, ldf) <- rank-major packed all-gather buffer (rank r's block is
// rows[r] x k with ld nrmax at offset r * nrmax * k; its rows start at global row offs[r])
__global__ void unpack_rows_kernel(int nranks, int nrmax, int k, const int* __restrict__ rows,
                                   const int* __restrict__ offs, const double* __restrict__ pack,
                                   double* __restrict__ full, int ldf) {
  const size_t per = (size_t)nrmax * k, total = per * nranks;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / per);
    const size_t w = e - (size_t)r * per;
    const int i = (int)(w % nrmax), j = (int)(w / nrmax);
    if (i < rows[r]) full[IDX(offs[r] + i, j, ldf)] = pack[e];
  }
}

// packed (ld = nrmax) copy of a local row block (the all-gather send buffer); rows >= nl zeroed
__global__ void pack_rows_kernel(int nl, int nrmax, int k, const double* __restrict__ src, int lds,
                                 double* __restrict__ dst) {
  const size_t total = (size_t)nrmax * k;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % nrmax), j = (int)(e / nrmax);
    dst[e] = (i < nl) ? src[IDX(i, j, lds)] : 0.0;
  }
}

// Z[:, j] /= norm[j] (and Z2 likewise when given); zero norms leave the column unchanged.
__global__ void scale_cols_kernel(int n, int cols, double* __restrict__ Z, int ld, double* __restrict__ Z2, int ld2,
                                  const double* __restrict__ norm) {
  size_t total = (size_t)n * cols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int i = (int)(e % n), j = (int)(e / n);
    double s = norm[j];
    if (s > 0.0) {
      double inv = 1.0 / s;
      Z[IDX(i, j, ld)] *= inv;
      if (Z2) Z2[IDX(i, j, ld2)] *= inv;
    }
  }
}

__global__ void gather_cols_kernel(int n, int cols, double* __restrict__ dst, int ldd, const double* __restrict__ src,
                                   int lds, const int* __restrict__ idx) {
  size_t total = (size_t)n * cols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int i = (int)(e % n), j = (int)(e / n);
    dst[IDX(i, j, ldd)] = src[IDX(i, idx[j], lds)];
  }
}

// Up to four column gathers in one launch: job q copies dst_q[:, j] = src_q[:, idx_q[j]]
// (idx_q null: src_q[:, j]) for j < cols_q; elements enumerated job by job.
struct GatherJob {
  double* dst;
  const double* src;
  const int* idx;
  int ldd, lds, cols;
};
struct GatherJobs {
  GatherJob j[4];
  int nj;
};
__global__ void gather_multi_kernel(int n, GatherJobs g) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  size_t total = 0;
  for (int q = 0; q < g.nj; ++q) total += (size_t)n * g.j[q].cols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t w = e;
    int q = 0;
    while (q + 1 < g.nj && w >= (size_t)n * g.j[q].cols) {
      w -= (size_t)n * g.j[q].cols;
      ++q;
    }
    const GatherJob& jb = g.j[q];
    const int i = (int)(w % n), c = (int)(w / n);
    jb.dst[IDX(i, c, jb.ldd)] = jb.src[IDX(i, jb.idx ? jb.idx[c] : c, jb.lds)];
  }
}

// dst[:, j] = src[:, j] * w[j]
__global__ void scale_copy_cols_kernel(int n, int cols, double* __restrict__ dst, int ldd,
                                       const double* __restrict__ src, int lds, const double* __restrict__ w) {
  size_t total = (size_t)n * cols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int i = (int)(e % n), j = (int)(e / n);
    dst[IDX(i, j, ldd)] = src[IDX(i, j, lds)] * w[j];
  }
}

// ---------------------------------------------------------------- Philox4x32-10 (R11)
__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
}

// raw uint32 stream (tests): out[4*i + j] = philox(counter=(i, c1, c2, c3), key)
__global__ void philox_raw_kernel(int count, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                                  uint32_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    uint32_t c[4] = {(uint32_t)i, c1, c2, c3};
    philox10(c, k0, k1);
    out[4 * i + 0] = c[0]; out[4 * i + 1] = c[1]; out[4 * i + 2] = c[2]; out[4 * i + 3] = c[3];
  }
}

__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6) + 0.5) * (1.0 / 9007199254740992.0);
}

// n x q standard normal block: linear index l = i + j*n; counter (l>>1, stream, ctx, tag)
__global__ void philox_gauss_kernel(int n, int q, double* __restrict__ dst, int ld, uint64_t seed, uint32_t stream,
                                    uint32_t ctx, uint32_t tag) {
  int64_t total = (int64_t)n * q;
  int64_t npairs = (total + 1) / 2;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < npairs; h += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[4] = {(uint32_t)h, stream, ctx, tag};
    philox10(c, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
    double u1 = u53(c[0], c[1]), u2 = u53(c[2], c[3]);
    double rad = sqrt(-2.0 * log(u1));
    double sv, cv;
    sincospi(2.0 * u2, &sv, &cv);
    int64_t l0 = 2 * h, l1 = 2 * h + 1;
    dst[IDX(l0 % n, l0 / n, ld)] = rad * cv;
    if (l1 < total) dst[IDX(l1 % n, l1 / n, ld)] = rad * sv;
  }
}

__global__ void philox_gauss_rows_kernel(int nl, int row0, int n, int q, double* __restrict__ dst, int ld,
                                         uint64_t seed, uint32_t stream, uint32_t ctx, uint32_t tag) {
  const int64_t total = (int64_t)nl * q;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % nl), j = (int)(e / nl);
    const int64_t l = (int64_t)(row0 + i) + (int64_t)j * n;
    uint32_t c[4] = {(uint32_t)(l >> 1), stream, ctx, tag};
    philox10(c, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
    const double u1 = u53(c[0], c[1]), u2 = u53(c[2], c[3]);
    const double rad = sqrt(-2.0 * log(u1));
    double sv, cv;
    sincospi(2.0 * u2, &sv, &cv);
    dst[IDX(i, j, ld)] = (l & 1) ? rad * sv : rad * cv;
  }
}

// W[:, j] = V[:, j] * sqrt(w[j]) (w > 0): Pi = W W^T is exactly symmetric entry by entry
__global__ void scale_sqrt_cols_kernel(int n, int cols, double* __restrict__ dst, int ldd,
                                       const double* __restrict__ src, int lds, const double* __restrict__ w) {
  size_t total = (size_t)n * cols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int i = (int)(e % n), j = (int)(e / n);
    dst[IDX(i, j, ldd)] = src[IDX(i, j, lds)] * sqrt(w[j]);
  }
}

// ---------------------------------------------------------------- a5 known blocks
// G, H (s x s, ld): symmetrise ((M + M^T)/2) and insert G[:kxG,:] = [I 0] (the directions are
// orthogonalised against X before the Gram), H[:kxH,:kxH] = diag(theta).
__global__ void insert_known_kernel(int s, int kxG, int kxH, double* __restrict__ G, double* __restrict__ H, int ld,
                                    const double* __restrict__ theta) {
  int total = s * s;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    int i = e % s, j = e / s;
    if (i > j) continue;
    // i <= j: i < kxG <= j is the X-W/P cross block, zero after the orthogonalisation
    double g = (j < kxG) ? ((i == j) ? 1.0 : 0.0)
                         : (i < kxG ? 0.0 : 0.5 * (G[IDX(i, j, ld)] + G[IDX(j, i, ld)]));
    double h = (j < kxH) ? ((i == j) ? theta[i] : 0.0) : 0.5 * (H[IDX(i, j, ld)] + H[IDX(j, i, ld)]);
    G[IDX(i, j, ld)] = g; G[IDX(j, i, ld)] = g;
    H[IDX(i, j, ld)] = h; H[IDX(j, i, ld)] = h;
  }
}

// One pass preparing the Rayleigh-Ritz pencil: insert_known_kernel's work, Li = [I 0; 0 0] (the
// Cholesky writes the L^-1 block), Gc = the direction block of G (the Cholesky input), status = 0.
// parts: bit 0 = the G side (G known blocks, Li, Gc, status), bit 1 = the H side (H known blocks).
__global__ void rr_prep_kernel(int s, int kxG, int kxH, double* __restrict__ G, double* __restrict__ H, int ld,
                               const double* __restrict__ theta, double* __restrict__ Li, double* __restrict__ Gc,
                               int* __restrict__ status, int parts) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  int total = s * s;
  const bool gs = parts & 1, hs = parts & 2;
  if (gs && blockIdx.x == 0 && threadIdx.x == 0) {
    *status = 0;
    *(unsigned long long*)(status + 16) = 0ull;  // linv_growth_kernel's key and block counter
    status[20] = 0;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    int i = e % s, j = e / s;
    if (gs) Li[IDX(i, j, ld)] = (i == j && i < kxG) ? 1.0 : 0.0;
    if (i > j) continue;
    if (gs) {
      double g = (j < kxG) ? ((i == j) ? 1.0 : 0.0)
                           : (i < kxG ? 0.0 : 0.5 * (G[IDX(i, j, ld)] + G[IDX(j, i, ld)]));
      G[IDX(i, j, ld)] = g; G[IDX(j, i, ld)] = g;
      if (i >= kxG) {
        Gc[IDX(i - kxG, j - kxG, ld)] = g;
        Gc[IDX(j - kxG, i - kxG, ld)] = g;
      }
    }
    if (hs) {
      double h = (j < kxH) ? ((i == j) ? theta[i] : 0.0) : 0.5 * (H[IDX(i, j, ld)] + H[IDX(j, i, ld)]);
      H[IDX(i, j, ld)] = h; H[IDX(j, i, ld)] = h;
    }
  }
}

// Hh's X rows / columns when L^-1 = [I 0; 0 Ld]: Hh[:kx, :kx] = H[:kx, :kx], Hh[kx:, :kx] = Z[kx:, :kx]
// (Z = L^-1 H, rows >= kx), Hh[:kx, kx:] = its transpose.
__global__ void rr_assemble_kernel(int s, int kx, const double* __restrict__ H, const double* __restrict__ Z,
                                   double* __restrict__ Hh, int ld) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl)
  const size_t total = (size_t)s * kx;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % s), j = (int)(e / s);  // column j < kx, row i
    if (i < kx) {
      Hh[IDX(i, j, ld)] = H[IDX(i, j, ld)];
    } else {
      const double z = Z[IDX(i, j, ld)];
      Hh[IDX(i, j, ld)] = z;
      Hh[IDX(j, i, ld)] = z;
    }
  }
}

// Cholesky-QR conditioning guard (reading R44): the pivot rule (R20) bounds 1 / L_jj but not the
// growth of the triangular inverse; a direction block whose L^-1 has an entry with
// |L^-1_ij|^2 > thresh (unit-norm directions: cond(G) >~ thresh, the caller passes 1e8) is treated
// like a failing pivot at row i, the direction nearly dependent on the ones before it, so the
// caller drops it (R41).
// Only sets *status when the Cholesky succeeded. Key / counter live at status[16..20] (reset by
// rr_prep_kernel); the last block to finish decides.
__global__ void linv_growth_kernel(int t, const double* __restrict__ Li, int ld, double thresh, int* status) {
  __shared__ unsigned long long wk[32];
  __shared__ bool last;
  unsigned long long* key = (unsigned long long*)(status + 16);
  unsigned* counter = (unsigned*)(status + 20);
  unsigned long long best = 0;
  const size_t total = (size_t)t * t;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % t), j = (int)(e / t);
    if (i >= j) {
      const float v = (float)fabs(Li[IDX(i, j, ld)]);
      const unsigned long long k = ((unsigned long long)__float_as_uint(v) << 32) | (unsigned)i;
      best = k > best ? k : best;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y > best ? y : best;
  }
  if ((threadIdx.x & 31) == 0) wk[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = wk[w] > best ? wk[w] : best;
    atomicMax(key, best);
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const unsigned long long k = atomicAdd(key, 0ull);
    const double v = (double)__uint_as_float((unsigned)(k >> 32));
    if (*status == 0 && !(v * v <= thresh)) *status = (int)(k & 0xffffffffu) + 1;
  }
}

// ---------------------------------------------------------------- a6 Cholesky (one CTA)
// In place on the lower triangle of G (s x s, ld). Fails (status = j+1) when a pivot is
// <= fail_rel * max diag(G) (R20). Upper triangle is zeroed on success.
template <int NT>
__global__ void __launch_bounds__(NT) cholesky_kernel(int s, double* __restrict__ G, int ld, double fail_rel,
                                                      int* __restrict__ status) {
  __shared__ double red[32];
  __shared__ double sh_ljj;
  __shared__ int sh_fail;
  double mx = 0.0;
  for (int i = threadIdx.x; i < s; i += NT) mx = fmax(mx, G[IDX(i, i, ld)]);
  // max reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < NT / 32; ++w) m = fmax(m, red[w]);
    red[0] = m;
    sh_fail = 0;
  }
  __syncthreads();
  const double floor_ = fail_rel * red[0];
  for (int j = 0; j < s; ++j) {
    if (threadIdx.x == 0) {
      double d = G[IDX(j, j, ld)];
      if (!(d > floor_)) {
        sh_fail = j + 1;
      } else {
        sh_ljj = sqrt(d);
        G[IDX(j, j, ld)] = sh_ljj;
      }
    }
    __syncthreads();
    if (sh_fail) break;
    double inv = 1.0 / sh_ljj;
    for (int i = j + 1 + threadIdx.x; i < s; i += NT) G[IDX(i, j, ld)] *= inv;
    __syncthreads();
    // trailing update of the lower triangle: G[i][k] -= L[i][j] L[k][j], j < k <= i
    int rem = s - j - 1;
    int64_t cnt = (int64_t)rem * (rem + 1) / 2;
    for (int64_t e = threadIdx.x; e < cnt; e += NT) {
      // column-wise enumeration of the lower triangle of the trailing (rem x rem) block
      int k = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);  // row of packed upper index
      // map e -> (kk, ii) with kk <= ii over a triangle: use k as the "column" of length rem-k
      // simple robust decode: walk from estimate
      int64_t base = (int64_t)k * (k + 1) / 2;
      while (base > e) { --k; base = (int64_t)k * (k + 1) / 2; }
      while ((int64_t)(k + 1) * (k + 2) / 2 <= e) { ++k; base = (int64_t)k * (k + 1) / 2; }
      int ii = k, kk = (int)(e - base);  // 0 <= kk <= ii < rem
      int gi = j + 1 + ii, gk = j + 1 + kk;
      G[IDX(gi, gk, ld)] -= G[IDX(gi, j, ld)] * G[IDX(gk, j, ld)];
    }
    __syncthreads();
  }
  __syncthreads();
  if (threadIdx.x == 0) *status = sh_fail;
  if (!sh_fail) {
    for (int e = threadIdx.x; e < s * s; e += NT) {
      int i = e % s, k = e / s;
      if (i < k) G[IDX(i, k, ld)] = 0.0;
    }
  }
}

// Linv = L^-1 (lower triangular), one warp per column j: x = L^-1 e_j by forward substitution.
__global__ void trinv_kernel(int s, const double* __restrict__ L, int ldl, double* __restrict__ Li, int ldi) {
  int warps = (blockDim.x >> 5) * gridDim.x;
  int lane = threadIdx.x & 31;
  for (int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < s; j += warps) {
    for (int i = lane; i < j; i += 32) Li[IDX(i, j, ldi)] = 0.0;
    for (int i = j; i < s; ++i) {
      double acc = 0.0;
      for (int k = j + lane; k < i; k += 32) acc += L[IDX(i, k, ldl)] * Li[IDX(k, j, ldi)];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) Li[IDX(i, j, ldi)] = ((i == j ? 1.0 : 0.0) - acc) / L[IDX(i, i, ldl)];
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------- a7 / a13 Jacobi
// Parallel-order (round-robin "circle method") two-sided Jacobi. N = s rounded up to even;
// a zero row/column pads odd s (its rotations never trigger). Round r pairs
//   k = 0: (r, N-1);  k >= 1: ((r + k) mod (N-1), (r - k) mod (N-1)),
// all N/2 rotations of a round are disjoint, so the 2x2 blocks (pair k1 x pair k2) of
// J^T A J update independently; the annihilated diagonal blocks are set exactly
// (a_pp - t a_pq, a_qq + t a_pq, 0) as in GvL §8.5.2. Skip test as in the oracle (R-J1):
//   |a_pq| <= u sqrt(|a_pp a_qq|) or |a_pq| <= u ||A||_F / s; stop after a rotation-free sweep.
__device__ __forceinline__ void rr_pair(int r, int k, int N, int& p, int& q) {
  int a, b;
  if (k == 0) {
    a = r; b = N - 1;
  } else {
    a = (r + k) % (N - 1);
    b = (r - k + (N - 1)) % (N - 1);
  }
  p = min(a, b); q = max(a, b);
}

constexpr int JAC_SMEM_MAX = 112;

// One CTA; A (s x s, lda) symmetric input; outputs w (s, unsorted) and V (s x s, ldv).
// info[0] = sweeps performed (-1: no convergence within max_sweeps).
// Each thread owns a fixed set of (pair-slot k1 <= pair-slot k2) blocks (decoded once) and a
// fixed set of (row, pair-slot) entries of V; per round only the rotation parameters change.
// The sweeps, on shared memory sm (2 N (N + 1) doubles): on return the eigenvalues are on the
// diagonal of M = sm (ld N + 1) and the eigenvectors are the columns of Q = sm + N (N + 1);
// returns the sweeps performed (-1: no convergence within max_sweeps).
template <int NT>
__device__ int jacobi_smem_core(int s, const double* __restrict__ A, int lda, double* sm, int max_sweeps) {
  constexpr int HM = JAC_SMEM_MAX / 2;
  constexpr int MAXB = (HM * (HM + 1) / 2 + NT - 1) / NT;
  const int N = s + (s & 1);
  const int H = N / 2;
  const int L = N + 1;     // odd leading dimension: column-strided accesses hit distinct banks
  double* M = sm;          // N x N (col-major, ld L)
  double* Q = sm + N * L;  // N x N (ld L)
  __shared__ double c_[HM], s_[HM], t_[HM];
  __shared__ int p_[HM], q_[HM], act_[HM];
  __shared__ double red[32];
  __shared__ int rot;
  double fro = 0.0;
  for (int e = threadIdx.x; e < N * N; e += NT) {
    int i = e % N, j = e / N;
    double v = 0.0;
    if (i < s && j < s) v = 0.5 * (A[IDX(i, j, lda)] + A[IDX(j, i, lda)]);
    M[i + j * L] = v;
    Q[i + j * L] = (i == j) ? 1.0 : 0.0;
    fro += v * v;
  }
  fro = sqrt(block_sum<NT>(fro, red));
  const double afloor = PSD_U * fro;  // absolute floor u ||A||_F (R39)
  // fixed block ownership
  const int nb = H * (H + 1) / 2;
  int bk1[MAXB], bk2[MAXB];
  int myb = 0;
#pragma unroll
  for (int j = 0; j < MAXB; ++j) {
    int b = threadIdx.x + j * NT;
    bk1[j] = 0; bk2[j] = 0;
    if (b < nb) {
      int r = 0, base = 0;
      while (base + (H - r) <= b) { base += H - r; ++r; }
      bk1[j] = r; bk2[j] = r + (b - base);
      myb = j + 1;
    }
  }
  int sweep = 0;
  bool done = (N <= 1);
  while (!done && sweep < max_sweeps) {
    if (threadIdx.x == 0) rot = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      for (int k = threadIdx.x; k < H; k += NT) {
        int p, q;
        rr_pair(r, k, N, p, q);
        double app = M[p + p * L], aqq = M[q + q * L], apq = M[p + q * L];
        int a = !(fabs(apq) <= PSD_U * sqrt(fabs(app) * fabs(aqq)) || fabs(apq) <= afloor);
        double c = 1.0, sn = 0.0, t = 0.0;
        if (a) schur2(app, apq, aqq, c, sn, t);
        p_[k] = p; q_[k] = q; c_[k] = c; s_[k] = sn; t_[k] = t; act_[k] = a;
        if (a) rot = 1;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < MAXB; ++j) {
        if (j >= myb) break;
        int k1 = bk1[j], k2 = bk2[j];
        int a1 = act_[k1], a2 = act_[k2];
        if (!a1 && !a2) continue;
        int p1 = p_[k1], q1 = q_[k1];
        if (k1 == k2) {
          double apq = M[p1 + q1 * L], t = t_[k1];
          M[p1 + p1 * L] -= t * apq;
          M[q1 + q1 * L] += t * apq;
          M[p1 + q1 * L] = 0.0; M[q1 + p1 * L] = 0.0;
          continue;
        }
        int p2 = p_[k2], q2 = q_[k2];
        double c1 = c_[k1], s1 = s_[k1], c2 = c_[k2], s2 = s_[k2];
        double b00 = M[p1 + p2 * L], b01 = M[p1 + q2 * L], b10 = M[q1 + p2 * L], b11 = M[q1 + q2 * L];
        double x00 = c1 * b00 - s1 * b10, x01 = c1 * b01 - s1 * b11;
        double x10 = s1 * b00 + c1 * b10, x11 = s1 * b01 + c1 * b11;
        double y00 = c2 * x00 - s2 * x01, y01 = s2 * x00 + c2 * x01;
        double y10 = c2 * x10 - s2 * x11, y11 = s2 * x10 + c2 * x11;
        M[p1 + p2 * L] = y00; M[p1 + q2 * L] = y01; M[q1 + p2 * L] = y10; M[q1 + q2 * L] = y11;
        M[p2 + p1 * L] = y00; M[q2 + p1 * L] = y01; M[p2 + q1 * L] = y10; M[q2 + q1 * L] = y11;
      }
      // V <- V J
      for (int e = threadIdx.x; e < N * H; e += NT) {
        int k = e / N;
        if (!act_[k]) continue;
        int i = e - k * N;
        int p = p_[k], q = q_[k];
        double c = c_[k], sn = s_[k];
        double vp = Q[i + p * L], vq = Q[i + q * L];
        Q[i + p * L] = c * vp - sn * vq;
        Q[i + q * L] = sn * vp + c * vq;
      }
      __syncthreads();
    }
    ++sweep;
    done = (rot == 0);
    __syncthreads();
  }
  return done ? sweep : -1;
}

template <int NT>
__global__ void __launch_bounds__(NT) jacobi_smem_kernel(int s, const double* __restrict__ A, int lda,
                                                         double* __restrict__ w, double* __restrict__ V, int ldv,
                                                         int max_sweeps, int* __restrict__ info) {
  extern __shared__ __align__(16) double sm[];
  const int sweeps = jacobi_smem_core<NT>(s, A, lda, sm, max_sweeps);
  const int N = s + (s & 1), L = N + 1;
  const double* M = sm;
  const double* Q = sm + N * L;
  for (int i = threadIdx.x; i < s; i += NT) w[i] = M[i + i * L];
  for (int e = threadIdx.x; e < s * s; e += NT) {
    int i = e % s, j = e / s;
    V[IDX(i, j, ldv)] = Q[i + j * L];
  }
  if (threadIdx.x == 0) { info[0] = sweeps; info[1] = 0; }
}

// ---------------------------------------------------------------- f4: many tiny cone blocks
// One CTA per block (n <= JAC_SMEM_MAX): the exact projection by the one-CTA Jacobi above, then
// Pi = sum_{lambda > 0} lambda v v^T, or A - sum_{lambda < 0} lambda v v^T when fewer eigenvalues are
// negative (the one-sided rule of PAPER.md:505 on the exact spectrum), each entry (i <= j) computed
// once and mirrored. npos[b] = number of positive eigenvalues (-1: no convergence).
struct TinyBlock {
  const double* A;
  double* Pi;
  int n, lda, ldpi, pad;
};
template <int NT>
__global__ void __launch_bounds__(NT) tiny_project_kernel(const TinyBlock* __restrict__ blocks, int max_sweeps,
                                                          int* __restrict__ npos) {
  extern __shared__ __align__(16) double sm[];
  const TinyBlock bk = blocks[blockIdx.x];
  const int s = bk.n;
  if (s <= 0) return;
  const int sweeps = jacobi_smem_core<NT>(s, bk.A, bk.lda, sm, max_sweeps);
  const int N = s + (s & 1), L = N + 1;
  const double* M = sm;
  const double* Q = sm + N * L;
  __shared__ int cnt[2];
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < s; k += NT) {
    const double lk = M[k + k * L];
    if (lk > 0.0) atomicAdd(&cnt[0], 1);
    if (lk < 0.0) atomicAdd(&cnt[1], 1);
  }
  __syncthreads();
  const bool pos_side = cnt[0] <= cnt[1];
  for (int e = threadIdx.x; e < s * s; e += NT) {
    const int i = e % s, j = e / s;
    if (i > j) continue;
    double acc = 0.0;
    for (int k = 0; k < s; ++k) {
      const double lk = M[k + k * L];
      if (pos_side ? (lk > 0.0) : (lk < 0.0)) acc = fma(lk * Q[i + k * L], Q[j + k * L], acc);
    }
    const double v = pos_side ? acc : 0.5 * (bk.A[IDX(i, j, bk.lda)] + bk.A[IDX(j, i, bk.lda)]) - acc;
    bk.Pi[IDX(i, j, bk.ldpi)] = v;
    bk.Pi[IDX(j, i, bk.ldpi)] = v;
  }
  if (threadIdx.x == 0 && npos) npos[blockIdx.x] = sweeps < 0 ? -1 : cnt[0];
}

// Cooperative multi-CTA variant for s > JAC_SMEM_MAX: the matrix is double-buffered in
// global memory (Ma -> Mb each round); each thread recomputes the two rotations of its
// block from the read buffer, so one grid barrier per round suffices. Only blocks k1 <= k2
// are computed and mirrored (exact symmetry). Q is updated in place (disjoint columns).
// counters[max_sweeps+1] are zeroed by the host; afloor = afl_scale * ||A||_F (*d_fro).
__device__ __forceinline__ void decode_upper(int64_t b, int H, int& k1, int& k2) {
  float hh = 2.0f * H + 1.0f;
  int r = (int)((hh - sqrtf(fmaxf(hh * hh - 8.0f * (float)b, 0.0f))) * 0.5f);
  r = max(0, min(r, H - 1));
  int64_t base = (int64_t)r * H - (int64_t)r * (r - 1) / 2;
  while (r > 0 && base > b) { --r; base = (int64_t)r * H - (int64_t)r * (r - 1) / 2; }
  while (base + (H - r) <= b) { base += H - r; ++r; }
  k1 = r;
  k2 = r + (int)(b - base);
}

__device__ __forceinline__ int jac_active(double app, double aqq, double apq, double afloor) {
  return !(fabs(apq) <= PSD_U * sqrt(fabs(app) * fabs(aqq)) || fabs(apq) <= afloor);
}

// One CTA per SM, one grid barrier per round. At the start of a round every CTA computes the
// rotation parameters of all N/2 pairs from the read buffer into shared memory (redundant
// across CTAs, no extra barrier), then updates its share of the k1 <= k2 blocks into the
// write buffer (mirrored) and its share of V's column pairs in place.
constexpr int JAC_COOP_MAXH = 1280;
__global__ void __launch_bounds__(512) jacobi_coop_kernel(int s, int N, double* __restrict__ Ma,
                                                          double* __restrict__ Mb, double* __restrict__ Q,
                                                          const double* __restrict__ d_fro, double afl_scale,
                                                          int max_sweeps, int* __restrict__ counters,
                                                          int* __restrict__ info) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sc[JAC_COOP_MAXH], ss[JAC_COOP_MAXH], st_[JAC_COOP_MAXH], sapq[JAC_COOP_MAXH];
  __shared__ unsigned char sact[JAC_COOP_MAXH];
  const int H = N / 2;
  const int64_t nb = (int64_t)H * H;  // all (k1, k2), k1 fastest: coalesced rows p1 = r + k1
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
  const double afloor = afl_scale * d_fro[0];
  double* cur = Ma;
  double* nxt = Mb;
  int sweep = 0;
  bool done = (N <= 1);
  while (!done && sweep < max_sweeps) {
    for (int r = 0; r < N - 1; ++r) {
      int cnt = 0;
      for (int k = threadIdx.x; k < H; k += blockDim.x) {
        int p, q;
        rr_pair(r, k, N, p, q);
        double app = cur[IDX(p, p, N)], aqq = cur[IDX(q, q, N)], apq = cur[IDX(p, q, N)];
        int a = jac_active(app, aqq, apq, afloor);
        double c = 1.0, sn = 0.0, t = 0.0;
        if (a) schur2(app, apq, aqq, c, sn, t);
        sc[k] = c; ss[k] = sn; st_[k] = t; sapq[k] = apq; sact[k] = (unsigned char)a;
        cnt += a;
      }
      if (blockIdx.x == 0 && cnt) atomicAdd(&counters[sweep], cnt);
      __syncthreads();
      for (int64_t b = gtid; b < nb; b += gsz) {
        int k1 = (int)(b % H), k2 = (int)(b / H);
        int p1, q1;
        rr_pair(r, k1, N, p1, q1);
        if (k1 == k2) {
          double app = cur[IDX(p1, p1, N)], aqq = cur[IDX(q1, q1, N)], apq = sapq[k1];
          if (sact[k1]) {
            double t = st_[k1];
            nxt[IDX(p1, p1, N)] = app - t * apq;
            nxt[IDX(q1, q1, N)] = aqq + t * apq;
            nxt[IDX(p1, q1, N)] = 0.0;
            nxt[IDX(q1, p1, N)] = 0.0;
          } else {
            nxt[IDX(p1, p1, N)] = app;
            nxt[IDX(q1, q1, N)] = aqq;
            nxt[IDX(p1, q1, N)] = apq;
            nxt[IDX(q1, p1, N)] = apq;
          }
          continue;
        }
        int p2, q2;
        rr_pair(r, k2, N, p2, q2);
        double c1 = sc[k1], s1 = ss[k1], c2 = sc[k2], s2 = ss[k2];
        double b00 = cur[IDX(p1, p2, N)], b01 = cur[IDX(p1, q2, N)], b10 = cur[IDX(q1, p2, N)],
               b11 = cur[IDX(q1, q2, N)];
        double x00 = c1 * b00 - s1 * b10, x01 = c1 * b01 - s1 * b11;
        double x10 = s1 * b00 + c1 * b10, x11 = s1 * b01 + c1 * b11;
        nxt[IDX(p1, p2, N)] = c2 * x00 - s2 * x01;
        nxt[IDX(p1, q2, N)] = s2 * x00 + c2 * x01;
        nxt[IDX(q1, p2, N)] = c2 * x10 - s2 * x11;
        nxt[IDX(q1, q2, N)] = s2 * x10 + c2 * x11;
      }
      for (int64_t e = gtid; e < (int64_t)N * H; e += gsz) {
        int i = (int)(e % N), k = (int)(e / N);
        if (!sact[k]) continue;
        int p, q;
        rr_pair(r, k, N, p, q);
        double c = sc[k], sn = ss[k];
        double vp = Q[IDX(i, p, N)], vq = Q[IDX(i, q, N)];
        Q[IDX(i, p, N)] = c * vp - sn * vq;
        Q[IDX(i, q, N)] = sn * vp + c * vq;
      }
      grid.sync();
      double* tmp = cur; cur = nxt; nxt = tmp;
    }
    done = (*(volatile int*)&counters[sweep] == 0);
    ++sweep;
  }
  if (gtid == 0) {
    info[0] = done ? sweep : -1;
    info[1] = (cur == Ma) ? 0 : 1;  // which buffer holds the result
  }
}

// Cluster variant: one thread-block cluster of CS CTAs (CS <= 16, non-portable) runs the whole
// Jacobi; the matrix stays in global memory (L2-resident) double-buffered, reads bypass L1
// (ld.global.cg), and rounds are separated by the cluster barrier (release/acquire), which
// is an order of magnitude cheaper than a grid-wide barrier. Every CTA computes all rotation
// parameters of the round itself (identical inputs -> identical decisions, no exchange).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

constexpr int JAC_CL_MAXH = 1280;
__global__ void __launch_bounds__(1024) jacobi_cluster_kernel(int s, int N, double* __restrict__ Ma,
                                                              double* __restrict__ Mb, double* __restrict__ Q,
                                                              const double* __restrict__ d_fro, double afl_scale,
                                                              int max_sweeps, int* __restrict__ info) {
  __shared__ double sc[JAC_CL_MAXH], ss[JAC_CL_MAXH], st_[JAC_CL_MAXH], sapq[JAC_CL_MAXH];
  __shared__ unsigned char sact[JAC_CL_MAXH];
  __shared__ int srot;
  const int H = N / 2;
  const int CS = (int)gridDim.x;  // the grid is exactly one cluster
  const int64_t nb = (int64_t)H * H;
  const int64_t gtid = (int64_t)cluster_ctarank() * blockDim.x + threadIdx.x;
  const int64_t gsz = (int64_t)CS * blockDim.x;
  const double afloor = afl_scale * __ldcg(d_fro);
  double* cur = Ma;
  double* nxt = Mb;
  int sweep = 0;
  bool done = (N <= 1);
  while (!done && sweep < max_sweeps) {
    if (threadIdx.x == 0) srot = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      int any = 0;
      for (int k = threadIdx.x; k < H; k += blockDim.x) {
        int p, q;
        rr_pair(r, k, N, p, q);
        double app = __ldcg(cur + IDX(p, p, N)), aqq = __ldcg(cur + IDX(q, q, N)), apq = __ldcg(cur + IDX(p, q, N));
        int a = jac_active(app, aqq, apq, afloor);
        double c = 1.0, sn = 0.0, t = 0.0;
        if (a) schur2(app, apq, aqq, c, sn, t);
        sc[k] = c; ss[k] = sn; st_[k] = t; sapq[k] = apq; sact[k] = (unsigned char)a;
        any |= a;
      }
      if (any) srot = 1;
      __syncthreads();
      for (int64_t b = gtid; b < nb; b += gsz) {
        int k1 = (int)(b % H), k2 = (int)(b / H);
        int p1, q1;
        rr_pair(r, k1, N, p1, q1);
        if (k1 == k2) {
          double app = __ldcg(cur + IDX(p1, p1, N)), aqq = __ldcg(cur + IDX(q1, q1, N)), apq = sapq[k1];
          if (sact[k1]) {
            double t = st_[k1];
            nxt[IDX(p1, p1, N)] = app - t * apq;
            nxt[IDX(q1, q1, N)] = aqq + t * apq;
            nxt[IDX(p1, q1, N)] = 0.0;
            nxt[IDX(q1, p1, N)] = 0.0;
          } else {
            nxt[IDX(p1, p1, N)] = app;
            nxt[IDX(q1, q1, N)] = aqq;
            nxt[IDX(p1, q1, N)] = apq;
            nxt[IDX(q1, p1, N)] = apq;
          }
          continue;
        }
        int p2, q2;
        rr_pair(r, k2, N, p2, q2);
        double c1 = sc[k1], s1 = ss[k1], c2 = sc[k2], s2 = ss[k2];
        double b00 = __ldcg(cur + IDX(p1, p2, N)), b01 = __ldcg(cur + IDX(p1, q2, N));
        double b10 = __ldcg(cur + IDX(q1, p2, N)), b11 = __ldcg(cur + IDX(q1, q2, N));
        double x00 = c1 * b00 - s1 * b10, x01 = c1 * b01 - s1 * b11;
        double x10 = s1 * b00 + c1 * b10, x11 = s1 * b01 + c1 * b11;
        nxt[IDX(p1, p2, N)] = c2 * x00 - s2 * x01;
        nxt[IDX(p1, q2, N)] = s2 * x00 + c2 * x01;
        nxt[IDX(q1, p2, N)] = c2 * x10 - s2 * x11;
        nxt[IDX(q1, q2, N)] = s2 * x10 + c2 * x11;
      }
      for (int64_t e = gtid; e < (int64_t)N * H; e += gsz) {
        int k = (int)(e / N);
        if (!sact[k]) continue;
        int i = (int)(e - (int64_t)k * N);
        int p, q;
        rr_pair(r, k, N, p, q);
        double c = sc[k], sn = ss[k];
        double vp = __ldcg(Q + IDX(i, p, N)), vq = __ldcg(Q + IDX(i, q, N));
        Q[IDX(i, p, N)] = c * vp - sn * vq;
        Q[IDX(i, q, N)] = sn * vp + c * vq;
      }
      cluster_sync_all();
      double* tmp = cur; cur = nxt; nxt = tmp;
    }
    __syncthreads();
    done = (srot == 0);
    ++sweep;
    __syncthreads();
  }
  if (gtid == 0) {
    info[0] = done ? sweep : -1;
    info[1] = (cur == Ma) ? 0 : 1;
  }
}

// load symmetric (s x s, lda) into an N x N zero-padded buffer; Q = I
__global__ void jacobi_prep_kernel(int s, int N, const double* __restrict__ A, int lda, double* __restrict__ M,
                                   double* __restrict__ Q) {
  int64_t total = (int64_t)N * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % N), j = (int)(e / N);
    double v = 0.0;
    if (i < s && j < s) v = 0.5 * (A[IDX(i, j, lda)] + A[IDX(j, i, lda)]);
    M[e] = v;
    Q[e] = (i == j) ? 1.0 : 0.0;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) fro_kernel(int64_t count, const double* __restrict__ M, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t e = threadIdx.x; e < count; e += NT) acc += M[e] * M[e];
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) out[0] = sqrt(acc);
}

// extract diag / V (s x s) from the padded Jacobi buffers (info[1] selects Ma or Mb)
__global__ void jacobi_extract_kernel(int s, int N, const double* __restrict__ Ma, const double* __restrict__ Mb,
                                      const double* __restrict__ Q, const int* __restrict__ info,
                                      double* __restrict__ w, double* __restrict__ V, int ldv) {
  const double* M = info[1] ? Mb : Ma;
  int64_t total = (int64_t)s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % s), j = (int)(e / s);
    V[IDX(i, j, ldv)] = Q[IDX(i, j, N)];
    if (i == j) w[i] = M[IDX(i, i, N)];
  }
}

// rank sort, descending, ties by index (R21): order[rank] = i, wsorted[rank] = w[i]
__global__ void sort_desc_kernel(int s, const double* __restrict__ w, int* __restrict__ order,
                                 double* __restrict__ wsorted) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s; i += gridDim.x * blockDim.x) {
    double wi = w[i];
    int rank = 0;
    for (int j = 0; j < s; ++j) {
      double wj = w[j];
      rank += (wj > wi) || (wj == wi && j < i);
    }
    order[rank] = i;
    wsorted[rank] = wi;
  }
}

// ||H - diag(theta)||_F over an s x s block (bound term of hard locking, R36)
template <int NT>
__global__ void __launch_bounds__(NT) offdiag_fro_kernel(int s, const double* __restrict__ H, int ld,
                                                         const double* __restrict__ theta, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)s * s; e += NT) {
    int i = (int)(e % s), j = (int)(e / s);
    double v = H[IDX(i, j, ld)] - (i == j ? theta[i] : 0.0);
    acc += v * v;
  }
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) out[0] = sqrt(acc);
}

// Certification defects (a10, R16/R36): out = sqrt(sum over (i, j) of (H_ij - delta_ij d_i)^2) with
// d_i = diag[i] (or dconst when diag is NULL), restricted to the pairs with mask[i] > 0 and
// mask[j] > 0 when mask is given (the positive block of a DIRECT eigendecomposition).
template <int NT>
__global__ void __launch_bounds__(NT) defect_fro_kernel(int s, const double* __restrict__ H, int ld,
                                                        const double* __restrict__ diag, double dconst,
                                                        const double* __restrict__ mask, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)s * s; e += NT) {
    int i = (int)(e % s), j = (int)(e / s);
    if (mask && !(mask[i] > 0.0 && mask[j] > 0.0)) continue;
    double v = H[IDX(i, j, ld)] - (i == j ? (diag ? diag[i] : dconst) : 0.0);
    acc += v * v;
  }
  acc = block_sum<NT>(acc, red);
  if (threadIdx.x == 0) out[0] = sqrt(acc);
}

// dense symmetric tridiagonal T (k x k, ld) from its diagonal a and off-diagonal b (f2 Lanczos matrix)
__global__ void tridiag_dense_kernel(int k, const double* __restrict__ a, const double* __restrict__ b,
                                     double* __restrict__ T, int ld) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % k), j = (int)(e / k);
    T[IDX(i, j, ld)] = i == j ? a[i] : ((i == j + 1 || j == i + 1) ? b[min(i, j)] : 0.0);
  }
}

__global__ void count_pos_kernel(int s, const double* __restrict__ w, int* __restrict__ out) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int c = 0;
  for (int i = threadIdx.x; i < s; i += blockDim.x) c += w[i] > 0.0;
  atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) *out = cnt;
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

// swap columns i and j of an n-row column-major matrix
__global__ void swap_cols_kernel(int n, double* __restrict__ X, int ld, int i, int j) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double a = X[IDX(r, i, ld)];
    X[IDX(r, i, ld)] = X[IDX(r, j, ld)];
    X[IDX(r, j, ld)] = a;
  }
}

__global__ void fill_identity_kernel(int k, double* __restrict__ M, int ld) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) M[IDX(i, i, ld)] = 1.0;
}

// P = (P + P^T)/2 in place (n x n, ld)
__global__ void symmetrize_kernel(int n, double* __restrict__ P, int ld) {
  int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % n), j = (int)(e / n);
    if (i >= j) continue;
    double a = P[IDX(i, j, ld)], b = P[IDX(j, i, ld)];
    double v = 0.5 * (a + b);
    P[IDX(i, j, ld)] = v;
    P[IDX(j, i, ld)] = v;
  }
}

// non-finite scan (E_NONFINITE, R-first pass): flag[0] |= 1 if any entry is inf/nan
// rows x cols block (rows = n, cols = n unsharded; the local row block in the row-sharded mode)
__global__ void nonfinite_kernel(int rows, int cols, const double* __restrict__ A, int lda, int* __restrict__ flag) {
  int64_t total = (int64_t)rows * cols;
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % rows), j = (int)(e / rows);
    if (!isfinite(A[IDX(i, j, lda)])) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Frobenius norm partials: out[block] = sum of squares of its slice (second pass on host order)
__global__ void fro_partial_kernel(int rows, int cols, const double* __restrict__ A, int lda, double* __restrict__ out) {
  __shared__ double red[32];
  int64_t total = (int64_t)rows * cols;
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % rows), j = (int)(e / rows);
    double v = A[IDX(i, j, lda)];
    acc += v * v;
  }
  acc = block_sum<256>(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

}  // namespace psd

namespace psd {
// ---------------------------------------------------------------- f1/f3: approximate ADMM, diagonal SDP
// Alg. 1 on  min <Q, X>  s.t.  X_ii = b_i (i with w_i = 1),  X in S+  written as
// A x = z, z in C with x = vec(X), A = [D_w; I] (D_w extracts the constrained diagonal entries),
// C = {b}^w x S+, P = 0 (MaxCut: b = 1, w = 1; f3's infeasible toys: some b_i < 0, or w = 0 with an
// indefinite Q). A^T A is diagonal (1 + w_i on the diagonal entries, 1 elsewhere), so line 3's KKT
// solve is elementwise. Readings (R43): line 5 projects alpha z~ + (1 - alpha) z^k + y^k / rho and
// line 6 updates y with that same relaxed z-hat (COSMO / Stellato 2017 form).
// b, w == nullptr mean b = 1, w = 1.
//
// Step 1 (lines 3-4 and the projection input of line 5): for every entry
//   X~ = (sigma X - Q + rho Zp - Yp + [i = j] w_i (rho b_i - ye_i)) / (sigma + rho (1 + [i = j] w_i))
//   X  <- alpha X~ + (1 - alpha) X;   Zh = alpha X~ + (1 - alpha) Zp;   V = Zh + Yp / rho
//   zeh_i = alpha X~_ii + (1 - alpha) b_i                  (z_eq = b after every projection)
__global__ void admm_maxcut_step1_kernel(int n, double* __restrict__ X, const double* __restrict__ Zp,
                                         const double* __restrict__ Yp, const double* __restrict__ ye,
                                         const double* __restrict__ Q, double sigma, double rho, double alpha,
                                         double* __restrict__ Zh, double* __restrict__ V, double* __restrict__ zeh,
                                         int ld, const double* __restrict__ bv, const double* __restrict__ wv) {
  const size_t total = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    const size_t o = IDX(i, j, ld);
    const bool dg = i == j;
    const double bi = (dg && bv) ? bv[i] : 1.0;
    const double wi = dg ? (wv ? wv[i] : 1.0) : 0.0;
    double xt = sigma * X[o] - Q[o] + rho * Zp[o] - Yp[o];
    if (dg) xt += wi * (rho * bi - ye[i]);
    xt /= sigma + rho * (1.0 + wi);
    X[o] = alpha * xt + (1.0 - alpha) * X[o];
    const double zh = alpha * xt + (1.0 - alpha) * Zp[o];
    Zh[o] = zh;
    V[o] = zh + Yp[o] / rho;
    if (dg) zeh[i] = alpha * xt + (1.0 - alpha) * bi;
  }
}

// Step 2 (line 6) and residual maxima (COSMO termination, PAPER.md:500 footnote; R33 absolute):
//   Yp <- Yp + rho (Zh - Zp),  ye <- ye + rho (zeh - b) (constrained i; ye = 0 elsewhere)
//   res[0] = max |X - Zp| (primal, PSD block), res[1] = max |X_ii - b_i| over w_i = 1 (equalities),
//   res[2] = max |Q + Yp + Diag(w ye)| (dual: P x + q + A^T y)
__global__ void admm_maxcut_step2_kernel(int n, const double* __restrict__ X, const double* __restrict__ Zp,
                                         const double* __restrict__ Zh, double* __restrict__ Yp,
                                         double* __restrict__ ye, const double* __restrict__ zeh,
                                         const double* __restrict__ Q, double rho, int ld,
                                         unsigned long long* __restrict__ res, const double* __restrict__ bv,
                                         const double* __restrict__ wv) {
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
  const size_t total = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    const size_t o = IDX(i, j, ld);
    const double yp = Yp[o] + rho * (Zh[o] - Zp[o]);
    Yp[o] = yp;
    r0 = fmax(r0, fabs(X[o] - Zp[o]));
    double dres = Q[o] + yp;
    if (i == j) {
      const double bi = bv ? bv[i] : 1.0, wi = wv ? wv[i] : 1.0;
      if (wi != 0.0) {
        const double y = ye[i] + rho * (zeh[i] - bi);
        ye[i] = y;  // each diagonal entry is visited by exactly one thread
        dres += y;
        r1 = fmax(r1, fabs(X[o] - bi));
      }
    }
    r2 = fmax(r2, fabs(dres));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r0 = fmax(r0, __shfl_xor_sync(0xffffffffu, r0, o));
    r1 = fmax(r1, __shfl_xor_sync(0xffffffffu, r1, o));
    r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (r0 > 0.0) atomicMax(res + 0, (unsigned long long)__double_as_longlong(r0));
    if (r1 > 0.0) atomicMax(res + 1, (unsigned long long)__double_as_longlong(r1));
    if (r2 > 0.0) atomicMax(res + 2, (unsigned long long)__double_as_longlong(r2));
  }
}
// f3 (Theorem 1; reading R49): the certificate terms of two successive ADMM
// iterates in one pass. Per block, partial sums (fixed order) of
//   0 ||dX||_F^2, 1 ||w dye||^2, 2 ||dYp||_F^2, 3 b . (w dye), 4 <Q, dX>, 5 ||w diag(dX)||^2
// and the maximum 6 max |dYp + Diag(w dye)|, with dX = X - X0, dye = ye - ye0, dYp = Yp - Yp0; also
// writes sym(dYp) and -sym(dX) (the arguments of the two PSD-part distances).
constexpr int CERT_TERMS = 7;
__global__ void admm_cert_partial_kernel(int n, const double* __restrict__ X, const double* __restrict__ X0,
                                         const double* __restrict__ ye, const double* __restrict__ ye0,
                                         const double* __restrict__ Yp, const double* __restrict__ Yp0,
                                         const double* __restrict__ Q, int ld, const double* __restrict__ bv,
                                         const double* __restrict__ wv, double* __restrict__ dYs,
                                         double* __restrict__ mdXs, double* __restrict__ part) {
  __shared__ double red[32];
  double a[CERT_TERMS] = {0, 0, 0, 0, 0, 0, 0};
  const size_t total = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    const size_t o = IDX(i, j, ld), ot = IDX(j, i, ld);
    const double dx = X[o] - X0[o], dy = Yp[o] - Yp0[o];
    dYs[o] = 0.5 * (dy + (Yp[ot] - Yp0[ot]));
    mdXs[o] = -0.5 * (dx + (X[ot] - X0[ot]));
    a[0] += dx * dx;
    a[2] += dy * dy;
    a[4] += Q[o] * dx;
    double m = dy;
    if (i == j) {
      const double wi = wv ? wv[i] : 1.0, bi = bv ? bv[i] : 1.0;
      const double dye = wi * (ye[i] - ye0[i]);
      a[1] += dye * dye;
      a[3] += bi * dye;
      a[5] += (wi * dx) * (wi * dx);
      m += dye;
    }
    a[6] = fmax(a[6], fabs(m));
  }
  for (int t = 0; t < CERT_TERMS; ++t) {
    double v = t == 6 ? a[t] : a[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = t == 6 ? fmax(v, u) : v + u;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double r = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = t == 6 ? fmax(r, red[w]) : r + red[w];
      part[(size_t)t * gridDim.x + blockIdx.x] = r;
    }
    __syncthreads();
  }
}

// fixed-order final reduction of admm_cert_partial_kernel's partials (one block)
__global__ void admm_cert_final_kernel(int nb, const double* __restrict__ part, double* __restrict__ out) {
  const int t = threadIdx.x;
  if (t >= CERT_TERMS) return;
  double r = 0.0;
  for (int b = 0; b < nb; ++b) r = t == 6 ? fmax(r, part[(size_t)t * nb + b]) : r + part[(size_t)t * nb + b];
  out[t] = r;
}

// Holds its stream until *flag >= seq (a kernel on another stream announced that it is resident)
// or timeout_ns passed; one thread.
__global__ void wait_flag_kernel(const int* __restrict__ flag, int seq, long long timeout_ns) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= seq) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if ((long long)(t1 - t0) > timeout_ns) break;
    __nanosleep(64);
  }
}

}  // namespace psd
