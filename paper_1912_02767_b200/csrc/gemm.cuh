// gemm.cuh -- fp64 DMMA GEMM for sm_100a (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
//   C[M x N] = alpha * op(A)[M x K] * op(B)[K x N] + beta * C       (all column-major)
//
// Used for every dense contraction on the path:
//   a3  block multiply   B.Z = s * A * Z          (A symmetric n x n, Z n x k)
//   a5  Gram / pencil    G = S^T S, H = S^T (BS)  (tall-skinny, split-K over n)
//   a8  rotation         X <- S C'                (n x s times s x m)
//   a11 low-rank update  Pi = beta A + (V w) V^T
// tcgen05.mma has no f64 kind, so FP64 tensor math on B200 is DMMA (measured 37.1 TF/s peak,
// profiles/peaks_fp64_r01.json). Operands are staged global->shared with cp.async (LDGSTS)
// in a STAGES-deep ring; shared layouts are padded so every 64-bit fragment load is
// bank-conflict free. Split-K partials are reduced in fixed order (deterministic).
#pragma once
#include "common.cuh"

namespace psd {

enum { OP_N = 0, OP_T = 1 };

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int WARPS_M = BM / WM;
  static constexpr int WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int MI = WM / 8;
  static constexpr int NI = WN / 8;
  // pitches (doubles): "outer x k" tiles use BK+4, "k x outer" tiles use BM/BN+4
  static constexpr int PK = BK + 4;
  static constexpr int PAM = BM + 4;
  static constexpr int PBN = BN + 4;
  static constexpr int A_ELEMS = (BM * PK > BK * PAM) ? BM * PK : BK * PAM;
  static constexpr int B_ELEMS = (BN * PK > BK * PBN) ? BN * PK : BK * PBN;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_ELEMS * sizeof(double);
};

// Load one k-tile of op(A) (BM x BK) or op(B) (BK x BN) into shared memory.
// kOuterContig: the gmem operand is contiguous along the "outer" (m or n) index.
template <int OUTER, int BK, int THREADS, bool OUTER_CONTIG, bool VEC>
__device__ __forceinline__ void load_tile(double* sm, const double* __restrict__ g, int ld, int o0,
                                          int k0, int O, int K, int tid) {
  if (OUTER_CONTIG) {
    // element (o, k) at g[o + k*ld]; smem [k][o] pitch OUTER+4
    constexpr int P = OUTER + 4;
    if (VEC) {
      constexpr int CH = BK * OUTER / 2;
      for (int c = tid; c < CH; c += THREADS) {
        int k = c / (OUTER / 2), o = (c % (OUTER / 2)) * 2;
        int go = o0 + o, gk = k0 + k;
        int valid = (gk < K) ? ((go + 1 < O) ? 2 : (go < O ? 1 : 0)) : 0;
        const double* src = g + (valid ? IDX(go, gk, ld) : 0);
        cp_async_16(sm + k * P + o, src, valid * 8);
      }
    } else {
      constexpr int CH = BK * OUTER;
      for (int c = tid; c < CH; c += THREADS) {
        int k = c / OUTER, o = c % OUTER;
        int go = o0 + o, gk = k0 + k;
        int valid = (gk < K && go < O) ? 1 : 0;
        const double* src = g + (valid ? IDX(go, gk, ld) : 0);
        cp_async_8(sm + k * P + o, src, valid * 8);
      }
    }
  } else {
    // element (o, k) at g[k + o*ld]; smem [o][k] pitch BK+4
    constexpr int P = BK + 4;
    if (VEC) {
      constexpr int CH = OUTER * BK / 2;
      for (int c = tid; c < CH; c += THREADS) {
        int o = c / (BK / 2), k = (c % (BK / 2)) * 2;
        int go = o0 + o, gk = k0 + k;
        int valid = (go < O) ? ((gk + 1 < K) ? 2 : (gk < K ? 1 : 0)) : 0;
        const double* src = g + (valid ? IDX(gk, go, ld) : 0);
        cp_async_16(sm + o * P + k, src, valid * 8);
      }
    } else {
      constexpr int CH = OUTER * BK;
      for (int c = tid; c < CH; c += THREADS) {
        int o = c / BK, k = c % BK;
        int go = o0 + o, gk = k0 + k;
        int valid = (go < O && gk < K) ? 1 : 0;
        const double* src = g + (valid ? IDX(gk, go, ld) : 0);
        cp_async_8(sm + o * P + k, src, valid * 8);
      }
    }
  }
}

// partial != nullptr: write raw accumulators to partial + z*M*N (ld = M) for split-K.
template <int OPA, int OPB, int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC>
__global__ void __launch_bounds__(GemmCfg<BM, BN, BK, WM, WN, STAGES>::THREADS)
    dgemm_kernel(int M, int N, int K, double alpha, const double* __restrict__ A, int lda,
                 const double* __restrict__ B, int ldb, double beta, double* __restrict__ C, int ldc,
                 double* __restrict__ partial, int ktiles_per_split) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % Cfg::WARPS_M, wn = warp / Cfg::WARPS_M;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KT = cdiv(K, BK);
  const int kt0 = blockIdx.z * ktiles_per_split;
  const int kt1 = min(KT, kt0 + ktiles_per_split);
  const int nkt = max(0, kt1 - kt0);

  double acc[Cfg::MI][Cfg::NI][2];
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stageA = [&](int s) { return smem + (size_t)s * Cfg::STAGE_ELEMS; };
  auto stageB = [&](int s) { return smem + (size_t)s * Cfg::STAGE_ELEMS + Cfg::A_ELEMS; };
  auto issue = [&](int s, int kt) {
    int k0 = kt * BK;
    load_tile<BM, BK, Cfg::THREADS, OPA == OP_N, VEC>(stageA(s), A, lda, m0, k0, M, K, tid);
    load_tile<BN, BK, Cfg::THREADS, OPB == OP_T, VEC>(stageB(s), B, ldb, n0, k0, N, K, tid);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) issue(s, kt0 + s);
    cp_async_commit();
  }
  const int ar = lane >> 2, ac = lane & 3;
  for (int it = 0; it < nkt; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nx = it + STAGES - 1;
      if (nx < nkt) issue(nx % STAGES, kt0 + nx);
      cp_async_commit();
    }
    const double* sA = stageA(it % STAGES);
    const double* sB = stageB(it % STAGES);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::MI], bf[Cfg::NI];
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i) {
        int m = wm * WM + i * 8 + ar, k = kk + ac;
        af[i] = (OPA == OP_N) ? sA[k * Cfg::PAM + m] : sA[m * Cfg::PK + k];
      }
#pragma unroll
      for (int j = 0; j < Cfg::NI; ++j) {
        int n = wn * WN + j * 8 + ar, k = kk + ac;
        bf[j] = (OPB == OP_T) ? sB[k * Cfg::PBN + n] : sB[n * Cfg::PK + k];
      }
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NI; ++j) dmma_884(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: accumulator (row = lane>>2, col = 2*(lane&3) + {0,1}) of each 8x8 subtile
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    int row = m0 + wm * WM + i * 8 + ar;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < Cfg::NI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int col = n0 + wn * WN + j * 8 + ac * 2 + h;
        if (col >= N) continue;
        double v = acc[i][j][h];
        if (partial) {
          partial[(size_t)blockIdx.z * M * N + IDX(row, col, M)] = v;
        } else {
          double* c = C + IDX(row, col, ldc);
          *c = (beta == 0.0) ? alpha * v : alpha * v + beta * (*c);
        }
      }
    }
  }
}

// Fixed-order (deterministic) sum of the split-K partials: grid (cdiv(M, 256), N), loads of all
// splits issued before the ordered adds.
__global__ void splitk_reduce_kernel(int M, int N, int splits, double alpha, const double* __restrict__ part,
                                     double beta, double* __restrict__ C, int ldc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see dgemm_kp_kernel
  const int row = blockIdx.x * blockDim.x + threadIdx.x, col = blockIdx.y;
  if (row >= M) return;
  const size_t total = (size_t)M * N, e = (size_t)row + (size_t)col * M;
  double s = 0.0;
  int z = 0;
  for (; z + 4 <= splits; z += 4) {
    const double p0 = __ldg(part + z * total + e), p1 = __ldg(part + (z + 1) * total + e);
    const double p2 = __ldg(part + (z + 2) * total + e), p3 = __ldg(part + (z + 3) * total + e);
    s += p0;
    s += p1;
    s += p2;
    s += p3;
  }
  for (; z < splits; ++z) s += __ldg(part + z * total + e);
  double* c = C + IDX(row, col, ldc);
  *c = (beta == 0.0) ? alpha * s : alpha * s + beta * (*c);
}

}  // namespace psd

namespace psd {

// ---------------------------------------------------------------- k-paired DMMA GEMM
// Same contract as dgemm_kernel. Shared tiles store k permuted in pairs (k, k+4) of every 8-block
// adjacent, so one LDS.128 feeds the fragments of two consecutive m8n8k4 MMAs:
//   element (o, k) of a BO x 16 tile -> s[(8 (k / 8) / 2 + (k % 4)) * P + 2 o + (k % 8) / 4]
// with pitch P = 2 BO + 4 (doubles; 2 BO + 4 = 4 mod 16 keeps the 8 lanes of each LDS.128 phase on
// distinct bank groups). Global -> shared by 8-byte cp.async (the permutation breaks 16-byte runs).
template <int BO, int THREADS, bool OUTER_CONTIG>
__device__ __forceinline__ void load_tile_kp(double* sm, const double* __restrict__ g, int ld, int o0, int k0, int O,
                                             int K, int tid) {
  constexpr int P = 2 * BO + 4;
  constexpr int CH = BO * 16;
#pragma unroll
  for (int c = tid; c < CH; c += THREADS) {
    int o, k;
    if (OUTER_CONTIG) {  // (o, k) at g[o + k ld]: o fastest across threads
      k = c / BO;
      o = c % BO;
    } else {  // (o, k) at g[k + o ld]: k fastest
      o = c / 16;
      k = c % 16;
    }
    const int go = o0 + o, gk = k0 + k;
    const bool valid = go < O && gk < K;
    const double* src = g + (valid ? (OUTER_CONTIG ? IDX(go, gk, ld) : IDX(gk, go, ld)) : 0);
    const int kp = (k >> 3) * 4 + (k & 3), h = (k >> 2) & 1;
    cp_async_8(sm + kp * P + 2 * o + h, src, valid ? 8 : 0);
  }
}

// TAG only separates the a3 block multiply B.Z (TAG = 1) from the other GEMMs in profiles.
// Two problems sharing op(B), M, N, K and the leading dimensions (A2 != nullptr): blockIdx.z =
// problem * splits + split, problem 1 reads A2 and writes C2 (one launch for X = S C' and
// BX = BS C' of the rotation).
template <int OPA, int OPB, int BM, int BN, int STAGES, int TAG = 0>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32, (BM * BN >= 8192) ? 2 : 3)
    dgemm_kp_kernel(int M, int N, int K, double alpha, const double* __restrict__ A, int lda,
                    const double* __restrict__ B, int ldb, double beta, double* __restrict__ C, int ldc,
                    double* __restrict__ partial, int ktiles_per_split, const double* __restrict__ A2,
                    double* __restrict__ C2, int splits) {
  // programmatic dependent launch: nothing before this line touches memory the previous kernel
  // in the stream writes (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (A2 && (int)blockIdx.z >= splits) {  // problem 1
    A = A2;
    C = C2;
    if (partial) partial += (size_t)splits * M * N;
  }
  const int zsplit = A2 ? (int)blockIdx.z % splits : (int)blockIdx.z;
  constexpr int WM = 32, WN = 32, BK = 16;
  constexpr int WARPS_M = BM / WM, THREADS = (BM / WM) * (BN / WN) * 32;
  constexpr int MI = WM / 8, NI = WN / 8;
  constexpr int PA = 2 * BM + 4, PB = 2 * BN + 4;
  constexpr int A_ELEMS = 8 * PA, B_ELEMS = 8 * PB, STAGE = A_ELEMS + B_ELEMS;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KT = cdiv(K, BK);
  const int kt0 = zsplit * ktiles_per_split;
  const int nkt = max(0, min(KT, kt0 + ktiles_per_split) - kt0);
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  auto issue = [&](int s, int kt) {
    double* sa = smem + (size_t)s * STAGE;
    load_tile_kp<BM, THREADS, OPA == OP_N>(sa, A, lda, m0, kt * BK, M, K, tid);
    load_tile_kp<BN, THREADS, OPB == OP_T>(sa + A_ELEMS, B, ldb, n0, kt * BK, N, K, tid);
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) issue(s, kt0 + s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int it = 0; it < nkt; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nx = it + STAGES - 1;
      if (nx < nkt) issue(nx % STAGES, kt0 + nx);
      cp_async_commit();
    }
    const double* sa = smem + (size_t)(it % STAGES) * STAGE;
    const double* sb = sa + A_ELEMS;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      double2 af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i)
        af[i] = *reinterpret_cast<const double2*>(sa + (q * 4 + fk) * PA + 2 * (wm * WM + i * 8 + fr));
#pragma unroll
      for (int j = 0; j < NI; ++j)
        bf[j] = *reinterpret_cast<const double2*>(sb + (q * 4 + fk) * PB + 2 * (wn * WN + j * 8 + fr));
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_884(acc[i][j], af[i].x, bf[j].x);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_884(acc[i][j], af[i].y, bf[j].y);
    }
  }
  cp_async_wait<0>();
  // the next kernel (split-K reduce) may be scheduled now; it waits for this grid's completion
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int row = m0 + wm * WM + i * 8 + fr;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * WN + j * 8 + fk * 2 + h;
        if (col >= N) continue;
        const double v = acc[i][j][h];
        if (partial) {
          partial[(size_t)zsplit * M * N + IDX(row, col, M)] = v;
        } else {
          double* c = C + IDX(row, col, ldc);
          *c = (beta == 0.0) ? alpha * v : alpha * v + beta * (*c);
        }
      }
    }
  }
}

}  // namespace psd
