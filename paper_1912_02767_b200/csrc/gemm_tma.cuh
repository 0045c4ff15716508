// gemm_tma.cuh -- the a3 block multiply Y = alpha A Z (A symmetric n x n, Z n x k, fp64) with TMA-staged
// operand tiles (cp.async.bulk.tensor, 128-byte swizzle, mbarrier-completed ring) and DMMA tensor-core
// math (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; tcgen05.mma has no f64 kind).
//
// Both operands are read along their contiguous dimension in 16-double (128 B) rows:
//   A tile  BM x 16: row m = A[k0 .. k0+15, m] (column m of A = row m, A symmetric), box {16, BM}
//   Z tile  BN x 16: row c = Z[k0 .. k0+15, c] (column c of Z),                       box {16, BN}
// so one TMA per operand per k-step, zero-filled past the matrix edges (ragged m, k, c need no
// predication). With SWIZZLE_128B the 16-byte chunk j of row r sits at chunk j ^ (r mod 8), and a lane
// (fr = lane / 4, fk = lane % 4) reading chunk q*4 + fk of rows fr + 8 i hits 8 distinct chunk slots
// per quarter-warp: one LDS.128 per fragment pair, 4 wavefronts per 512 B, conflict-free. The chunk holds
// k = 2c, 2c + 1: the two MMAs of a pair take k = {0,2,4,6} + 8q and {1,3,5,7} + 8q -- a permutation of
// the k sum applied identically to both operands.
//
// One thread issues the TMA for stage it + STAGES - 1 after the CTA barrier that ends the reads of that
// stage (consumed at it - 1); every thread waits on the stage's mbarrier phase (complete_tx bytes).
// Split-K partials and the epilogue are those of dgemm_kp_kernel (gemm.cuh); PDL as there.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace psd {

__device__ __forceinline__ uint32_t tma_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tma_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tma_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tma_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(tma_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          tma_smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(tma_smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          tma_smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(tma_smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma_884t(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int BM, int BN, int STAGES>
struct TmaGemmCfg {
  static constexpr int WN = BN < 32 ? BN : 32;  // warp tile width (BN = 16: the HBM-bound small-k variant)
  static constexpr int THREADS = (BM / 32) * (BN / WN) * 32;
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128, STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 64;  // + 1024-B alignment, barriers
};

// Y (M x N, ldc) = alpha A Z with A symmetric M x M (tensor map mapA over A, inner dim = row), Z M x N
// (mapB). partial != nullptr: raw split-K partials (ld M) as dgemm_kp_kernel.
template <int BM, int BN, int STAGES, int TAG = 1>
__global__ void __launch_bounds__(TmaGemmCfg<BM, BN, STAGES>::THREADS, (BM * BN >= 4096) ? 2 : 3)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M,
                     int N, int K, double alpha, double* __restrict__ C, int ldc, double* __restrict__ partial,
                     int ktiles_per_split) {
  using Cfg = TmaGemmCfg<BM, BN, STAGES>;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL (launch_pdl): inputs written by the predecessor
  constexpr int WM = 32, WN = Cfg::WN, BK = 16;
  constexpr int WARPS_M = BM / WM;
  constexpr int MI = WM / 8, NI = WN / 8;
  extern __shared__ __align__(16) unsigned char tma_smem_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)tma_smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * Cfg::STAGE_BYTES);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  // column tiles fastest: the CTAs that share a row panel of A run together and read it from L2 once
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int KT = cdiv(K, BK);
  const int kt0 = blockIdx.z * ktiles_per_split;
  const int nkt = max(0, min(KT, kt0 + ktiles_per_split) - kt0);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) tma_mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  __syncthreads();
  auto issue = [&](int s, int kt) {
    unsigned char* st = base + (size_t)s * Cfg::STAGE_BYTES;
    tma_mbar_expect_tx(full + s, Cfg::STAGE_BYTES);
    tma_load_2d(st, &mapA, kt * BK, m0, full + s);
    tma_load_2d(st + Cfg::A_BYTES, &mapB, kt * BK, n0, full + s);
  };
  if (tid == 0)
    for (int s = 0; s < STAGES - 1 && s < nkt; ++s) issue(s, kt0 + s);
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;
  for (int it = 0; it < nkt; ++it) {
    const int s = it % STAGES;
    tma_mbar_wait(full + s, (uint32_t)((it / STAGES) & 1));
    __syncthreads();  // every thread finished stage (it - 1) % STAGES: it may be refilled
    if (tid == 0) {
      const int nx = it + STAGES - 1;
      if (nx < nkt) issue(nx % STAGES, kt0 + nx);
    }
    const unsigned char* sa = base + (size_t)s * Cfg::STAGE_BYTES;
    const unsigned char* sb = sa + Cfg::A_BYTES;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = q * 4 + fk;  // 16-byte chunk: k = 2c, 2c + 1 of this 16-wide k tile
      double2 af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int r = wm * WM + i * 8 + fr;
        af[i] = *reinterpret_cast<const double2*>(sa + r * 128 + ((c ^ (r & 7)) << 4));
      }
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int r = wn * WN + j * 8 + fr;
        bf[j] = *reinterpret_cast<const double2*>(sb + r * 128 + ((c ^ (r & 7)) << 4));
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_884t(acc[i][j], af[i].x, bf[j].x);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_884t(acc[i][j], af[i].y, bf[j].y);
    }
  }
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
        if (partial)
          partial[(size_t)blockIdx.z * M * N + IDX(row, col, M)] = v;
        else
          C[IDX(row, col, ldc)] = alpha * v;
      }
    }
  }
}

// Row-panel variant for N <= 64 (the a3 shapes of a converging LOBPCG call): one CTA owns 32 rows of
// Y and the WHOLE k range, so no split-K partials go through HBM and no reduce kernel runs.
// 256 consumer threads = BN / WN column warps (WN = min(BN, 32)) x KG k-groups, plus one producer
// warp that refills a stage as soon as the eight consumer warps released it (full / empty mbarriers); a stage holds KG consecutive 16-wide k tiles
// (one TMA per operand per k tile, the same swizzled boxes as dgemm_tma_kernel) and k-group g
// consumes tile g of every stage. After the k loop the KG partial 32 x BN tiles are summed in
// shared memory in fixed order g = 0 .. KG-1 (deterministic) and written with coalesced stores.
// n = 4000: 125 CTAs, one per SM (A read once from HBM; Z, 2 MB at BN = 64, from L2). BN = 16 is the
// HBM-bound small-k case (8 k-groups keep 4 stages x 32 KB of A in flight per SM).
template <int BN>
struct PanelGemmCfg {
  static constexpr int BM = 32, WN = BN < 32 ? BN : 32, NWN = BN / WN, KG = 8 / NWN, THREADS = 256 + 32;
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128, TILE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGE_BYTES = KG * TILE_BYTES;
  static constexpr int STAGES = (4 * STAGE_BYTES + 2048 <= 200 * 1024) ? 4 : 3;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 128;
  static_assert((size_t)KG * BM * BN * 8 <= (size_t)STAGES * STAGE_BYTES, "reduction buffer fits the stages");
};

template <int BN, bool T3>
__global__ void __launch_bounds__(288, 1)
    dgemm_tma_panel_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M,
                           int N, int K, double alpha, double* __restrict__ C, int ldc) {
  using Cfg = PanelGemmCfg<BN>;
  constexpr int BM = Cfg::BM, KG = Cfg::KG, STAGES = Cfg::STAGES, BK = 16;
  constexpr int MI = 4, NI = Cfg::WN / 8;  // 32 x WN warp tile
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) unsigned char tma_smem_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)tma_smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wn = warp % Cfg::NWN, g = warp / Cfg::NWN;  // column warp, k-group (warp 8: producer)
  const int m0 = blockIdx.x * BM;
  const int KT = cdiv(K, BK);
  const int NST = cdiv(KT, KG);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tma_mbar_init(full + s, 1);
      tma_mbar_init(empty + s, 8);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  __syncthreads();
  // stage layout: the KG A tiles (A_BYTES each), then the KG Z tiles (B_BYTES each)
  auto issue = [&](int s, int st) {
    unsigned char* sp = base + (size_t)s * Cfg::STAGE_BYTES;
    if (T3) {
      // 3-D maps {16, columns, k tiles}: one TMA per operand per stage, and every column of the A
      // panel is fetched as KG x 128 B = one contiguous run (DRAM-page friendly) instead of KG
      // separate 128-byte pieces 32 KB apart; k tiles past the end are zero-filled (n % 16 == 0)
      tma_mbar_expect_tx(full + s, (uint32_t)Cfg::STAGE_BYTES);
      tma_load_3d(sp, &mapA, 0, m0, st * KG, full + s);
      tma_load_3d(sp + KG * Cfg::A_BYTES, &mapB, 0, 0, st * KG, full + s);
    } else {
      const int nt = min(KG, KT - st * KG);  // k tiles in this stage (the last stage may be short)
      tma_mbar_expect_tx(full + s, (uint32_t)(nt * Cfg::TILE_BYTES));
      for (int t = 0; t < nt; ++t) {
        const int kk = (st * KG + t) * BK;
        tma_load_2d(sp + t * Cfg::A_BYTES, &mapA, kk, m0, full + s);
        tma_load_2d(sp + KG * Cfg::A_BYTES + t * Cfg::B_BYTES, &mapB, kk, 0, full + s);
      }
    }
  };
  if (warp == 8) {
    // producer: refill a slot once all eight consumer warps released it (empty barrier), so the
    // consumers never meet at a CTA-wide barrier inside the k loop
    if (lane == 0)
      for (int it = 0; it < NST; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) tma_mbar_wait(empty + s, (uint32_t)(((it / STAGES) - 1) & 1));
        issue(s, it);
      }
    return;
  }
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;
  for (int it = 0; it < NST; ++it) {
    const int s = it % STAGES;
    tma_mbar_wait(full + s, (uint32_t)((it / STAGES) & 1));
    if (it * KG + g < KT) {
      const unsigned char* sa = base + (size_t)s * Cfg::STAGE_BYTES + g * Cfg::A_BYTES;
      const unsigned char* sb = base + (size_t)s * Cfg::STAGE_BYTES + KG * Cfg::A_BYTES + g * Cfg::B_BYTES;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = q * 4 + fk;
        double2 af[MI], bf[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int r = i * 8 + fr;
          af[i] = *reinterpret_cast<const double2*>(sa + r * 128 + ((c ^ (r & 7)) << 4));
        }
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int r = wn * Cfg::WN + j * 8 + fr;
          bf[j] = *reinterpret_cast<const double2*>(sb + r * 128 + ((c ^ (r & 7)) << 4));
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma_884t(acc[i][j], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma_884t(acc[i][j], af[i].y, bf[j].y);
      }
    }
    __syncwarp();
    if (lane == 0) tma_mbar_arrive(empty + s);  // this warp is done reading slot s
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // every stage consumed (the producer warp has exited): the stage buffers become the reduction buffer
  asm volatile("bar.sync 1, 256;" ::: "memory");
  double* red = reinterpret_cast<double*>(base);  // [g][col 0..BN)[row 0..32)
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = i * 8 + fr, col = wn * Cfg::WN + j * 8 + fk * 2 + h;
        red[((size_t)g * BN + col) * BM + row] = acc[i][j][h];
      }
  asm volatile("bar.sync 1, 256;" ::: "memory");
  for (int e = tid; e < BM * BN; e += 256) {
    const int row = e % BM, col = e / BM;
    if (m0 + row >= M || col >= N) continue;
    double v = red[(size_t)col * BM + row];
#pragma unroll
    for (int gg = 1; gg < KG; ++gg) v += red[((size_t)gg * BN + col) * BM + row];
    C[IDX(m0 + row, col, ldc)] = alpha * v;
  }
}

}  // namespace psd
