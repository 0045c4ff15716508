// psdproj.cu -- C ABI + host orchestration of the warm-started LOBPCG PSD-cone projection.
//
// The LOBPCG control flow (convergence, locking, active set, expansion) runs on the host
// (C++17); every arithmetic step runs in the sm_100a kernels of gemm.cuh / kernels.cuh on the
// caller's stream. Per LOBPCG iteration the host reads back two small vectors (the residual
// norms r and the Rayleigh-Ritz values theta); everything n-sized stays in HBM.
//
// Algorithm (restated in DESIGN.md §2; readings R*): Alg. 3 of PAPER.md:398-412 on B = s*A
// (s = +1/-1), started from the previous call's block (warm) or a Philox block
// (cold), Rayleigh-Ritz by implicit Cholesky-QR + Jacobi (Alg. 2), residual
// basis (footnote PAPER.md:377), BLOPEX P direction (R5), hard/soft locking (R35), random
// expansion (line 8, R8-R11), stopping rule with guard (R12), Theorem-3 bound
// (R14-R16, R36), side rule (R17-R18).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <initializer_list>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "psdproj.h"
#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "tridiag.cuh"
#include "cluster_la.cuh"
#include "tridiag_tile.cuh"
#include "tridiag_warp.cuh"
#include "gemm_tma.cuh"
#include "tiny_lobpcg.cuh"
#include "sbr.cuh"
#include "tridiag_rep.cuh"

using namespace psd;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) return set_err(PSDPROJ_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x, \
                                          cudaGetErrorString(e_));                              \
  } while (0)
static thread_local long long g_launches = 0;  // kernels issued by this thread (info.launches)
#define CKL()              \
  do {                     \
    ++g_launches;          \
    CK(cudaGetLastError()); \
  } while (0)
#define TRY(x)              \
  do {                      \
    int rc_ = (x);          \
    if (rc_ < 0) return rc_; \
  } while (0)

static inline int rup(int x, int a) { return (x + a - 1) / a * a; }
constexpr int EIG_MAX = 2048;  // largest dense eigenproblem of the RR / DIRECT eigensolver
constexpr int TRINV_MAX = 1280;  // largest direction block of the pencil's triangular inverse (trinv_run)

// ------------------------------------------------------------------ NCCL (row-sharded mode, §8.e)
// Loaded on first use with dlopen (the library in the process -- torch's -- or PSDPROJ_NCCL_LIB), so
// libpsdproj.so has no link-time NCCL dependency and the single-GPU path never touches it.
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};
static NcclApi g_nccl;
static int nccl_load() {
  if (g_nccl.tried) return g_nccl.ok ? 0 : set_err(PSDPROJ_E_NCCL, "NCCL library not available");
  g_nccl.tried = true;
  void* h = nullptr;
  if (const char* e = getenv("PSDPROJ_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_err(PSDPROJ_E_NCCL, "dlopen(libnccl.so.2) failed: %s", dlerror());
  g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
  g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
  g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.allReduce && g_nccl.allGather &&
              g_nccl.commDestroy && g_nccl.getErrorString;
  return g_nccl.ok ? 0 : set_err(PSDPROJ_E_NCCL, "NCCL symbols missing");
}
#define NK(x)                                                                                                  \
  do {                                                                                                         \
    ncclResult_t r_ = (x);                                                                                     \
    if (r_ != ncclSuccess) return set_err(PSDPROJ_E_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #x,             \
                                          g_nccl.getErrorString ? g_nccl.getErrorString(r_) : "nccl error"); \
  } while (0)
static int g_sms = 0;
static int sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}
static inline int grid1d(size_t work, int nt = 256) {
  size_t b = (work + nt - 1) / nt;
  size_t cap = (size_t)sms() * 8;
  return (int)std::max<size_t>(1, std::min(b, cap));
}

// host-side profile of psdproj_project (PSDPROJ_HOSTPROF=1): time blocked in stream syncs
static const bool g_hostprof = getenv("PSDPROJ_HOSTPROF") != nullptr;
static thread_local double g_sync_s = 0.0;
static thread_local long g_nsync = 0;

// SMs held by a concurrently running kernel (the overlapped Cholesky cluster): the split-K choice
// of a GEMM launched meanwhile sizes its grid for the rest, so it stays one wave
static thread_local int g_sm_reserve = 0;

// kernels that begin with griddepcontrol.wait are launched as programmatic dependents of the
// previous kernel in the stream (their launch overlaps its tail); PSDPROJ_PDL=0: ordinary launches
static const bool g_pdl = !(getenv("PSDPROJ_PDL") && atoi(getenv("PSDPROJ_PDL")) == 0);
template <typename... KArgs, typename... Args>
static int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  if (!g_pdl) {
    kern<<<grid, block, smem, st>>>(args...);
    CKL();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...));
  ++g_launches;
  return 0;
}

// D2D copy of a rows x cols block as a (PDL) kernel: stays inside the chain of dependent launches
// where a copy-engine memcpy would break it
static int copy_block_pdl(cudaStream_t st, int rows, int cols, double* dst, int ldd, const double* src, int lds) {
  if (rows <= 0 || cols <= 0) return 0;
  GatherJobs g{};
  g.j[0] = GatherJob{dst, src, nullptr, ldd, lds, cols};
  g.nj = 1;
  return launch_pdl(gather_multi_kernel, dim3(grid1d((size_t)rows * cols)), dim3(256), 0, st, rows, g);
}

// ------------------------------------------------------------------ GEMM dispatch
namespace {
constexpr int GBM = 64, GBN = 64, GBK = 16, GWM = 32, GWN = 32, GST = 4;
using GCfg = GemmCfg<GBM, GBN, GBK, GWM, GWN, GST>;

template <int OA, int OB, bool V>
int gemm_launch(cudaStream_t st, int M, int N, int K, double alpha, const double* A, int lda, const double* B,
                int ldb, double beta, double* C, int ldc, double* part, int splits, int ktps) {
  auto kern = dgemm_kernel<OA, OB, GBM, GBN, GBK, GWM, GWN, GST, V>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GCfg::SMEM));
    attr = true;
  }
  dim3 grid(cdiv(M, GBM), cdiv(N, GBN), splits);
  kern<<<grid, GCfg::THREADS, GCfg::SMEM, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                                splits > 1 ? part : nullptr, ktps);
  CKL();
  if (splits > 1) {
    splitk_reduce_kernel<<<dim3(cdiv(M, 256), N), 256, 0, st>>>(M, N, splits, alpha, part, beta, C, ldc);
    CKL();
  }
  return 0;
}
}  // namespace

template <int OA, int OB, int BM, int BN, int ST, int TAG = 0>
static int gemm_kp_launch(cudaStream_t st, int M, int N, int K, double alpha, const double* A, int lda,
                          const double* B, int ldb, double beta, double* C, int ldc, double* part, size_t part_elems,
                          const double* A2 = nullptr, double* C2 = nullptr) {
  constexpr int THREADS = (BM / 32) * (BN / 32) * 32;
  constexpr size_t SMEM = (size_t)ST * 8 * ((2 * BM + 4) + (2 * BN + 4)) * sizeof(double);
  auto kern = dgemm_kp_kernel<OA, OB, BM, BN, ST, TAG>;
  static bool attr = false;
  static int per_sm = 1;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, SMEM));
    per_sm = std::max(per_sm, 1);
    attr = true;
  }
  const int KT = cdiv(std::max(K, 1), 16);
  const int nprob = A2 ? 2 : 1;
  const int tiles = cdiv(M, BM) * cdiv(N, BN) * nprob;
  const int slots = std::max(1, sms() - g_sm_reserve) * per_sm;
  int splits = 1;
  if (part && tiles < slots && KT >= 8) {
    splits = std::min(std::max(1, slots / tiles), KT / 4);
    splits = std::max(1, std::min(splits, 32));
    while (splits > 1 && (size_t)splits * nprob * M * N > part_elems) --splits;
  }
  const int ktps = cdiv(KT, splits);
  splits = cdiv(KT, ktps);
  dim3 grid(cdiv(M, BM), cdiv(N, BN), splits * nprob);
  TRY(launch_pdl(kern, grid, dim3(THREADS), SMEM, st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                 splits > 1 ? part : (double*)nullptr, ktps, A2, C2, splits));
  if (splits > 1) {
    TRY(launch_pdl(splitk_reduce_kernel, dim3(cdiv(M, 256), N), dim3(256), 0, st, M, N, splits, alpha,
                   (const double*)part, beta, C, ldc));
    if (A2)
      TRY(launch_pdl(splitk_reduce_kernel, dim3(cdiv(M, 256), N), dim3(256), 0, st, M, N, splits, alpha,
                     (const double*)(part + (size_t)splits * M * N), beta, C2, ldc));
  }
  return 0;
}

// ---------------------------------------------------------------- a3 with TMA-staged tiles (gemm_tma.cuh)
typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encode() {
  static TmapEncodeFn f = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = (TmapEncodeFn)p;
  }
  return f;
}
// 2-D fp64 tensor map: inner dimension `inner` (contiguous), outer `outer` (stride ld doubles), box
// {16, box_outer}, 128-byte swizzle, out-of-bounds elements zero-filled
static int make_tmap(CUtensorMap* m, const double* ptr, int inner, int outer, int ld, int box_outer) {
  TmapEncodeFn f = tmap_encode();
  if (!f) return set_err(PSDPROJ_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {16, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PSDPROJ_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}
// Y (n x k, ldy) = alpha A Z, A symmetric n x n (lda even, 16-B aligned), Z n x k (ldz even): the a3
// block multiply on TMA-staged tiles; split-K over the SMs left free as gemm_kp_launch
template <int BM, int BN, int ST>
static int gemm_tma_launch(cudaStream_t st, int n, int k, double alpha, const double* A, int lda, const double* Z,
                           int ldz, double* Y, int ldy, double* part, size_t part_elems) {
  using Cfg = TmaGemmCfg<BM, BN, ST>;
  auto kern = dgemm_tma_kernel<BM, BN, ST, 1>;
  static bool attr = false;
  static int per_sm = 1;
  if (!attr) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::THREADS, Cfg::SMEM));
    per_sm = std::max(per_sm, 1);
    attr = true;
  }
  CUtensorMap ma, mb;
  TRY(make_tmap(&ma, A, n, n, lda, BM));
  TRY(make_tmap(&mb, Z, n, k, ldz, BN));
  const int KT = cdiv(std::max(n, 1), 16);
  const int tiles = cdiv(n, BM) * cdiv(k, BN);
  const int slots = std::max(1, sms() - g_sm_reserve) * per_sm;
  // split-K count with the best wave efficiency tiles * splits / (waves * slots) (fewer splits on ties)
  int splits = 1;
  if (part && KT >= 8) {
    double best = 0.0;
    for (int sp = 1; sp <= std::min(16, KT / 4); ++sp) {
      if ((size_t)sp * n * k > part_elems) break;
      const int waves = cdiv(tiles * sp, slots);
      const double eff = (double)tiles * sp / ((double)waves * slots);
      if (eff > best + 0.02) {
        best = eff;
        splits = sp;
      }
    }
  }
  const int ktps = cdiv(KT, splits);
  splits = cdiv(KT, ktps);
  dim3 grid(cdiv(k, BN), cdiv(n, BM), splits);
  TRY(launch_pdl(kern, grid, dim3(Cfg::THREADS), Cfg::SMEM, st, ma, mb, n, k, n, alpha, Y, ldy,
                 splits > 1 ? part : (double*)nullptr, ktps));
  if (splits > 1)
    TRY(launch_pdl(splitk_reduce_kernel, dim3(cdiv(n, 256), k), dim3(256), 0, st, n, k, splits, alpha,
                   (const double*)part, 0.0, Y, ldy));
  return 0;
}

// 3-D fp64 tensor map {16, cols, k tiles} over a column-major matrix with `rows` = 16 * ktiles rows:
// element (r, c, t) at ptr[16 t + r + c ld] (strides ld * 8 and 128 bytes), box {16, box_cols, box_t},
// 128-byte swizzle
static int make_tmap3(CUtensorMap* m, const double* ptr, int ktiles, int cols, int ld, int box_cols, int box_t) {
  TmapEncodeFn f = tmap_encode();
  if (!f) return set_err(PSDPROJ_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {16, (cuuint64_t)cols, (cuuint64_t)ktiles};
  cuuint64_t strides[2] = {(cuuint64_t)ld * sizeof(double), 16 * sizeof(double)};
  cuuint32_t box[3] = {16, (cuuint32_t)box_cols, (cuuint32_t)box_t};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 1;
}

// Row-panel variant (gemm_tma.cuh: dgemm_tma_panel_kernel): 32 rows x the whole k range per CTA, no
// split-K partials; 3-D tensor maps (one TMA per operand per stage, contiguous 128 KG-byte runs per
// column) when n % 16 == 0, else 2-D maps (one TMA per 16-wide k tile)
template <int BN>
static int gemm_tma_panel_launch(cudaStream_t st, int n, int k, double alpha, const double* A, int lda,
                                 const double* Z, int ldz, double* Y, int ldy) {
  using Cfg = PanelGemmCfg<BN>;
  static const int t3_env = getenv("PSDPROJ_A3_PANEL3D") ? atoi(getenv("PSDPROJ_A3_PANEL3D")) : 1;
  CUtensorMap ma, mb;
  bool t3 = t3_env && n % 16 == 0;
  if (t3) t3 = make_tmap3(&ma, A, n / 16, n, lda, Cfg::BM, Cfg::KG) == 0 && make_tmap3(&mb, Z, n / 16, k, ldz, BN, Cfg::KG) == 0;
  auto kern = t3 ? dgemm_tma_panel_kernel<BN, true> : dgemm_tma_panel_kernel<BN, false>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(dgemm_tma_panel_kernel<BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    CK(cudaFuncSetAttribute(dgemm_tma_panel_kernel<BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    attr = true;
  }
  if (!t3) {
    TRY(make_tmap(&ma, A, n, n, lda, Cfg::BM));
    TRY(make_tmap(&mb, Z, n, k, ldz, BN));
  }
  TRY(launch_pdl(kern, dim3(cdiv(n, Cfg::BM)), dim3(Cfg::THREADS), Cfg::SMEM, st, ma, mb, n, k, n, alpha, Y, ldy));
  return 0;
}

// a3 tile choice: the row-panel kernel when k <= 64 and its cdiv(n, 32) CTAs fill at least 3/4
// of the SMs left (one CTA per SM); otherwise 64-row tiles with split-K -- 16 columns for k <= 16
// (HBM-bound: no DMMA on zero padding), 32 when the last 64-tile would be at most half full, else 64
static int a3_multiply_tma(cudaStream_t st, int n, int k, double alpha, const double* A, int lda, const double* Z, int ldz,
                  double* Y, int ldy, double* part, size_t part_elems) {
  static const int panel_on = getenv("PSDPROJ_A3_PANEL") ? atoi(getenv("PSDPROJ_A3_PANEL")) : 1;
  const int free_sms = std::max(1, sms() - g_sm_reserve);
  if (panel_on && k <= 64 && 4 * cdiv(n, 32) >= 3 * free_sms)
    return k <= 16   ? gemm_tma_panel_launch<16>(st, n, k, alpha, A, lda, Z, ldz, Y, ldy)
           : k <= 32 ? gemm_tma_panel_launch<32>(st, n, k, alpha, A, lda, Z, ldz, Y, ldy)
                     : gemm_tma_panel_launch<64>(st, n, k, alpha, A, lda, Z, ldz, Y, ldy);
  const bool narrow = k <= 96 && (k % 64) != 0 && (k % 64) <= 32;
  if (k <= 16) return gemm_tma_launch<64, 16, 6>(st, n, k, alpha, A, lda, Z, ldz, Y, ldy, part, part_elems);
  if (narrow) return gemm_tma_launch<64, 32, 4>(st, n, k, alpha, A, lda, Z, ldz, Y, ldy, part, part_elems);
  return gemm_tma_launch<64, 64, 4>(st, n, k, alpha, A, lda, Z, ldz, Y, ldy, part, part_elems);
}

// Two products C = alpha A B + beta C and C2 = alpha A2 B + beta C2 (same B, shapes and leading
// dimensions) in one launch (k-paired kernel, 64 x 64 or 64 x 32 tiles).
static int dgemm2(cudaStream_t st, int M, int N, int K, double alpha, const double* A, const double* A2, int lda,
                  const double* B, int ldb, double beta, double* C, double* C2, int ldc, double* part,
                  size_t part_elems) {
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0) {
    if (beta == 0.0) {
      CK(cudaMemset2DAsync(C, (size_t)ldc * 8, 0, (size_t)M * 8, N, st));
      CK(cudaMemset2DAsync(C2, (size_t)ldc * 8, 0, (size_t)M * 8, N, st));
    }
    return 0;
  }
  const bool narrow = N <= 96 && (N % 64) != 0 && (N % 64) <= 32;
  return narrow ? gemm_kp_launch<OP_N, OP_N, 64, 32, 4>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, part,
                                                         part_elems, A2, C2)
                : gemm_kp_launch<OP_N, OP_N, 64, 64, 4>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, part,
                                                         part_elems, A2, C2);
}

static int dgemm(cudaStream_t st, int opA, int opB, int M, int N, int K, double alpha, const double* A, int lda,
                 const double* B, int ldb, double beta, double* C, int ldc, double* part, size_t part_elems) {
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0 && beta == 0.0) {
    CK(cudaMemset2DAsync(C, (size_t)ldc * 8, 0, (size_t)M * 8, N, st));
    return 0;
  }
  static int mode = -1;  // 0: k-paired kernel (default), 1: first-cut kernel
  if (mode < 0) mode = (getenv("PSDPROJ_GEMM") && std::string(getenv("PSDPROJ_GEMM")) == "old") ? 1 : 0;
  if (mode == 0) {
    static int tile = -1;
    if (tile < 0) tile = getenv("PSDPROJ_GEMM_TILE") ? atoi(getenv("PSDPROJ_GEMM_TILE")) : 64;
    const bool big = tile == 128 && M >= 1024 && N >= 48;
    // narrow tiles when a 64-wide last column tile would be at most half used (N mod 64 in 1..32)
    const bool narrow = !big && N <= 96 && (N % 64) != 0 && (N % 64) <= 32;
#define GK(OA, OB)                                                                                                     \
  return big      ? gemm_kp_launch<OA, OB, 128, 64, 4>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, part, part_elems) \
         : narrow ? gemm_kp_launch<OA, OB, 64, 32, 4>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, part, part_elems)  \
                  : gemm_kp_launch<OA, OB, 64, 64, 4>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, part, part_elems)
    if (opA == OP_N && opB == OP_N) GK(OP_N, OP_N);
    if (opA == OP_T && opB == OP_N) GK(OP_T, OP_N);
    if (opA == OP_N && opB == OP_T) GK(OP_N, OP_T);
    GK(OP_T, OP_T);
#undef GK
  }
  bool vec = (lda % 2 == 0) && (ldb % 2 == 0) && (((uintptr_t)A & 15) == 0) && (((uintptr_t)B & 15) == 0);
  int KT = cdiv(std::max(K, 1), GBK);
  int tiles = cdiv(M, GBM) * cdiv(N, GBN);
  int splits = 1;
  int target = sms() * 2;
  if (tiles < target && part && KT >= 8) {
    splits = std::min(cdiv(target, tiles), KT / 4);
    splits = std::max(1, std::min(splits, 32));
    while (splits > 1 && (size_t)splits * M * N > part_elems) --splits;
  }
  int ktps = cdiv(KT, splits);
  splits = cdiv(KT, ktps);
#define GL(OA, OB)                                                                                       \
  return vec ? gemm_launch<OA, OB, true>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, part, splits, ktps) \
             : gemm_launch<OA, OB, false>(st, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, part, splits, ktps)
  if (opA == OP_N && opB == OP_N) GL(OP_N, OP_N);
  if (opA == OP_T && opB == OP_N) GL(OP_T, OP_N);
  if (opA == OP_N && opB == OP_T) GL(OP_N, OP_T);
  GL(OP_T, OP_T);
#undef GL
}

// ------------------------------------------------------------------ Jacobi dispatch
static int g_coop_blocks = 0;
static int jacobi_run(cudaStream_t st, int s, const double* A, int lda, double* w, double* V, int ldv, double* M,
                      double* M2, double* Q, int* d_info, int* d_counters, double* d_fro, int max_sweeps = 60) {
  if (s <= 0) return 0;
  static int smem_max = -1;
  if (smem_max < 0) {
    smem_max = JAC_SMEM_MAX;
    if (const char* e = getenv("PSDPROJ_JACOBI_SMEM_MAX")) smem_max = std::min(JAC_SMEM_MAX, atoi(e));
  }
  if (s <= smem_max) {
    int N = s + (s & 1);
    size_t smem = (size_t)2 * N * (N + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(jacobi_smem_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(2 * JAC_SMEM_MAX * (JAC_SMEM_MAX + 1) * sizeof(double))));
      attr = true;
    }
    jacobi_smem_kernel<512><<<1, 512, smem, st>>>(s, A, lda, w, V, ldv, max_sweeps, d_info);
    CKL();
    return 0;
  }
  int N = s + (s & 1);
  jacobi_prep_kernel<<<grid1d((size_t)N * N), 256, 0, st>>>(s, N, A, lda, M, Q);
  CKL();
  fro_kernel<1024><<<1, 1024, 0, st>>>((int64_t)N * N, M, d_fro);
  CKL();
  CK(cudaMemsetAsync(d_counters, 0, sizeof(int) * (max_sweeps + 2), st));
  int mode = 1;  // 1 = cluster, 2 = cooperative grid
  if (const char* e = getenv("PSDPROJ_JACOBI_MODE")) mode = atoi(e);
  double afl_scale = PSD_U;  // absolute floor u ||A||_F (R39)
  if (mode == 1) {
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(jacobi_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attr = true;
    }
    if (N / 2 > JAC_CL_MAXH) return set_err(PSDPROJ_E_CAPACITY, "Jacobi size %d > %d", s, 2 * JAC_CL_MAXH);
    int cs = s <= 160 ? 8 : 16;
    if (const char* e = getenv("PSDPROJ_JACOBI_CS")) cs = std::max(1, std::min(16, atoi(e)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel, s, N, M, M2, Q, (const double*)d_fro, afl_scale, max_sweeps,
                          d_info));
    ++g_launches;
  } else {
    if (!g_coop_blocks) {
      int per = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, jacobi_coop_kernel, 512, 0));
      if (per < 1) return set_err(PSDPROJ_E_CUDA, "jacobi_coop_kernel cannot be co-resident");
      g_coop_blocks = sms();  // one CTA per SM: the grid barrier is the per-round cost
      if (const char* e = getenv("PSDPROJ_JACOBI_CTAS")) g_coop_blocks = std::max(1, std::min(atoi(e), sms()));
    }
    if (N / 2 > JAC_COOP_MAXH) return set_err(PSDPROJ_E_CAPACITY, "Jacobi size %d > %d", s, 2 * JAC_COOP_MAXH);
    void* args[] = {(void*)&s, (void*)&N, (void*)&M, (void*)&M2, (void*)&Q, (void*)&d_fro, (void*)&afl_scale,
                    (void*)&max_sweeps, (void*)&d_counters, (void*)&d_info};
    CK(cudaLaunchCooperativeKernel((void*)jacobi_coop_kernel, dim3(g_coop_blocks), dim3(512), args, 0, st));
    ++g_launches;
  }
  jacobi_extract_kernel<<<grid1d((size_t)s * s), 256, 0, st>>>(s, N, M, M2, Q, d_info, w, V, ldv);
  CKL();
  return 0;
}

// ------------------------------------------------------------------ cluster launch helpers
// cluster size for a cluster_la.cuh kernel of order s: the preferred size (PSDPROJ_CLA_CS overrides),
// doubled until the kernel's shared-memory footprint fits; 0 if it does not fit in 16 CTAs
static int cla_cluster_size(int s, size_t (*smem_doubles)(int, int)) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("PSDPROJ_CLA_CS");
    forced = e ? std::max(1, std::min(16, atoi(e))) : 0;
  }
  int cs = forced ? forced : (s > 160 ? 16 : (s > 64 ? 8 : 4));
  while (cs < 16 && smem_doubles(s, cs) * sizeof(double) > (size_t)CLA_SMEM_BYTES) cs *= 2;
  return smem_doubles(s, cs) * sizeof(double) <= (size_t)CLA_SMEM_BYTES ? cs : 0;
}

template <typename... KArgs, typename... Args>
static int launch_cluster(void (*kern)(KArgs...), int cs, int nt, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, args...));
  ++g_launches;
  return 0;
}

static int cla_attrs() {
  static bool done = false;
  if (done) return 0;
  const int mx = CLA_SMEM_BYTES;
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<24, 256, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<24, 256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<40, 256, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<40, 256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<4, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<4, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<8, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<8, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<14, 256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<14, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<20, 256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<20, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(cholesky_cluster_kernel<false, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(cholesky_cluster_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(cholesky_cluster_kernel<false, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(cholesky_cluster_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(cholesky_cluster_kernel<true, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(cholesky_cluster_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  const int tmx = (int)(TI_KB * 32 * 40 * sizeof(double));
  CK(cudaFuncSetAttribute(trinv_panel_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
  CK(cudaFuncSetAttribute(trinv_panel_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
  CK(cudaFuncSetAttribute(trinv_panel_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
  CK(cudaFuncSetAttribute(trinv_panel_kernel<40>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
  const int bmx = CLA_SMEM_BYTES;
  CK(cudaFuncSetAttribute(backtransform_wy_kernel<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_wy_kernel<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_wy_kernel<20, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_wy_col_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_wy_col_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_wy_col_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_panel_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_panel_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_panel_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_panel_kernel<BT_PER_LANE>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(backtransform_panel_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, bmx));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<64, 256, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(tridiag_cluster_kernel<64, 256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
#define TRI_REG_ATTR(KR, CR)                                                                                          \
  CK(cudaFuncSetAttribute(tridiag_reg_kernel<KR, CR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)); \
  CK(cudaFuncSetAttribute(tridiag_reg_kernel<KR, CR>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));   \
  CK(cudaFuncSetAttribute(tridiag_rep_kernel<KR, CR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)); \
  CK(cudaFuncSetAttribute(tridiag_rep_kernel<KR, CR>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  TRI_REG_ATTR(3, 5)
  TRI_REG_ATTR(4, 4)
  TRI_REG_ATTR(6, 6)
  TRI_REG_ATTR(7, 7)
  TRI_REG_ATTR(8, 8)
#undef TRI_REG_ATTR
  CK(cudaFuncSetAttribute(sb1_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(sb1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CK(cudaFuncSetAttribute(sb2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  {
    const int spread = getenv("PSDPROJ_TRI_SPREAD") ? atoi(getenv("PSDPROJ_TRI_SPREAD")) : 1;
    CK(cudaMemcpyToSymbol(g_tri_bulk_spread, &spread, sizeof(int)));
  }
  done = true;
  return 0;
}

// L = chol(G) in place (t x t, ld); status = failing pivot + 1 or 0 (a6, R20)
// L = chol(G) in place; with Linv != nullptr also L^-1 (fused when it fits in shared memory, else a
// separate panel-streamed inverse). Returns 0 or a negative error.
static int trinv_run(cudaStream_t st, int t, const double* L, int ldl, double* Li, int ldi);
static int cholesky_run(cudaStream_t st, int t, double* G, int ld, int* d_status, double* gscratch = nullptr,
                        size_t gscratch_elems = 0, double* Linv = nullptr, int ldi = 0, int* started = nullptr,
                        int seq = 0) {
  TRY(cla_attrs());
  static int fuse = getenv("PSDPROJ_CHOL_NOFUSE") ? 0 : 1;
  const double frel = 1e-12;  // R20
  // an 8-CTA cluster when it holds the factor and its inverse (t <= ~300): measured ~1% faster per
  // LOBPCG step than 16 (fewer DSMEM peers per panel broadcast, easier to co-schedule with the
  // block multiply it overlaps)
  static int chol_cs = getenv("PSDPROJ_CHOL_CS") ? atoi(getenv("PSDPROJ_CHOL_CS")) : 8;
  if (Linv && fuse && t > 64 && chol_cs > 0 &&
      chol_inv_smem_doubles(t, chol_cs) * sizeof(double) <= (size_t)CLA_SMEM_BYTES) {
    return launch_cluster(cholesky_cluster_kernel<false, true>, chol_cs, CLA_NT,
                          chol_inv_smem_doubles(t, chol_cs) * sizeof(double), st, t, G, ld, 1e-12, d_status,
                          (double*)nullptr, Linv, ldi, started, seq);
  }
  if (Linv && fuse) {
    if (int cs = cla_cluster_size(t, chol_inv_smem_doubles)) {
      return launch_cluster(cholesky_cluster_kernel<false, true>, cs, CLA_NT,
                            chol_inv_smem_doubles(t, cs) * sizeof(double), st, t, G, ld, frel, d_status,
                            (double*)nullptr, Linv, ldi, started, seq);
    }
  }
  if (int cs = cla_cluster_size(t, chol_smem_doubles)) {
    TRY(launch_cluster(cholesky_cluster_kernel<false, false>, cs, CLA_NT, chol_smem_doubles(t, cs) * sizeof(double),
                       st, t, G, ld, frel, d_status, (double*)nullptr, (double*)nullptr, 0, started, seq));
    return Linv ? trinv_run(st, t, G, ld, Linv, ldi) : 0;
  }
  if (gscratch && (size_t)16 * chol_local_cols(t, 16) * t <= gscratch_elems && t <= 4096) {
    TRY(launch_cluster(cholesky_cluster_kernel<true, false>, 16, CLA_NT, chol_smem_doubles_ga(t, 16) * sizeof(double),
                       st, t, G, ld, frel, d_status, gscratch, (double*)nullptr, 0, started, seq));
    return Linv ? trinv_run(st, t, G, ld, Linv, ldi) : 0;
  }
  if (started) {
    set_int_kernel<<<1, 1, 0, st>>>(started, seq);
    CKL();
  }
  cholesky_kernel<1024><<<1, 1024, 0, st>>>(t, G, ld, frel, d_status);
  CKL();
  return Linv ? trinv_run(st, t, G, ld, Linv, ldi) : 0;
}

// Li = L^-1 (lower triangular t x t)
static int trinv_run(cudaStream_t st, int t, const double* L, int ldl, double* Li, int ldi) {
  TRY(cla_attrs());
  const size_t sm = (size_t)TI_KB * t * sizeof(double);
  const int g = cdiv(t, 8);
  if (t <= 32 * 8)
    trinv_panel_kernel<8><<<g, 256, sm, st>>>(t, L, ldl, Li, ldi);
  else if (t <= 32 * 16)
    trinv_panel_kernel<16><<<g, 256, sm, st>>>(t, L, ldl, Li, ldi);
  else if (t <= 32 * 24)
    trinv_panel_kernel<24><<<g, 256, sm, st>>>(t, L, ldl, Li, ldi);
  else if (t <= 32 * 40)
    trinv_panel_kernel<40><<<g, 256, sm, st>>>(t, L, ldl, Li, ldi);
  else
    return set_err(PSDPROJ_E_CAPACITY, "trinv supports t <= 1280");
  CKL();
  return 0;
}

// ------------------------------------------------------------------ tridiagonal eigensolver (a7)
// Top-m eigenpairs (descending) of the symmetric s x s matrix H: Householder tridiagonalisation
// (cluster_la.cuh for s <= CLA_MAX, one CTA above), multisection bisection, inverse iteration,
// back-transformation (tridiag.cuh), then two Newton-Schulz steps towards the polar factor
// Y <- Y (3I - Y^T Y)/2 restore orthonormality lost inside tight eigenvalue clusters (any
// orthonormal basis of a cluster's invariant subspace diagonalises H to the cluster width).
// With mgs = true the slow robust path (clustered modified Gram-Schmidt, dstein's rule) is used.
struct EighScratch {
  double *td, *te, *ttau, *te2, *tbounds, *tscr, *tG;
  int ldg;
  double* Vh;
  int ldv;
  double *nsM, *nsZ, *nsY;  // m x m, m x m, s x m (ld = ldv)
  unsigned long long* dev;   // NS deviation (double bits)
  size_t tscr_elems;
  void* mark_obj = nullptr;  // optional phase marker (profile bit 1): mark_fn(mark_obj, phase)
  int (*mark_fn)(void*, int) = nullptr;
  int mark(int ph) const { return mark_fn ? mark_fn(mark_obj, ph) : 0; }
  // optional timing of the tridiagonalisation launch (profile bit 2): tri_fn(mark_obj, 0 / 1) around it
  int (*tri_fn)(void*, int) = nullptr;
  int tri(int e) const { return tri_fn ? tri_fn(mark_obj, e) : 0; }
  // side stream + fork/join events for the T factors of the back-transformation (owned by the caller:
  // the context, or psdproj_eigh for the duration of its call)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_f = nullptr, ev_j = nullptr;
};

// `steps` Newton-Schulz steps Y <- Y (3I - Y^T Y) / 2; w.dev records max|Y^T Y - I| before the last
// one (the deviation after it is about 3/4 of its square).
static int ns_run(cudaStream_t st, int s, int m, double* Yv, int ldy, const EighScratch& w, double* part,
                  size_t part_elems, int steps) {
  for (int it = 0; it < steps; ++it) {
    TRY(dgemm(st, OP_T, OP_N, m, m, s, 1.0, Yv, ldy, Yv, ldy, 0.0, w.nsM, m, part, part_elems));
    const bool lastst = it == steps - 1;
    if (lastst) CK(cudaMemsetAsync(w.dev, 0, sizeof(unsigned long long), st));
    TRY(launch_pdl(ns_coeff_kernel, dim3(grid1d((size_t)m * m)), dim3(256), 0, st, m, (const double*)w.nsM, m, w.nsZ,
                   m, lastst ? w.dev : w.dev + 1));
    TRY(dgemm(st, OP_N, OP_N, s, m, m, 1.0, Yv, ldy, w.nsZ, m, 0.0, w.nsY, w.ldv, part, part_elems));
    TRY(copy_block_pdl(st, s, m, Yv, ldy, w.nsY, w.ldv));
  }
  return 0;
}

static int eigh_top(cudaStream_t st, int s, const double* Hs, int ldh, int m, double* lam, double* Yv, int ldy,
                    int* npos, const EighScratch& w, double* part, size_t part_elems, bool mgs, int ns_steps = 2) {
  TRY(cla_attrs());
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(tridiag_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)((size_t)(TRI_SMEM_MAX * (TRI_SMEM_MAX + 1) + 10 * TRI_SMEM_MAX) * sizeof(double))));
    CK(cudaFuncSetAttribute(tri_inviter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(tri_twisted_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(tri_bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    CK(cudaFuncSetAttribute(tri_bisect_ms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    attr = true;
  }
  if (s > EIG_MAX) return set_err(PSDPROJ_E_CAPACITY, "eigensolver supports s <= %d", EIG_MAX);
  static int tri_mode = -1;  // 0 auto, 1 force one-CTA
  if (tri_mode < 0) tri_mode = getenv("PSDPROJ_TRI_ONECTA") ? 1 : 0;
  int tcs = (tri_mode == 0 && s > 64) ? cla_cluster_size(s, tri_smem_doubles) : 0;
  static long long* dprof = nullptr;
  static int want_prof = getenv("PSDPROJ_TRI_PROF") ? 1 : 0;
  static int tri_dbg = getenv("PSDPROJ_TRI_DBG") ? atoi(getenv("PSDPROJ_TRI_DBG")) : 0;  // timing experiments only
  if (want_prof && !dprof) CK(cudaMalloc(&dprof, 16 * 12 * sizeof(long long)));
  if (want_prof) CK(cudaMemsetAsync(dprof, 0, 16 * 12 * sizeof(long long), st));
  TRY(w.tri(0));
  // one-CTA tiled tridiagonalisation (tridiag_tile.cuh) up to s = PSDPROJ_TRI_TILE (default 64: measured
  // 145 vs 234 us at s = 64 against the one-CTA shared-memory kernel; the 16-CTA cluster kernel is
  // faster from s ~ 100 up, 230 vs 339 us at s = 128, 567 vs 1183 us at s = 256 -- DESIGN.md §6)
  static const int tri_tile = getenv("PSDPROJ_TRI_TILE") ? atoi(getenv("PSDPROJ_TRI_TILE")) : 64;
  // two-stage reduction (sbr.cuh: dense -> band on a 16-CTA cluster, band -> tridiagonal in one CTA) for
  // PSDPROJ_SBR_MIN <= s <= PSDPROJ_SBR_MAX when its shared memory and the scratch fit
  static const int sbr_min = getenv("PSDPROJ_SBR_MIN") ? atoi(getenv("PSDPROJ_SBR_MIN")) : 96;
  static const int sbr_max = getenv("PSDPROJ_SBR_MAX") ? atoi(getenv("PSDPROJ_SBR_MAX")) : SB_MAX;
  static const int sbr_on = getenv("PSDPROJ_SBR") ? atoi(getenv("PSDPROJ_SBR")) : 0;  // measured slower
  const bool use_sbr = sbr_on && tri_mode == 0 && s >= std::max(sbr_min, 3 * SB) && s <= std::min(sbr_max, SB_MAX) &&
                       sb1_smem_doubles(s, 16) * sizeof(double) <= (size_t)CLA_SMEM_BYTES &&
                       ((size_t)s * SB_LDW + SB2_NW * SB + s) * sizeof(double) <= (size_t)CLA_SMEM_BYTES &&
                       sb_refl_doubles(s) + (size_t)SB_LDW * s <= (size_t)s * s;
  double* sb_Vr = w.tG;
  double* sb_Bg = w.tG + (size_t)s * s - (size_t)SB_LDW * s;
  double* sb_Tq = w.tG + (size_t)s * s;
  if (use_sbr) {
    TRY(launch_cluster(sb1_kernel, 16, SB1_NT, sb1_smem_doubles(s, 16) * sizeof(double), st, s, Hs, ldh, sb_Bg, w.Vh,
                       w.ldv, sb_Tq));
    sb2_kernel<<<1, SB2_NW * 32, ((size_t)s * SB_LDW + SB2_NW * SB + s) * sizeof(double), st>>>(s, sb_Bg, w.td, w.te,
                                                                                            sb_Vr);
    CKL();
    tcs = 0;
  }
  // one-CTA warp-cyclic register kernel (tridiag_warp.cuh: two CTA barriers per column, no DSMEM hop)
  // up to s = PSDPROJ_TRI_WARP (default 64: 87 vs 145 us for the tiled kernel at s = 64; its 4 x 8
  // register variant measured 216 / 276 us at s = 100 / 128 against 170 / 230 us for the 16-CTA
  // cluster kernel, so s > 64 stays on the cluster -- DESIGN.md §6)
  static const int tri_warp = getenv("PSDPROJ_TRI_WARP") ? atoi(getenv("PSDPROJ_TRI_WARP")) : 64;
  const bool use_warp = !use_sbr && tri_mode == 0 && s >= 3 && s <= std::min(tri_warp, 128);
  if (use_warp) {
    if (s <= 64)
      tridiag_warp_kernel<2, 4><<<1, TW_NT, 0, st>>>(s, Hs, ldh, w.td, w.te, w.ttau, w.Vh, w.ldv);
    else
      tridiag_warp_kernel<4, 8><<<1, TW_NT, 0, st>>>(s, Hs, ldh, w.td, w.te, w.ttau, w.Vh, w.ldv);
    CKL();
    tcs = 0;
  }
  const bool use_tile = !use_warp && !use_sbr && tri_mode == 0 && s >= 3 && s <= std::min(tri_tile, TT_SMAX);
  if (use_tile) {
    static bool tattr = false;
    if (!tattr) {
      CK(cudaFuncSetAttribute(tridiag_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(tri_tile_smem_doubles(TT_SMAX) * sizeof(double))));
      tattr = true;
    }
    tridiag_tile_kernel<<<1, TT_NT, tri_tile_smem_doubles(s) * sizeof(double), st>>>(s, Hs, ldh, w.td, w.te, w.ttau,
                                                                                      w.Vh, w.ldv);
    CKL();
    tcs = 0;
  }
#define TRI_LAUNCH(PL, NTH, GA, CSZ, SMEM)                                                                         \
  TRY(launch_cluster(tridiag_cluster_kernel<PL, NTH, GA>, CSZ, NTH, SMEM, st, s, Hs, ldh, w.td, w.te, w.ttau, w.Vh, \
                     w.ldv, dprof, w.tG, tri_dbg))
  static int tri_reg = getenv("PSDPROJ_TRI_NOREG") ? 0 : 1;
  const int kr = cdiv(s, 64), cr = tcs ? cdiv(cdiv(s, tcs), TRI_TCG) : 99;
  if (use_warp || use_tile || use_sbr) {
    // done above
  } else if (tcs && tri_reg && kr <= 8 && cr <= 8 &&
      tri_reg_smem_doubles(s, tcs) * sizeof(double) <= (size_t)CLA_SMEM_BYTES) {
    const size_t tsm = tri_reg_smem_doubles(s, tcs) * sizeof(double);
    // one-hop variant (tridiag_rep.cuh): the step's column replicated in every CTA a step ahead
    static const int tri_rep = getenv("PSDPROJ_TRI_REP") ? atoi(getenv("PSDPROJ_TRI_REP")) : 0;
    const size_t tsm_rep = tri_rep_smem_doubles(s, tcs) * sizeof(double);
    const bool rep = tri_rep && !want_prof && tsm_rep <= (size_t)CLA_SMEM_BYTES;
#define TRI_REG(KR, CR)                                                                                              \
  if (rep)                                                                                                          \
    TRY(launch_cluster(tridiag_rep_kernel<KR, CR>, tcs, 256, tsm_rep, st, s, Hs, ldh, w.td, w.te, w.ttau, w.Vh, w.ldv)); \
  else                                                                                                              \
    TRY(launch_cluster(tridiag_reg_kernel<KR, CR>, tcs, 256, tsm, st, s, Hs, ldh, w.td, w.te, w.ttau, w.Vh, w.ldv, dprof, tri_dbg))
    if (kr <= 3 && cr <= 5)
      TRI_REG(3, 5);
    else if (kr <= 4 && cr <= 4)
      TRI_REG(4, 4);
    else if (kr <= 6 && cr <= 6)
      TRI_REG(6, 6);
    else if (kr <= 7 && cr <= 7)
      TRI_REG(7, 7);
    else
      TRI_REG(8, 8);
#undef TRI_REG
    static int verify = getenv("PSDPROJ_TRI_VERIFY") ? 1 : 0;  // debugging: compare with the smem kernel
    if (verify) {
      static double* vb = nullptr;
      if (!vb) CK(cudaMalloc(&vb, sizeof(double) * ((size_t)2 * EIG_MAX * EIG_MAX + 4 * EIG_MAX)));
      double *vd = vb, *ve = vb + EIG_MAX, *vt = vb + 2 * EIG_MAX, *vV = vb + 4 * EIG_MAX;
      const size_t tsm2 = tri_smem_doubles(s, tcs) * sizeof(double);
      if (s <= 32 * 8)
        TRY(launch_cluster(tridiag_cluster_kernel<8, 512>, tcs, 512, tsm2, st, s, Hs, ldh, vd, ve, vt, vV, w.ldv,
                           (long long*)nullptr, w.tG, 0));
      else if (s <= 32 * 14)
        TRY(launch_cluster(tridiag_cluster_kernel<14, 256>, tcs, 256, tsm2, st, s, Hs, ldh, vd, ve, vt, vV, w.ldv,
                           (long long*)nullptr, w.tG, 0));
      else
        TRY(launch_cluster(tridiag_cluster_kernel<20, 256>, tcs, 256, tsm2, st, s, Hs, ldh, vd, ve, vt, vV, w.ldv,
                           (long long*)nullptr, w.tG, 0));
      CK(cudaStreamSynchronize(st));
      std::vector<double> a1(2 * s), a2(2 * s);
      CK(cudaMemcpy(a1.data(), w.td, s * sizeof(double), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(a1.data() + s, w.te, (s - 1) * sizeof(double), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(a2.data(), vd, s * sizeof(double), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(a2.data() + s, ve, (s - 1) * sizeof(double), cudaMemcpyDeviceToHost));
      double mx = 0, df = 0;
      int at = -1;
      for (int i = 0; i < 2 * s - 1; ++i) {
        mx = std::max(mx, std::fabs(a2[i]));
        const double dd = std::fabs(std::fabs(a1[i]) - std::fabs(a2[i]));
        if (!(dd <= df)) { df = dd; at = i; }
      }
      {
        // reflectors: tau and Vh columns 0..s-3 (rows below the diagonal)
        std::vector<double> t1(s), t2(s), V1((size_t)s * w.ldv), V2((size_t)s * w.ldv);
        CK(cudaMemcpy(t1.data(), w.ttau, (s - 2) * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(t2.data(), vt, (s - 2) * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(V1.data(), w.Vh, (size_t)s * w.ldv * sizeof(double), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(V2.data(), vV, (size_t)s * w.ldv * sizeof(double), cudaMemcpyDeviceToHost));
        double dt = 0, dv = 0;
        int atv = -1;
        for (int g = 0; g + 2 < s; ++g) {
          dt = std::max(dt, std::fabs(t1[g] - t2[g]));
          for (int i = g + 1; i < s; ++i) {
            const double dd = std::fabs(V1[(size_t)g * w.ldv + i] - V2[(size_t)g * w.ldv + i]);
            if (!(dd <= dv)) { dv = dd; atv = g; }
          }
        }
        if (!(dt <= 1e-9) || !(dv <= 1e-9)) {
          fprintf(stderr, "TRI_VERIFY s=%d cs=%d: tau diff %g, Vh diff %g (column %d)\n", s, tcs, dt, dv, atv);
          df = 1.0;
          mx = 0.0;
        }
      }
      if (!(df <= 1e-10 * mx)) {
        static int nb = 0;
        fprintf(stderr, "TRI_VERIFY s=%d cs=%d: max |d,e| diff %g at %d (scale %g)\n", s, tcs, df, at, mx);
        if (nb < 3) {
          std::vector<double> H((size_t)s * s);
          CK(cudaMemcpy2D(H.data(), s * sizeof(double), Hs, (size_t)ldh * sizeof(double), s * sizeof(double), s,
                          cudaMemcpyDeviceToHost));
          char fn[128];
          snprintf(fn, sizeof fn, "gpurun_out/tri_bad_%d.bin", nb++);
          if (FILE* f = fopen(fn, "wb")) {
            fwrite(H.data(), sizeof(double), H.size(), f);
            fclose(f);
          }
        }
      }
    }
  } else if (tcs) {
    const size_t tsm = tri_smem_doubles(s, tcs) * sizeof(double);
    if (s <= 32 * 4)
      TRI_LAUNCH(4, 512, false, tcs, tsm);
    else if (s <= 32 * 8)
      TRI_LAUNCH(8, 512, false, tcs, tsm);
    else if (s <= 32 * 14)
      TRI_LAUNCH(14, 256, false, tcs, tsm);
    else
      TRI_LAUNCH(20, 256, false, tcs, tsm);
  } else if (tri_mode == 0 && s > 64 && s <= EIG_MAX) {
    // too large for shared memory: own columns in the L2-resident scratch tG (16-CTA cluster)
    const size_t tsm = tri_smem_doubles_ga(s, 16) * sizeof(double);
    if (s <= 32 * 24)
      TRI_LAUNCH(24, 256, true, 16, tsm);
    else if (s <= 32 * 40)
      TRI_LAUNCH(40, 256, true, 16, tsm);
    else
      TRI_LAUNCH(64, 256, true, 16, tsm);
  } else {
    const size_t vecs = (size_t)s * 10;
    size_t dyn = ((s <= TRI_SMEM_MAX) ? (size_t)s * (s + 1) : 0) + vecs;
    dyn *= sizeof(double);
    if (s > TRI_SMEM_MAX && dyn > 200 * 1024) return set_err(PSDPROJ_E_CAPACITY, "tridiag smem %zu for s=%d", dyn, s);
    tridiag_kernel<1024><<<1, 1024, dyn, st>>>(s, Hs, ldh, w.td, w.te, w.ttau, w.Vh, w.ldv, w.tG, w.ldg);
    CKL();
  }
#undef TRI_LAUNCH
  TRY(w.tri(1));
  if (want_prof && tcs) {
    long long h[192];
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(h, dprof, sizeof(h), cudaMemcpyDeviceToHost));
    for (int r = 0; r < std::min(tcs, 3); ++r)
      fprintf(stderr, "tri prof s=%d cs=%d rank %d: house %lld B1 %lld vgather %lld cols %lld B2 %lld U2 %lld D %lld (cycles/step) owner-steps %lld house/owner-step %lld\n",
              s, tcs, r, h[r * 8 + 0] / (s - 2), h[r * 8 + 1] / (s - 2), h[r * 8 + 2] / (s - 2), h[r * 8 + 3] / (s - 2),
              h[r * 8 + 4] / (s - 2), h[r * 8 + 5] / (s - 2), h[r * 8 + 6] / (s - 2), h[r * 8 + 7],
              h[r * 8 + 7] ? h[r * 8 + 0] / h[r * 8 + 7] : 0);
    for (int r = 0; r < std::min(tcs, 3); ++r)
      if (h[r * 8 + 7])
        fprintf(stderr, "   owner-step: U1 %lld syncthreads %lld scalars %lld (cycles)\n", h[128 + r * 4] / h[r * 8 + 7],
                h[128 + r * 4 + 1] / h[r * 8 + 7], h[128 + r * 4 + 2] / h[r * 8 + 7]);
  }
  static int dbg_eigh = getenv("PSDPROJ_DEBUG_EIGH") ? 1 : 0;
  if (dbg_eigh) {
    double hb[4] = {0, 0, 0, 0};
    cudaError_t e0 = cudaStreamSynchronize(st);
    cudaMemcpy(hb, w.td, sizeof(double) * std::min(s, 4), cudaMemcpyDeviceToHost);
    fprintf(stderr, "eigh s=%d m=%d mgs=%d tcs=%d sync=%s d0=%g\n", s, m, (int)mgs, tcs, cudaGetErrorString(e0), hb[0]);
  }
  TRY(w.mark(8));
  static int bt_mode = -1;  // 0: compact-WY (default for s <= 640), 1: reflector-by-reflector panels
  if (bt_mode < 0) bt_mode = getenv("PSDPROJ_BT_SIMPLE") ? 1 : 0;
  // one-CTA-per-column WY apply when the m CTAs fit in one wave (s <= 768)
  static const int bt_col = getenv("PSDPROJ_BT_WARP") ? 0 : 1;
  const size_t bt_col_smem = bt_col_smem_doubles(s) * sizeof(double);
  const bool col_ok = bt_col && s <= 768 && bt_col_smem <= (size_t)CLA_SMEM_BYTES &&
                      m <= sms() * (int)std::max<size_t>(1, (size_t)(228 * 1024) / (bt_col_smem + 1024));
  const bool wy = !use_sbr && s > 2 && bt_mode == 0 && (s <= 32 * 20 || col_ok) && m > 0;
  cudaEvent_t tri_side_join = nullptr;
  if (wy) {
    cudaStream_t side = w.side;
    cudaEvent_t ev_f = w.ev_f, ev_j = w.ev_j;
    if (!side || !ev_f || !ev_j) return set_err(PSDPROJ_E_INVALID, "eigensolver side stream missing");
    // the T factors of the compact-WY back-transformation need only the reflectors: computed on a
    // side stream, hidden behind the bisection and inverse iteration (the stream and events belong to
    // the caller's context, so concurrent contexts never share them)
    CK(cudaEventRecord(ev_f, st));
    CK(cudaStreamWaitEvent(side, ev_f, 0));
    larft_kernel<<<cdiv(s - 2, WY_PB), 256, 0, side>>>(s, w.Vh, w.ldv, w.ttau, w.tG);
    CKL();
    CK(cudaEventRecord(ev_j, side));
    tri_side_join = ev_j;
  }
  tri_prep_kernel<<<1, 1024, 0, st>>>(s, w.td, w.te, w.te2, w.tbounds);
  CKL();
  {
    // multisection points per eigenvalue (PSDPROJ_BISECT_G, multiple of 32; 32 = one warp each)
    static const int bg = getenv("PSDPROJ_BISECT_G") ? std::max(32, std::min(1024, atoi(getenv("PSDPROJ_BISECT_G")) / 32 * 32)) : 256;
    if (bg == 32) {
      tri_bisect_kernel<<<cdiv(m + 1, 2), 64, (size_t)2 * s * sizeof(double), st>>>(s, m, w.td, w.te2, w.tbounds, lam,
                                                                                    npos);
      CKL();
    } else {
      TRY(launch_pdl(tri_bisect_ms_kernel, dim3(m + 1), dim3(bg), (size_t)2 * s * sizeof(double), st, s, m,
                     (const double*)w.td, (const double*)w.te2, (const double*)w.tbounds, lam, npos));
    }
  }
  if (m <= 0) return 0;  // (wy is false for m <= 0: no side-stream work in flight)
  TRY(w.mark(9));
  // inverse iteration: vectors per CTA so that the per-thread arrays fit in shared memory
  int vpb = 64;
  while (vpb > 1 && tri_inviter_smem_bytes(s, vpb) > (size_t)220 * 1024) --vpb;
  int smem_ok = tri_inviter_smem_bytes(s, vpb) <= (size_t)220 * 1024;
  if (!smem_ok) vpb = 64;
  if (!smem_ok && (size_t)6 * s * (size_t)m > w.tscr_elems) return set_err(PSDPROJ_E_CAPACITY, "eigensolver scratch");
  size_t ism = smem_ok ? tri_inviter_smem_bytes(s, vpb) : (size_t)2 * s * sizeof(double);
  if (mgs) {
    for (int pass = 0; pass < 2; ++pass) {
      tri_inviter_kernel<<<cdiv(m, vpb), vpb, ism, st>>>(s, m, w.td, w.te, lam, w.tbounds, Yv, ldy, w.tscr,
                                                         pass ? 1 : 2, pass, smem_ok);
      CKL();
      tri_cluster_mgs_kernel<1024><<<1, 1024, 0, st>>>(s, m, lam, w.tbounds, Yv, ldy);
      CKL();
    }
  } else {
    static int twisted = getenv("PSDPROJ_INVITER") ? 0 : 1;
    if (twisted && (size_t)(7 * s + 2) * sizeof(double) <= (size_t)220 * 1024) {
      TRY(launch_pdl(tri_twisted_kernel, dim3(m), dim3(32), (size_t)(7 * s + 2) * sizeof(double), st, s, m,
                     (const double*)w.td, (const double*)w.te, (const double*)lam, Yv, ldy));
    } else {
      tri_inviter_kernel<<<cdiv(m, vpb), vpb, ism, st>>>(s, m, w.td, w.te, lam, w.tbounds, Yv, ldy, w.tscr, 2, 0,
                                                         smem_ok);
      CKL();
    }
  }
  TRY(w.mark(10));
  if (s > 2 && use_sbr) {
    sbr_bt_kernel<<<m, SBT_NT, (size_t)(s + 2 * SB) * sizeof(double), st>>>(s, m, sb_Vr, w.Vh, w.ldv, sb_Tq, Yv, ldy);
    CKL();
  } else if (s > 2) {
    if (wy) {
      double* Tb = w.tG;  // T factors from larft_kernel (side stream, launched after the tridiagonalisation)
      CK(cudaStreamWaitEvent(st, tri_side_join, 0));
#define BT_WY(PL)                                                                                          \
  backtransform_wy_kernel<PL, 4><<<cdiv(m, 4), 128, bt_wy_smem_doubles(PL, 4) * sizeof(double), st>>>( \
      s, m, w.Vh, w.ldv, Tb, Yv, ldy)
#define BT_COL(PLW)                                                                                        \
  backtransform_wy_col_kernel<PLW><<<m, 256, bt_col_smem_doubles(s) * sizeof(double), st>>>(s, m, w.Vh, w.ldv, \
                                                                                           Tb, Yv, ldy)
      if (col_ok) {
        if (s <= 256)
          BT_COL(1);
        else if (s <= 512)
          BT_COL(2);
        else
          BT_COL(3);
      } else if (s <= 32 * 8)
        BT_WY(8);
      else if (s <= 32 * 16)
        BT_WY(16);
      else
        BT_WY(20);
#undef BT_WY
#undef BT_COL
      CKL();
    } else {
    const int pb = (int)std::max<size_t>(1, std::min<size_t>(BT_PB, (size_t)CLA_SMEM_BYTES / (2 * (size_t)s * sizeof(double))));
    const size_t bsm = (size_t)2 * pb * s * sizeof(double);
    if (s <= 32 * 8)
      backtransform_panel_kernel<8><<<cdiv(m, 8), 256, bsm, st>>>(s, m, w.Vh, w.ldv, w.ttau, Yv, ldy, pb);
    else if (s <= 32 * 16)
      backtransform_panel_kernel<16><<<cdiv(m, 8), 256, bsm, st>>>(s, m, w.Vh, w.ldv, w.ttau, Yv, ldy, pb);
    else if (s <= 32 * 24)
      backtransform_panel_kernel<24><<<cdiv(m, 8), 256, bsm, st>>>(s, m, w.Vh, w.ldv, w.ttau, Yv, ldy, pb);
    else if (s <= 32 * BT_PER_LANE)
      backtransform_panel_kernel<BT_PER_LANE><<<cdiv(m, 8), 256, bsm, st>>>(s, m, w.Vh, w.ldv, w.ttau, Yv, ldy, pb);
    else
      backtransform_panel_kernel<64><<<cdiv(m, 8), 256, bsm, st>>>(s, m, w.Vh, w.ldv, w.ttau, Yv, ldy, pb);
    }
    CKL();
  }
  TRY(w.mark(11));
  if (!mgs) {
    TRY(ns_run(st, s, m, Yv, ldy, w, part, part_elems, ns_steps));
  }
  return 0;
}

// ------------------------------------------------------------------ context
struct psdproj_ctx_s {
  int n = 0, ld = 0;
  // row-sharded mode (§8.e): this rank holds rows [row0, row0 + nr) of every n-sized block; the
  // tall-skinny buffers have nr rows (ld = rup(nr, 8)); Gram / norm partials are all-reduced, the
  // block multiply gathers Z. Unsharded: nr = n, row0 = 0, nranks = 1.
  bool sharded = false;
  int rank = 0, nranks = 1, row0 = 0, nr = 0, nrmax = 0, ldn = 0;
  ncclComm_t comm = nullptr;
  int *d_rows = nullptr, *d_offs = nullptr;
  double *zsend = nullptr, *zpack = nullptr, *zfull = nullptr, *gbuf = nullptr;
  psdproj_params prm{};
  int m0 = 0, q = 0, m_max = 0, s_max = 0, NJ = 0, tcols = 0;
  // device (carved from the caller's workspace)
  double *S = nullptr, *BS = nullptr, *S2 = nullptr, *BS2 = nullptr, *T = nullptr, *T2 = nullptr, *E = nullptr;
  double *Pb = nullptr, *BPb = nullptr, *R = nullptr, *Xw = nullptr;
  double *G = nullptr, *Hm = nullptr, *Gc = nullptr, *Li = nullptr, *Y = nullptr, *Hh = nullptr, *Vj = nullptr,
         *Cp = nullptr;
  double *jM = nullptr, *jM2 = nullptr, *jQ = nullptr;
  double* part = nullptr;
  size_t part_elems = 0;
  double *d_thU = nullptr, *d_r = nullptr, *d_norm = nullptr, *d_w = nullptr, *d_ths = nullptr, *d_scal = nullptr;
  int *d_idx = nullptr, *d_order = nullptr, *d_status = nullptr, *d_counters = nullptr;
  double* stage = nullptr;  // host_io staging (n x n, ld)
  // tridiagonal eigensolver scratch (a7)
  double *td = nullptr, *te = nullptr, *ttau = nullptr, *te2 = nullptr, *tbounds = nullptr, *tscr = nullptr,
         *tG = nullptr;
  int* tnpos = nullptr;
  size_t tscr_elems = 0;
  // pinned host mirrors
  double* h_d = nullptr;
  int* h_i = nullptr;
  size_t h_d_len = 0, h_i_len = 0;
  // host state
  bool warm = false;
  int block_side = 0, m_warm = 0;
  std::vector<double> th_warm;
  bool have_counts = false;
  int last_pos = 0, last_neg = 0;
  int calls = 0;
  bool poisoned = false;
  std::vector<cudaEvent_t> ev;
  std::vector<cudaEvent_t> pev;  // phase-timing events (profile & 2)
  // side stream: the direction-block Gram and its Cholesky run there, overlapping the block multiply
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int* d_flag = nullptr;  // residency signal of the side-stream Cholesky (sequence number)
  // eigensolver side stream (T factors of the back-transformation) and its fork/join events
  cudaStream_t st3 = nullptr;
  cudaEvent_t ev3_f = nullptr, ev3_j = nullptr;
  std::vector<cudaEvent_t> tev;  // tridiagonalisation timing events (profile & 4)
  // psdproj_project_batched: this context's stream and fork / join events (created on first use)
  cudaStream_t bst = nullptr;
  cudaEvent_t bev_fork = nullptr, bev_join = nullptr;
  int chol_seq = 0;
  double* part2 = nullptr;
};

struct Carver {
  char* base;
  size_t off, cap;
  bool dry;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) / 256 * 256;
    T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
};

static void resolve(int n, const psdproj_params* in, psdproj_params& p, int& m0, int& q, int& m_max, int& s_max,
                    int& NJ, int& tcols, bool sharded = false) {
  if (in)
    p = *in;
  else
    psdproj_default_params(&p);
  m0 = p.m0 > 0 ? std::min(p.m0, n) : std::max(1, (int)std::ceil(0.1 * n));
  q = p.expand_q > 0 ? p.expand_q : std::max(1, (int)std::ceil(0.05 * n));
  // default capacity n/3: a wider block is the exact-eig regime anyway (R18)
  m_max = p.m_max > 0 ? std::min(p.m_max, n) : std::min(n, (n + 2) / 3 + 1);
  m_max = std::max(m_max, std::min(n, m0));
  const int dpt = std::max(1, p.krylov_depth);
  m_max = std::max(1, std::min(m_max, (EIG_MAX - q) / (dpt + 2)));  // the RR basis (<= (d + 2) m + q) must fit the eigensolver
  m_max = std::max(1, std::min(m_max, (TRINV_MAX - q) / (dpt + 1)));  // and its direction block (<= (d + 1) m + q) the L^-1 kernel
  m0 = std::min(m0, m_max);
  s_max = (dpt + 2) * m_max + q;
  // the DIRECT path (tridiagonal eigensolver for n <= EIG_MAX) runs in the s_max-sized eigensolver
  // scratch (reflectors, column store, Newton-Schulz buffers): keep s_max >= n there
  if (!sharded && n <= EIG_MAX) s_max = std::max(s_max, n);
  NJ = sharded ? s_max : std::max(s_max, n);  // the sharded mode has no DIRECT path
  NJ += NJ & 1;
  tcols = sharded ? s_max : std::max(s_max, n);
}

static size_t carve(psdproj_ctx_s* c, int n, const psdproj_params& p, int m_max, int s_max, int NJ, int tcols,
                    char* base, size_t cap, bool dry, int nl = -1, int nranks = 1, int nrmax = 0) {
  Carver cv{base, 0, cap, dry};
  if (nl < 0) nl = n;
  int ld = rup(std::max(nl, 1), 8);
  size_t nS = (size_t)ld * s_max, nM = (size_t)ld * m_max, nT = (size_t)ld * tcols, s2 = (size_t)s_max * s_max;
  // S, BS and their rotation targets each carry an m_max-column prefix: the hard-locked block X_L (and
  // B X_L) lives right-aligned in front of S (mirrored in front of S2), so [X_L | X_U] is one
  // contiguous n x (nL + mU) block for the projections (one Gram and one update GEMM, not two)
  const size_t pre = (size_t)ld * m_max;
  c->S = cv.take<double>(nS + pre); c->BS = cv.take<double>(nS + pre);
  c->S2 = cv.take<double>(nS + pre); c->BS2 = cv.take<double>(nS + pre);
  if (!dry) {
    c->S += pre; c->BS += pre; c->S2 += pre; c->BS2 += pre;
  }
  c->T = cv.take<double>(nT); c->T2 = cv.take<double>(nT);
  c->E = cv.take<double>(nT);
  c->Pb = cv.take<double>(nM); c->BPb = cv.take<double>(nM);
  c->R = cv.take<double>(nM); c->Xw = cv.take<double>(nM);
  c->G = cv.take<double>(s2); c->Hm = cv.take<double>(s2); c->Gc = cv.take<double>(s2);
  c->Li = cv.take<double>(s2); c->Y = cv.take<double>(s2); c->Hh = cv.take<double>(s2);
  c->Vj = cv.take<double>(s2); c->Cp = cv.take<double>(s2);
  size_t nj = (size_t)NJ * NJ;
  c->jM = cv.take<double>(nj); c->jM2 = cv.take<double>(nj); c->jQ = cv.take<double>(nj);
  c->part_elems = 2 * std::max(s2, nM);
  c->part = cv.take<double>(c->part_elems);
  c->part2 = cv.take<double>(c->part_elems);
  int vlen = std::max(s_max, n) + 8;
  c->d_thU = cv.take<double>(vlen); c->d_r = cv.take<double>(vlen); c->d_norm = cv.take<double>(vlen);
  c->d_w = cv.take<double>(vlen); c->d_ths = cv.take<double>(vlen); c->d_scal = cv.take<double>(64);
  c->d_idx = cv.take<int>((size_t)8 * (std::max(s_max, n) + 64)); c->d_order = cv.take<int>(vlen); c->d_status = cv.take<int>(64);
  c->d_counters = cv.take<int>(128);
  c->stage = p.host_io ? cv.take<double>((size_t)ld * n) : nullptr;
  c->td = cv.take<double>(vlen); c->te = cv.take<double>(vlen); c->ttau = cv.take<double>(vlen);
  c->te2 = cv.take<double>(vlen); c->tbounds = cv.take<double>(8); c->tnpos = cv.take<int>(8);
  c->tscr_elems = (size_t)6 * s_max * (size_t)(std::min(s_max, m_max + (s_max - 3 * m_max)) + 1);
  c->tscr = cv.take<double>(c->tscr_elems);
  c->tG = cv.take<double>(s2 + 16 * (size_t)s_max + 2048);  // also the GA tridiagonalisation scratch
  if (nranks > 1 || nl != n || nrmax > 0) {  // row-sharded buffers
    const int ldn = rup(n, 8);
    const size_t nz = (size_t)std::max(nrmax, 1) * s_max;
    c->zsend = cv.take<double>(nz);
    c->zpack = cv.take<double>(nz * nranks);
    c->zfull = cv.take<double>((size_t)ldn * s_max);
    c->gbuf = cv.take<double>(s2);
    c->d_rows = cv.take<int>(nranks + 8);
    c->d_offs = cv.take<int>(nranks + 8);
  }
  return cv.off + 256;
}

extern "C" void psdproj_default_params(psdproj_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->max_iter = 500;
  p->guard = 1;
  p->side = PSDPROJ_SIDE_AUTO;
  p->locking = PSDPROJ_LOCK_HARD;
  p->keep_extra = -1;
  p->seed = 0x5eed1912ull;
}

extern "C" size_t psdproj_workspace_bytes(int n, const psdproj_params* in) {
  if (n <= 0) return 0;
  psdproj_params p;
  int m0, q, m_max, s_max, NJ, tcols;
  resolve(n, in, p, m0, q, m_max, s_max, NJ, tcols);
  psdproj_ctx_s tmp;
  return carve(&tmp, n, p, m_max, s_max, NJ, tcols, nullptr, 0, true);
}

extern "C" int psdproj_create(int n, const psdproj_params* in, void* ws, size_t ws_bytes, psdproj_ctx* out) {
  if (!out) return set_err(PSDPROJ_E_INVALID, "out is NULL");
  *out = nullptr;
  if (n <= 0) return set_err(PSDPROJ_E_INVALID, "n must be positive (got %d)", n);
  if (!ws || ((uintptr_t)ws & 255)) return set_err(PSDPROJ_E_WORKSPACE, "workspace NULL or not 256-byte aligned");
  psdproj_params p;
  int m0, q, m_max, s_max, NJ, tcols;
  resolve(n, in, p, m0, q, m_max, s_max, NJ, tcols);
  if (p.max_iter < 0 || p.guard < 1 || (p.locking != PSDPROJ_LOCK_SOFT && p.locking != PSDPROJ_LOCK_HARD) ||
      (p.side != 0 && p.side != 1 && p.side != -1 && p.side != 2))
    return set_err(PSDPROJ_E_INVALID, "invalid params");
  psdproj_ctx_s tmp;
  size_t need = carve(&tmp, n, p, m_max, s_max, NJ, tcols, nullptr, 0, true);
  if (ws_bytes < need) return set_err(PSDPROJ_E_WORKSPACE, "workspace %zu < needed %zu", ws_bytes, need);
  auto* c = new psdproj_ctx_s();
  c->n = n;
  c->ld = rup(n, 8);
  c->ldn = c->ld;
  c->nr = n;
  c->prm = p;
  c->m0 = m0; c->q = q; c->m_max = m_max; c->s_max = s_max; c->NJ = NJ; c->tcols = tcols;
  carve(c, n, p, m_max, s_max, NJ, tcols, (char*)ws, ws_bytes, false);
  c->h_d_len = (size_t)4 * (std::max(s_max, n) + 64);
  c->h_i_len = (size_t)8 * (std::max(s_max, n) + 64);
  if (cudaMallocHost(&c->h_d, c->h_d_len * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&c->h_i, c->h_i_len * sizeof(int)) != cudaSuccess) {
    delete c;
    return set_err(PSDPROJ_E_CUDA, "cudaMallocHost failed");
  }
  *out = c;
  return PSDPROJ_OK;
}

extern "C" int psdproj_get_nccl_uid(void* uid_out) {
  if (!uid_out) return set_err(PSDPROJ_E_INVALID, "uid_out NULL");
  TRY(nccl_load());
  ncclUniqueId id;
  NK(g_nccl.getUniqueId(&id));
  std::memcpy(uid_out, &id, sizeof(id));
  return PSDPROJ_OK;
}

extern "C" size_t psdproj_workspace_bytes_sharded(int n, int nrows_max, int nranks, const psdproj_params* in) {
  if (n <= 0 || nrows_max <= 0 || nranks <= 0) return 0;
  psdproj_params p;
  int m0, q, m_max, s_max, NJ, tcols;
  resolve(n, in, p, m0, q, m_max, s_max, NJ, tcols, true);
  psdproj_ctx_s tmp;
  return carve(&tmp, n, p, m_max, s_max, NJ, tcols, nullptr, 0, true, nrows_max, nranks, nrows_max);
}

extern "C" int psdproj_create_sharded(int n, int row0, int nrows, const void* nccl_uid, int rank, int nranks,
                                      const psdproj_params* in, void* ws, size_t ws_bytes, psdproj_ctx* out) {
  if (!out) return set_err(PSDPROJ_E_INVALID, "out is NULL");
  *out = nullptr;
  if (n <= 0 || nrows <= 0 || row0 < 0 || row0 + nrows > n || nranks <= 0 || rank < 0 || rank >= nranks || !nccl_uid)
    return set_err(PSDPROJ_E_INVALID, "invalid sharded arguments (n=%d row0=%d nrows=%d rank=%d/%d)", n, row0, nrows,
                   rank, nranks);
  if (!ws || ((uintptr_t)ws & 255)) return set_err(PSDPROJ_E_WORKSPACE, "workspace NULL or not 256-byte aligned");
  psdproj_params p;
  int m0, q, m_max, s_max, NJ, tcols;
  resolve(n, in, p, m0, q, m_max, s_max, NJ, tcols, true);
  if (p.side == PSDPROJ_SIDE_DIRECT || p.host_io) return set_err(PSDPROJ_E_INVALID, "sharded mode: no DIRECT side / host_io");
  TRY(nccl_load());
  ncclComm_t comm;
  ncclUniqueId id;
  std::memcpy(&id, nccl_uid, sizeof(id));
  NK(g_nccl.commInitRank(&comm, nranks, id, rank));
  // every rank's row block (all-gather of (row0, nrows) through the new communicator)
  int* dv = nullptr;
  CK(cudaMalloc(&dv, sizeof(int) * 2 * (nranks + 1)));
  int mine[2] = {row0, nrows};
  CK(cudaMemcpy(dv, mine, sizeof(mine), cudaMemcpyHostToDevice));
  NK(g_nccl.allGather(dv, dv + 2, 2, ncclInt32, comm, 0));
  std::vector<int> all(2 * nranks);
  CK(cudaMemcpy(all.data(), dv + 2, sizeof(int) * 2 * nranks, cudaMemcpyDeviceToHost));
  CK(cudaFree(dv));
  std::vector<int> offs(nranks), rows(nranks);
  int nrmax = 0, covered = 0;
  for (int r = 0; r < nranks; ++r) {
    offs[r] = all[2 * r];
    rows[r] = all[2 * r + 1];
    nrmax = std::max(nrmax, rows[r]);
    if (offs[r] != covered) {
      g_nccl.commDestroy(comm);
      return set_err(PSDPROJ_E_INVALID, "row blocks must be contiguous and ordered by rank");
    }
    covered += rows[r];
  }
  if (covered != n) {
    g_nccl.commDestroy(comm);
    return set_err(PSDPROJ_E_INVALID, "row blocks cover %d of %d rows", covered, n);
  }
  psdproj_ctx_s tmp;
  size_t need = carve(&tmp, n, p, m_max, s_max, NJ, tcols, nullptr, 0, true, nrows, nranks, nrmax);
  if (ws_bytes < need) {
    g_nccl.commDestroy(comm);
    return set_err(PSDPROJ_E_WORKSPACE, "workspace %zu < needed %zu", ws_bytes, need);
  }
  auto* c = new psdproj_ctx_s();
  c->n = n;
  c->ld = rup(nrows, 8);
  c->ldn = rup(n, 8);
  c->prm = p;
  c->m0 = m0; c->q = q; c->m_max = m_max; c->s_max = s_max; c->NJ = NJ; c->tcols = tcols;
  c->sharded = true;
  c->rank = rank; c->nranks = nranks; c->row0 = row0; c->nr = nrows; c->nrmax = nrmax;
  c->comm = comm;
  carve(c, n, p, m_max, s_max, NJ, tcols, (char*)ws, ws_bytes, false, nrows, nranks, nrmax);
  CK(cudaMemcpy(c->d_rows, rows.data(), sizeof(int) * nranks, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_offs, offs.data(), sizeof(int) * nranks, cudaMemcpyHostToDevice));
  c->h_d_len = (size_t)4 * (std::max(s_max, n) + 64);
  c->h_i_len = (size_t)8 * (std::max(s_max, n) + 64);
  if (cudaMallocHost(&c->h_d, c->h_d_len * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&c->h_i, c->h_i_len * sizeof(int)) != cudaSuccess) {
    g_nccl.commDestroy(comm);
    delete c;
    return set_err(PSDPROJ_E_CUDA, "cudaMallocHost failed");
  }
  *out = c;
  return PSDPROJ_OK;
}

extern "C" int psdproj_destroy(psdproj_ctx c) {
  if (!c) return PSDPROJ_OK;
  if (c->comm && g_nccl.ok) g_nccl.commDestroy(c->comm);
  if (c->h_d) cudaFreeHost(c->h_d);
  if (c->h_i) cudaFreeHost(c->h_i);
  for (auto e : c->ev) cudaEventDestroy(e);
  for (auto e : c->pev) cudaEventDestroy(e);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->st3) {
    cudaStreamSynchronize(c->st3);
    cudaStreamDestroy(c->st3);
  }
  if (c->ev3_f) cudaEventDestroy(c->ev3_f);
  if (c->ev3_j) cudaEventDestroy(c->ev3_j);
  for (auto e : c->tev) cudaEventDestroy(e);
  if (c->bst) {
    cudaStreamSynchronize(c->bst);
    cudaStreamDestroy(c->bst);
  }
  if (c->bev_fork) cudaEventDestroy(c->bev_fork);
  if (c->bev_join) cudaEventDestroy(c->bev_join);
  if (c->d_flag) cudaFree(c->d_flag);
  delete c;
  return PSDPROJ_OK;
}

extern "C" int psdproj_reset(psdproj_ctx c) {
  if (!c) return set_err(PSDPROJ_E_INVALID, "ctx NULL");
  c->warm = false;
  c->block_side = 0;
  c->m_warm = 0;
  c->have_counts = false;
  c->th_warm.clear();
  return PSDPROJ_OK;
}

extern "C" const char* psdproj_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ small helpers
namespace {
struct Run {
  psdproj_ctx_s* c;
  cudaStream_t st;
  psdproj_info* info;
  double* part = nullptr;  // split-K partials of this Run's stream (c->part, or c->part2 on the side stream)
  int ihost = 0;  // next free int slot in the pinned buffer (per iteration)
  int rr_npos = 0;  // positive Ritz values among all s of the last Rayleigh-Ritz (expansion test)
  int nev = 0;
  int ntev = 0;  // timed tridiagonalisation launches (profile & 4)
  double anorm = 0.0;
  std::vector<int> marks;  // phase id of each recorded phase event (profile & 2)
  // issued by rr() right before its host sync (the next iteration's rotation and residual norms,
  // speculatively: one sync per LOBPCG iteration instead of two); spec_redo: rr() changed C' or the
  // Ritz values after that point (second Newton-Schulz step / robust path), the speculative work is void
  std::function<int()> spec_fn;
  bool spec_redo = false;

  // phase boundary: the GPU time from this mark to the next is charged to phase ph
  int mark(int ph) {
    if (!(c->prm.profile & 2)) return 0;
    size_t k = marks.size();
    while (c->pev.size() <= k) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->pev.push_back(e);
    }
    CK(cudaEventRecord(c->pev[k], st));
    marks.push_back(ph);
    return 0;
  }

  int upload_idx(const std::vector<int>& v, int* dev) {
    if (v.empty()) return 0;
    if (ihost + (int)v.size() > (int)c->h_i_len - 64) return set_err(PSDPROJ_E_CAPACITY, "pinned index buffer full");
    int* h = c->h_i + ihost;
    std::memcpy(h, v.data(), v.size() * sizeof(int));
    ihost += (int)v.size();
    CK(cudaMemcpyAsync(dev, h, v.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    return 0;
  }
  int sync() {
    if (g_hostprof) {
      const auto t0 = std::chrono::steady_clock::now();
      CK(cudaStreamSynchronize(st));
      g_sync_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      g_nsync++;
      ihost = 0;
      return 0;
    }
    CK(cudaStreamSynchronize(st));
    ihost = 0;
    return 0;
  }
  int gemm(int oa, int ob, int M, int N, int K, double al, const double* A, int lda, const double* B, int ldb,
           double be, double* C, int ldc) {
    if (info) {
      info->flops += 2.0 * M * N * (double)K;
      info->bytes += 8.0 * ((double)M * K + (double)K * N + (double)M * N);
    }
    return dgemm(st, oa, ob, M, N, K, al, A, lda, B, ldb, be, C, ldc, part ? part : c->part, c->part_elems);
  }
  // row-sharded mode: sum over ranks (in place, on the call's stream); no-op otherwise
  int allreduce(double* buf, size_t count) {
    if (!c->sharded || count == 0) return 0;
    NK(g_nccl.allReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, st));
    return 0;
  }
  // Gram C = A^T B (M x N) over the rows of tall-skinny blocks: local rows, then summed over ranks
  int gram(int M, int N, const double* A, int lda, const double* B, int ldb, double* C, int ldc) {
    if (M <= 0 || N <= 0) return 0;
    if (!c->sharded) return gemm(OP_T, OP_N, M, N, c->nr, 1.0, A, lda, B, ldb, 0.0, C, ldc);
    TRY(gemm(OP_T, OP_N, M, N, c->nr, 1.0, A, lda, B, ldb, 0.0, c->gbuf, M));
    TRY(allreduce(c->gbuf, (size_t)M * N));
    CK(cudaMemcpy2DAsync(C, (size_t)ldc * 8, c->gbuf, (size_t)M * 8, (size_t)M * 8, N, cudaMemcpyDeviceToDevice, st));
    return 0;
  }
  // all n rows of a tall-skinny block (k columns) into c->zfull (ld c->ldn): pack, all-gather, unpack
  int gather_full(const double* Zl, int ldz, int k) {
    if (k <= 0) return 0;
    const size_t per = (size_t)c->nrmax * k;
    pack_rows_kernel<<<grid1d(per), 256, 0, st>>>(c->nr, c->nrmax, k, Zl, ldz, c->zsend);
    CKL();
    NK(g_nccl.allGather(c->zsend, c->zpack, per, ncclFloat64, c->comm, st));
    unpack_rows_kernel<<<grid1d(per * c->nranks), 256, 0, st>>>(c->nranks, c->nrmax, k, c->d_rows, c->d_offs, c->zpack,
                                                                 c->zfull, c->ldn);
    CKL();
    return 0;
  }
  // block multiply (a3): Y = sgn * A * Z, the hot kernel; optionally timed with events. Sharded:
  // Y (local rows) = sgn * A_local (nr x n) * Z_full, Z_full all-gathered from the ranks' rows.
  int amul(double sgn, const double* A, int lda, const double* Z, int ldz, int k, double* Y, int ldy) {
    if (k <= 0) return 0;
    int n = c->n, nl = c->nr;
    info->a_passes++;
    info->a_cols += k;
    info->amul_flops += 2.0 * nl * (double)n * k;
    info->amul_bytes += 8.0 * nl * (double)n;
    info->flops += 2.0 * nl * (double)n * k;
    info->bytes += 8.0 * nl * (double)n + 16.0 * n * (double)k;
    if (c->sharded) {
      TRY(gather_full(Z, ldz, k));
      Z = c->zfull;
      ldz = c->ldn;
    }
    bool prof = c->prm.profile & 1;
    if (prof) {
      while ((int)c->ev.size() < 2 * (nev + 1)) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->ev.push_back(e);
      }
      CK(cudaEventRecord(c->ev[2 * nev], st));
    }
    static const int a3_tma = getenv("PSDPROJ_A3_TMA") ? atoi(getenv("PSDPROJ_A3_TMA")) : 1;
    const bool tma_ok = a3_tma && !c->sharded && lda % 2 == 0 && ldz % 2 == 0 && ((uintptr_t)A & 15) == 0 &&
                        ((uintptr_t)Z & 15) == 0;
    if (tma_ok) {
      int rc_ = a3_multiply_tma(st, n, k, sgn, A, lda, Z, ldz, Y, ldy, c->part, c->part_elems);
      if (rc_ < 0) return rc_;
    } else {
      const bool narrow = k <= 96 && (k % 64) != 0 && (k % 64) <= 32;
      int rc_ = narrow ? gemm_kp_launch<OP_N, OP_N, 64, 32, 4, 1>(st, nl, k, n, sgn, A, lda, Z, ldz, 0.0, Y, ldy,
                                                                  c->part, c->part_elems)
                       : gemm_kp_launch<OP_N, OP_N, 64, 64, 4, 1>(st, nl, k, n, sgn, A, lda, Z, ldz, 0.0, Y, ldy,
                                                                  c->part, c->part_elems);
      if (rc_ < 0) return rc_;
    }
    if (prof) {
      CK(cudaEventRecord(c->ev[2 * nev + 1], st));
      nev++;
    }
    return 0;
  }
  // N(0,1) rows [row0, row0 + nr) of the global n x q Philox block (R11)
  int philox(int q, double* dst, int ldd, uint32_t tag) {
    if (q <= 0) return 0;
    if (!c->sharded) {
      philox_gauss_kernel<<<grid1d(((size_t)c->n * q + 1) / 2), 256, 0, st>>>(c->n, q, dst, ldd, c->prm.seed,
                                                                           (uint32_t)c->calls, c->prm.ctx_id, tag);
    } else {
      philox_gauss_rows_kernel<<<grid1d((size_t)c->nr * q), 256, 0, st>>>(c->nr, c->row0, c->n, q, dst, ldd,
                                                                          c->prm.seed, (uint32_t)c->calls,
                                                                          c->prm.ctx_id, tag);
    }
    CKL();
    return 0;
  }
  int gather(int n, int cols, double* dst, int ldd, const double* src, int lds, const std::vector<int>& idx) {
    if (cols <= 0) return 0;
    int* d = c->d_idx;
    // use a fresh region of d_idx per gather within an iteration: offset by ihost
    int off = ihost;
    TRY(upload_idx(idx, d + off));
    gather_cols_kernel<<<grid1d((size_t)n * cols), 256, 0, st>>>(n, cols, dst, ldd, src, lds, d + off);
    CKL();
    return 0;
  }
  // several gathers (idx empty: plain column copy) in one launch, their indices in one upload
  struct GJ {
    double* dst;
    int ldd;
    const double* src;
    int lds;
    int cols;
    const std::vector<int>* idx;
  };
  int gather_multi(int n, std::initializer_list<GJ> jobs) {
    GatherJobs g{};
    std::vector<int> all;
    std::vector<int> offs;
    for (const GJ& j : jobs) {
      if (j.cols <= 0) continue;
      offs.push_back(j.idx ? (int)all.size() : -1);
      if (j.idx) all.insert(all.end(), j.idx->begin(), j.idx->end());
      g.j[g.nj++] = GatherJob{j.dst, j.src, nullptr, j.ldd, j.lds, j.cols};
    }
    if (g.nj == 0) return 0;
    int* d = c->d_idx + ihost;
    TRY(upload_idx(all, d));
    size_t total = 0;
    for (int q = 0; q < g.nj; ++q) {
      if (offs[q] >= 0) g.j[q].idx = d + offs[q];
      total += (size_t)n * g.j[q].cols;
    }
    TRY(launch_pdl(gather_multi_kernel, dim3(grid1d(total)), dim3(256), 0, st, n, g));
    return 0;
  }
  int copy_cols(int n, int cols, double* dst, int ldd, const double* src, int lds) {
    if (cols <= 0) return 0;
    CK(cudaMemcpy2DAsync(dst, (size_t)ldd * 8, src, (size_t)lds * 8, (size_t)n * 8, cols, cudaMemcpyDeviceToDevice,
                         st));
    return 0;
  }
  int normalize(int n, int cols, double* Z, int ldz, double* Z2, int ldz2) {
    if (cols <= 0) return 0;
    if (!c->sharded) {
      TRY(launch_pdl(colnorm_scale_kernel<256>, dim3(cols), dim3(256), 0, st, n, Z, ldz, Z2, ldz2, c->d_norm));
      return 0;
    }
    colnorm_kernel<256><<<cols, 256, 0, st>>>(n, Z, ldz, c->d_norm, c->sharded ? 1 : 0);
    CKL();
    if (c->sharded) {
      TRY(allreduce(c->d_norm, cols));
      sqrt_inplace_kernel<<<cdiv(cols, 256), 256, 0, st>>>(cols, c->d_norm);
      CKL();
    }
    scale_cols_kernel<<<grid1d((size_t)n * cols), 256, 0, st>>>(n, cols, Z, ldz, Z2, ldz2, c->d_norm);
    CKL();
    return 0;
  }
  EighScratch eig_scratch() {
    EighScratch w;
    w.td = c->td; w.te = c->te; w.ttau = c->ttau; w.te2 = c->te2; w.tbounds = c->tbounds; w.tscr = c->tscr;
    w.tG = c->tG; w.ldg = c->s_max; w.Vh = c->Vj; w.ldv = c->s_max;
    // free while the eigensolver runs: G/Hm were consumed by the Cholesky copy and L^-1 H, Gc (L) by trinv
    w.nsM = c->G; w.nsZ = c->Hm; w.nsY = c->Gc;
    w.dev = reinterpret_cast<unsigned long long*>(c->d_scal + 16);
    w.tscr_elems = c->tscr_elems;
    w.mark_obj = this;
    w.mark_fn = [](void* o, int ph) { return static_cast<Run*>(o)->mark(ph); };
    w.tri_fn = [](void* o, int e) { return static_cast<Run*>(o)->tri_mark(e); };
    if (!c->st3) {
      if (cudaStreamCreateWithFlags(&c->st3, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev3_f, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev3_j, cudaEventDisableTiming) != cudaSuccess)
        c->st3 = nullptr;  // eigh_top reports the missing stream
    }
    w.side = c->st3; w.ev_f = c->ev3_f; w.ev_j = c->ev3_j;
    return w;
  }
  // profile bit 2: events around every tridiagonalisation launch (the step's dominant kernel)
  int tri_mark(int e) {
    if (!(c->prm.profile & 4)) return 0;
    const size_t k = 2 * (size_t)ntev + (e ? 1 : 0);
    while (c->tev.size() <= k) {
      cudaEvent_t ev_;
      CK(cudaEventCreate(&ev_));
      c->tev.push_back(ev_);
    }
    CK(cudaEventRecord(c->tev[k], st));
    if (e) ntev++;
    return 0;
  }
  int tri_eig(int s, const double* Hs, int ldh, int m, double* lam, double* Yv, int ldy, int* npos, bool mgs,
              int ns_steps = 2) {
    if (info && (c->prm.profile & 4)) info->tri_flops += 4.0 / 3.0 * s * (double)s * s;  // Householder tridiagonalisation
    return eigh_top(st, s, Hs, ldh, m, lam, Yv, ldy, npos, eig_scratch(), c->part, c->part_elems, mgs, ns_steps);
  }
  // Rayleigh-Ritz on the pencil (H, G) in c->G / c->Hm (s x s, ld s_max):
  // returns 0 (ok), >0 (Cholesky failed at that pivot), <0 error. Outputs Cp (s x mU), theta desc in h_d[0..s).
  // G side of the pencil: known blocks of G, Li = [I 0; 0 0], Cholesky (+ L^-1) of the direction
  // block D (size s - kxG). May run on the side stream (stream_, part_ of a Run bound to it).
  int rr_factor(int s, int kxG, int* started = nullptr, int seq = 0) {
    const int ldm = c->s_max, kx = kxG, t = s - kxG;
    rr_prep_kernel<<<grid1d((size_t)s * s), 256, 0, st>>>(s, kxG, 0, c->G, c->Hm, ldm, nullptr, c->Li, c->Gc,
                                                          c->d_status, 1);
    CKL();
    if (t > 0) {
      TRY(cholesky_run(st, t, c->Gc, ldm, c->d_status, c->tG, (size_t)c->s_max * c->s_max + 16 * (size_t)c->s_max + 2048,
                       c->Li + kx + (size_t)kx * ldm, ldm, started, seq));
      // R44: reject a direction block with max |L^-1|^2 > 1e8 (unit-norm directions: cond(G) >~ 1e8).
      // Cholesky-QR leaves the new block orthonormal only to ~u cond(G), and the pencil takes
      // X^T X = I for granted in the next step; the pivot rule (R20) alone admits cond(G) ~ 1e12
      static double gmax = getenv("PSDPROJ_LINV_MAX") ? atof(getenv("PSDPROJ_LINV_MAX")) : 1e8;
      if (gmax > 0) {
        linv_growth_kernel<<<std::min(296, cdiv(t * t, 256)), 256, 0, st>>>(
            t, c->Li + kx + (size_t)kx * ldm, ldm, gmax, c->d_status);
        CKL();
      }
    }
    return 0;
  }
  // C' = L^-T Y (s x mU) with L^-1 = [I 0; 0 Ld]: rows < kx copied, rows >= kx = Ld^T Y[kx:, :]
  int li_t_apply(int s, int kx, int mU) {
    const int ldm = c->s_max, t = s - kx;
    TRY(dgemm(st, OP_T, OP_N, t, mU, t, 1.0, c->Li + kx + (size_t)kx * ldm, ldm, c->Y + kx, ldm, 0.0, c->Cp + kx, ldm,
              c->part, c->part_elems));
    if (kx > 0) {
      TRY(copy_block_pdl(st, kx, mU, c->Cp, ldm, c->Y, ldm));
    }
    return 0;
  }
  int rr(int s, int kxG, int kxH, const double* d_theta_known, int mU, bool prefactored = false) {
    int ldm = c->s_max;
    info->rr_max = std::max(info->rr_max, s);
    info->flops += 9.0 * s * (double)s * s + s * (double)s * s / 3.0 + 2.0 * s * (double)s * s;
    TRY(mark(3));
    // G = [I 0; 0 D]: factor only the direction block D = L22 L22^T (size t = s - kxG)
    const int kx = kxG;
    if (prefactored) {
      CK(cudaStreamWaitEvent(st, c->ev_join, 0));
    } else {
      TRY(rr_factor(s, kxG));
    }
    TRY(launch_pdl(rr_prep_kernel, dim3(grid1d((size_t)s * s)), dim3(256), 0, st, s, kxG, kxH, c->G, c->Hm, ldm,
                   d_theta_known, c->Li, c->Gc, c->d_status, 2));
    // Hh = L^-1 H L^-T with L^-1 = [I 0; 0 Ld] (Ld = the direction block's inverse factor, t x t):
    // Z = Ld H[kx:, :] (t x s), Hh[kx:, kx:] = Z[:, kx:] Ld^T, the X rows/columns copied
    {
      const int t = s - kx;
      double* Ld = c->Li + kx + (size_t)kx * ldm;
      TRY(dgemm(st, OP_N, OP_N, t, s, t, 1.0, Ld, ldm, c->Hm + kx, ldm, 0.0, c->Y + kx, ldm, c->part, c->part_elems));
      TRY(dgemm(st, OP_N, OP_T, t, t, t, 1.0, c->Y + kx + (size_t)kx * ldm, ldm, Ld, ldm, 0.0,
                c->Hh + kx + (size_t)kx * ldm, ldm, c->part, c->part_elems));
      if (kx > 0) {
        TRY(launch_pdl(rr_assemble_kernel, dim3(grid1d((size_t)s * kx)), dim3(256), 0, st, s, kx, (const double*)c->Hm,
                       (const double*)c->Y, c->Hh, ldm));
      }
    }
    // eigensolver choice by measured crossover: tridiagonal path while the matrix fits in shared memory (s <= 160),
    // cooperative Jacobi above (single-SM tridiagonalisation in global memory is L2-bandwidth bound)
    TRY(mark(4));
    static int rr_mode = -1;  // 0 auto, 1 jacobi, 2 tridiag
    if (rr_mode < 0) {
      const char* e = getenv("PSDPROJ_RR");
      rr_mode = !e ? 0 : (std::string(e) == "jacobi" ? 1 : (std::string(e) == "tridiag" ? 2 : 0));
    }
    bool use_jacobi = rr_mode == 1;
    if (use_jacobi) {
      TRY(jacobi_run(st, s, c->Hh, ldm, c->d_w, c->Vj, ldm, c->jM, c->jM2, c->jQ, c->d_status + 4, c->d_counters,
                     c->d_scal));
      sort_desc_kernel<<<cdiv(s, 256), 256, 0, st>>>(s, c->d_w, c->d_order, c->d_ths);
      CKL();
      count_pos_kernel<<<1, 256, 0, st>>>(s, c->d_w, c->tnpos);
      CKL();
      // C' = L^-T V[:, order[:mU]]
      gather_cols_kernel<<<grid1d((size_t)s * mU), 256, 0, st>>>(s, mU, c->Y, ldm, c->Vj, ldm, c->d_order);
      CKL();
    } else {
      TRY(tri_eig(s, c->Hh, ldm, mU, c->d_ths, c->Y, ldm, c->tnpos, false, 1));
      CK(cudaMemcpyAsync(c->h_d + c->h_d_len - 16, c->d_scal + 16, sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    TRY(li_t_apply(s, kx, mU));
    TRY(mark(7));
    CK(cudaMemcpyAsync(c->h_d, c->d_ths, sizeof(double) * mU, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(c->h_i + c->h_i_len - 16, c->d_status, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(c->h_i + c->h_i_len - 24, c->tnpos, sizeof(int), cudaMemcpyDeviceToHost, st));
    spec_redo = false;
    if (spec_fn) TRY(spec_fn());
    TRY(sync());
    int chol = c->h_i[c->h_i_len - 16];
    int sweeps = c->h_i[c->h_i_len - 16 + 4];
    rr_npos = c->h_i[c->h_i_len - 24];
    if (chol) return chol + kx;
    // one Newton-Schulz step ran (the deviation before it is ~1e-15 for separated Ritz values); a
    // deviation above 1e-4 gets a second step, one still above 1e-4 the robust path
    if (!use_jacobi && !(c->h_d[c->h_d_len - 16] <= 1e-4) && c->h_d[c->h_d_len - 16] < 0.5) {
      TRY(ns_run(st, s, mU, c->Y, ldm, eig_scratch(), c->part, c->part_elems, 1));
      TRY(li_t_apply(s, kx, mU));
      CK(cudaMemcpyAsync(c->h_d + c->h_d_len - 16, c->d_scal + 16, sizeof(double), cudaMemcpyDeviceToHost, st));
      TRY(sync());
      spec_redo = true;
    }
    if (!use_jacobi && !(c->h_d[c->h_d_len - 16] <= 1e-4)) {
      // Newton-Schulz could not restore orthonormality (near-multiple eigenvalues): robust path
      TRY(tri_eig(s, c->Hh, ldm, mU, c->d_ths, c->Y, ldm, c->tnpos, true));
      TRY(li_t_apply(s, kx, mU));
      CK(cudaMemcpyAsync(c->h_d, c->d_ths, sizeof(double) * mU, cudaMemcpyDeviceToHost, st));
      TRY(sync());
      spec_redo = true;
    }
    if (use_jacobi && sweeps < 0) return set_err(PSDPROJ_E_DEGENERATE, "Jacobi did not converge (s=%d)", s);
    return 0;
  }
};
}  // namespace

// ------------------------------------------------------------------ side rule
static int select_mode(psdproj_ctx_s* c) {
  // PAPER.md:505 (< n/3, strict, R17); ties -> smaller count then positive
  int side = c->prm.side;
  if (side != PSDPROJ_SIDE_AUTO) return side;
  if (!c->have_counts) return PSDPROJ_SIDE_POS;
  double third = c->n / 3.0;
  bool pos_ok = c->last_pos < third, neg_ok = c->last_neg < third;
  if (pos_ok && neg_ok) return c->last_pos <= c->last_neg ? PSDPROJ_SIDE_POS : PSDPROJ_SIDE_NEG;
  if (pos_ok) return PSDPROJ_SIDE_POS;
  if (neg_ok) return PSDPROJ_SIDE_NEG;
  return PSDPROJ_SIDE_DIRECT;
}

static int keep_count(const psdproj_ctx_s* c, int p, int m) {
  // R37 (revised, R56): p + max(g, ceil(p/10), 16) columns -- a guard band at least 16 wide, so that a
  // near-zero cluster (C2-cl: 20 eigenvalues within +-5e-3 of 0 next to a gap to -0.1) sits inside the
  // warm block instead of straddling its edge, where the block's convergence rate collapses
  int extra = c->prm.keep_extra >= 0 ? c->prm.keep_extra
                                     : std::max(std::max(c->prm.guard, 16), std::max(1, (int)std::ceil(0.1 * p)));
  return std::min(m, p + extra);
}

// ------------------------------------------------------------------ a10: certification (R16, R36, R53)
// Theorem 3 needs the residual R = B V - V Theta of the RETURNED vectors: one
// explicit block multiply B V at exit (R16; the implicitly rotated B X drifts by ~u ||C'|| per
// iteration), the squared column norms of R, the defect d = ||V^T B V - Theta||_F (hard-locked
// columns are frozen, so V^T B V is only nearly diagonal, R36) and the orthonormality defect
// e = ||V^T V - I||_F (R53). V: nl x p (ld, local rows), d_theta aligned with V's columns, BV: nl x p
// scratch, Hbuf: p x p scratch (ldh). pos_mask: restrict d to the pairs with theta > 0 (DIRECT).
struct Cert {
  std::vector<double> r2;  // squared residual norms, one per column of V
  double defect = 0.0, orth = 0.0;
};
static int certify(Run& run, double sgn, const double* A, int lda, const double* V, int p, const double* d_theta,
                   double* BV, double* Hbuf, int ldh, bool pos_mask, Cert& out) {
  psdproj_ctx_s* c = run.c;
  cudaStream_t st = run.st;
  const int ld = c->ld, nl = c->nr;
  out.r2.assign(p, 0.0);
  out.defect = out.orth = 0.0;
  if (p <= 0) return 0;
  TRY(run.amul(sgn, A, lda, V, ld, p, BV, ld));
  TRY(launch_pdl(resid_norm_kernel<256>, dim3(p), dim3(256), 0, st, nl, V, ld, (const double*)BV, ld, d_theta,
                 (double*)nullptr, 0, c->d_r, 1));
  TRY(run.allreduce(c->d_r, p));  // sums of squares over the ranks' rows (row-sharded mode)
  TRY(run.gram(p, p, V, ld, BV, ld, Hbuf, ldh));
  defect_fro_kernel<1024><<<1, 1024, 0, st>>>(p, Hbuf, ldh, d_theta, 0.0, pos_mask ? d_theta : nullptr,
                                               c->d_scal + 32);
  CKL();
  TRY(run.gram(p, p, V, ld, V, ld, Hbuf, ldh));
  defect_fro_kernel<1024><<<1, 1024, 0, st>>>(p, Hbuf, ldh, nullptr, 1.0, nullptr, c->d_scal + 33);
  CKL();
  CK(cudaMemcpyAsync(c->h_d, c->d_r, sizeof(double) * p, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c->h_d + c->h_d_len - 40, c->d_scal + 32, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
  TRY(run.sync());
  out.r2.assign(c->h_d, c->h_d + p);
  out.defect = c->h_d[c->h_d_len - 40];
  out.orth = c->h_d[c->h_d_len - 39];
  return 0;
}

// eps = (1 + e) sqrt(2 rs + perp^2) + (1 + sqrt 2) d + 7 e theta_max + 4 n u ||A||_F   (R36, R53, R15)
static double theorem3_bound(int n, double rs, double perp, double defect, double orth, double thmax, double anorm) {
  return (1.0 + orth) * std::sqrt(2.0 * rs + perp * perp) + (1.0 + std::sqrt(2.0)) * defect +
         7.0 * orth * std::max(thmax, 0.0) + 4.0 * n * PSD_U * anorm;
}

// ------------------------------------------------------------------ DIRECT path (a13)
static int direct_path(Run& run, const double* A, int lda, double* Pi, int ldpi) {
  psdproj_ctx_s* c = run.c;
  cudaStream_t st = run.st;
  int n = c->n, ld = c->ld;
  run.info->side = PSDPROJ_SIDE_DIRECT;
  run.info->flops += 9.0 * n * (double)n * n;
  // eigendecomposition of A; V into jQ-free region: use T as V (ld x n)
  double* V = c->T;
  static int dmode = -1;  // 1: Jacobi for DIRECT (PSDPROJ_RR=jacobi)
  if (dmode < 0) dmode = (getenv("PSDPROJ_RR") && std::string(getenv("PSDPROJ_RR")) == "jacobi") ? 1 : 0;
  if (dmode == 0 && n <= EIG_MAX) {
    // tridiagonal eigensolver, all n pairs, descending; order = identity
    TRY(run.tri_eig(n, A, lda, n, c->d_ths, V, ld, c->tnpos, false));
    CK(cudaMemcpyAsync(c->h_d + c->h_d_len - 16, c->d_scal + 16, sizeof(double), cudaMemcpyDeviceToHost, st));
    TRY(run.sync());
    if (!(c->h_d[c->h_d_len - 16] <= 1e-7)) TRY(run.tri_eig(n, A, lda, n, c->d_ths, V, ld, c->tnpos, true));
    CK(cudaMemcpyAsync(c->h_d, c->d_ths, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    TRY(run.sync());
    for (int i = 0; i < n; ++i) c->h_i[i] = i;
  } else {
    TRY(jacobi_run(st, n, A, lda, c->d_w, V, ld, c->jM, c->jM2, c->jQ, c->d_status + 4, c->d_counters, c->d_scal));
    sort_desc_kernel<<<cdiv(n, 256), 256, 0, st>>>(n, c->d_w, c->d_order, c->d_ths);
    CKL();
    CK(cudaMemcpyAsync(c->h_d, c->d_ths, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(c->h_i + c->h_i_len - 16, c->d_status, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(c->h_i, c->d_order, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    TRY(run.sync());
    if (c->h_i[c->h_i_len - 16 + 4] < 0) return set_err(PSDPROJ_E_DEGENERATE, "Jacobi (DIRECT) did not converge");
  }
  std::vector<double> w(c->h_d, c->h_d + n);
  std::vector<int> order(c->h_i, c->h_i + n);
  int p = 0;
  while (p < n && w[p] > 0.0) ++p;
  {
    double f2 = 0.0;
    for (int i = 0; i < p; ++i) f2 += w[i] * w[i];
    run.info->pi_fro = std::sqrt(f2);  // ||Pi(A)||_F of the returned projection's eigenvalues
  }
  // a10 for DIRECT (R53), before the assembly (Pi may alias A): Theorem 3 with V~ = the computed positive eigenvectors; its perp term is
  // bounded by the residual of the others: ||Pi(V-^T A V-)||_F = dist(V-^T A V-, NSD) <=
  // ||V-^T A V- - Theta-||_F <= ||V-|| ||A V- - V- Theta-||_F (Theta- <= 0 is in the NSD cone)
  {
    const bool tri = (dmode == 0 && n <= EIG_MAX);
    const double* thcol = tri ? c->d_ths : c->d_w;  // eigenvalues aligned with V's columns
    std::vector<double> wcol(n);
    for (int i = 0; i < n; ++i) wcol[order[i]] = w[i];
    Cert ct;
    TRY(certify(run, 1.0, A, lda, V, n, thcol, c->T2, c->jM, c->NJ, true, ct));
    double rsp = 0.0, rsn = 0.0, thmax = 0.0;
    for (int j = 0; j < n; ++j) {
      if (wcol[j] > 0.0) {
        rsp += ct.r2[j];
        thmax = std::max(thmax, wcol[j]);
      } else {
        rsn += ct.r2[j];
      }
    }
    const double perp = (1.0 + ct.orth) * std::sqrt(rsn);
    run.info->resid_fro = std::sqrt(rsp);
    run.info->lock_defect = ct.defect;
    run.info->orth_defect = ct.orth;
    run.info->perp_est = perp;
    run.info->err_bound = theorem3_bound(n, rsp, perp, ct.defect, ct.orth, thmax, run.anorm);
  }
  // Pi = V+ diag(w+) V+^T
  std::vector<int> pidx(order.begin(), order.begin() + p);
  TRY(run.gather(n, p, c->T2, ld, V, ld, pidx));
  if (p > 0) {
    CK(cudaMemcpyAsync(c->d_w, c->d_ths, sizeof(double) * p, cudaMemcpyDeviceToDevice, st));
    scale_copy_cols_kernel<<<grid1d((size_t)n * p), 256, 0, st>>>(n, p, c->E, ld, c->T2, ld, c->d_w);
    CKL();
    TRY(run.gemm(OP_N, OP_T, n, n, p, 1.0, c->E, ld, c->T2, ld, 0.0, Pi, ldpi));
    symmetrize_kernel<<<grid1d((size_t)n * n), 256, 0, st>>>(n, Pi, ldpi);
    CKL();
  } else {
    CK(cudaMemset2DAsync(Pi, (size_t)ldpi * 8, 0, (size_t)n * 8, n, st));
  }
  run.info->bytes += 16.0 * n * (double)n;
  double z = 1e-9 * (1.0 + run.anorm);
  int np = 0, nn = 0;
  for (double x : w) {
    np += x > z;
    nn += x < -z;
  }
  c->last_pos = np;
  c->last_neg = nn;
  c->have_counts = true;
  run.info->npos = p;
  run.info->m = n;
  // seed the warm block for the side the next call will use
  int nxt = select_mode(c);
  if (nxt == PSDPROJ_SIDE_POS || nxt == PSDPROJ_SIDE_NEG) {
    std::vector<int> idx;
    std::vector<double> th;
    if (nxt == PSDPROJ_SIDE_POS) {
      int keep = keep_count(c, p, std::min(n, c->m_max));
      for (int i = 0; i < keep; ++i) { idx.push_back(order[i]); th.push_back(w[i]); }
    } else {
      int pn = 0;
      while (pn < n && w[n - 1 - pn] < 0.0) ++pn;
      int keep = keep_count(c, pn, std::min(n, c->m_max));
      for (int i = 0; i < keep; ++i) { idx.push_back(order[n - 1 - i]); th.push_back(-w[n - 1 - i]); }
    }
    TRY(run.gather(n, (int)idx.size(), c->Xw, ld, V, ld, idx));
    c->m_warm = (int)idx.size();
    c->th_warm = th;
    c->block_side = nxt;
    c->warm = true;
  } else {
    c->warm = false;
    c->block_side = 0;
  }
  return PSDPROJ_OK;
}

// ------------------------------------------------------------------ f2: perp term (R48)
// Upper bound on the perp term of Theorem 3, ||Pi(V~perp^T B V~perp)||_F <= sqrt(n - p) max(lambda_max(D), 0)
// with D = B restricted to span(V)^perp (the "projected Lanczos" of PAPER.md:508).
// k Lanczos steps on D = (I - V V^T) B (I - V V^T) (V: n x p, orthonormal) from a Philox start (tag
// 0xC0000000, uniform on the sphere of span(V)^perp after deflation), full reorthogonalisation (two CGS
// passes against V and the Lanczos basis, held in c->E); mu = the largest eigenvalue of the Lanczos
// matrix T_k (the path's tridiagonal eigensolver). Kuczynski & Wozniakowski (1992): for a PSD matrix M
// of order N, P{xi_k < (1 - eps) lambda_1(M)} <= 1.648 sqrt(N) exp(-sqrt(eps) (2k - 1)). Applied to
// M = D - c I with c = -||A||_F <= lambda_min(D) (certified), with probability >= 1 - delta:
//   lambda_max(D) <= c + (mu - c) / (1 - eps),  sqrt(eps) = ln(1.648 sqrt(N) / delta) / (2k - 1)
// (vacuous when eps >= 1: then lambda_max(D) <= ||A||_F is used). A Lanczos breakdown (invariant
// Krylov space) or k = N gives mu = lambda_max(D) itself (a random start has a component along every
// eigenspace with probability 1). Reading R48 (revised in round 2).
static int perp_estimate(Run& run, double sgn, const double* A, int lda, const double* V, int p, int steps,
                         double* perp) {
  psdproj_ctx_s* c = run.c;
  const int n = c->n, ld = c->ld, ldm = c->s_max, nl = c->nr;
  const int neff = n - p;
  const int k = std::min(std::min(steps, c->s_max), std::min(neff, c->tcols - 1));
  *perp = 0.0;
  if (neff <= 0 || k <= 0) return 0;
  double* Q = c->E;   // n x (k + 1): the expansion buffer (ld x max(s_max, n)) is free at exit
  double* w = c->T2;  // n x 1 (free after the certification)
  auto deflate = [&](double* z, int nq) -> int {
    for (int pass = 0; pass < 2; ++pass) {
      if (p > 0) {
        TRY(run.gram(p, 1, V, ld, z, ld, c->Y, ldm));
        TRY(run.gemm(OP_N, OP_N, nl, 1, p, -1.0, V, ld, c->Y, ldm, 1.0, z, ld));
      }
      if (nq > 0) {
        TRY(run.gram(nq, 1, Q, ld, z, ld, c->Y, ldm));
        TRY(run.gemm(OP_N, OP_N, nl, 1, nq, -1.0, Q, ld, c->Y, ldm, 1.0, z, ld));
      }
    }
    return 0;
  };
  TRY(run.philox(1, Q, ld, 0xC0000000u));
  TRY(deflate(Q, 0));
  TRY(run.normalize(nl, 1, Q, ld, nullptr, 0));
  std::vector<double> alpha, beta;
  const double anorm = std::max(run.anorm, 1e-300);
  const double tiny = 1e-14 * anorm;
  bool breakdown = false;
  for (int j = 0; j < k; ++j) {
    double* qj = Q + (size_t)j * ld;
    TRY(run.amul(sgn, A, lda, qj, ld, 1, w, ld));
    if (p > 0) {
      TRY(run.gram(p, 1, V, ld, w, ld, c->Y, ldm));
      TRY(run.gemm(OP_N, OP_N, nl, 1, p, -1.0, V, ld, c->Y, ldm, 1.0, w, ld));
    }
    TRY(run.gram(1, 1, qj, ld, w, ld, c->Y, ldm));  // alpha_j = q_j^T D q_j
    CK(cudaMemcpyAsync(c->h_d, c->Y, sizeof(double), cudaMemcpyDeviceToHost, run.st));
    TRY(deflate(w, j + 1));
    TRY(run.normalize(nl, 1, w, ld, nullptr, 0));
    CK(cudaMemcpyAsync(c->h_d + 1, c->d_norm, sizeof(double), cudaMemcpyDeviceToHost, run.st));
    TRY(run.sync());
    alpha.push_back(c->h_d[0]);
    beta.push_back(c->h_d[1]);
    if (c->h_d[1] <= tiny) {
      breakdown = true;
      break;
    }
    if (j == k - 1) break;
    CK(cudaMemcpy2DAsync(Q + (size_t)(j + 1) * ld, (size_t)ld * 8, w, (size_t)ld * 8, (size_t)nl * 8, 1,
                         cudaMemcpyDeviceToDevice, run.st));
  }
  // mu = lambda_max(T_k) on the device (T_k from the host-read alpha, beta: marshalling only)
  const int kk = (int)alpha.size();
  for (int i = 0; i < kk; ++i) {
    c->h_d[i] = alpha[i];
    c->h_d[kk + i] = beta[i];
  }
  CK(cudaMemcpyAsync(c->d_r, c->h_d, sizeof(double) * kk, cudaMemcpyHostToDevice, run.st));
  CK(cudaMemcpyAsync(c->d_thU, c->h_d + kk, sizeof(double) * kk, cudaMemcpyHostToDevice, run.st));
  tridiag_dense_kernel<<<grid1d((size_t)kk * kk), 256, 0, run.st>>>(kk, c->d_r, c->d_thU, c->Hh, ldm);
  CKL();
  TRY(run.tri_eig(kk, c->Hh, ldm, 1, c->d_ths, c->Y, ldm, c->tnpos, false, 1));
  CK(cudaMemcpyAsync(c->h_d, c->d_ths, sizeof(double), cudaMemcpyDeviceToHost, run.st));
  TRY(run.sync());
  const double mu = c->h_d[0];
  const double delta = c->prm.perp_delta > 0.0 ? c->prm.perp_delta : 1e-6;
  double ub;
  if (breakdown || kk >= neff) {
    ub = mu + 4.0 * kk * PSD_U * anorm;
  } else {
    const double se = std::log(1.648 * std::sqrt((double)neff) / delta) / (2.0 * kk - 1.0);
    const double eps = se * se;
    const double c0 = -anorm;
    ub = eps >= 1.0 ? anorm : std::min(anorm, c0 + (mu - c0) / (1.0 - eps));
  }
  run.info->perp_mu = mu;
  *perp = std::sqrt((double)neff) * std::max(ub, 0.0);
  return 0;
}

// ------------------------------------------------------------------ LOBPCG path
static int lobpcg_path(Run& run, int side, const double* A, int lda, double* Pi, int ldpi, double tol,
                       bool& abort_direct) {
  psdproj_ctx_s* c = run.c;
  psdproj_info* info = run.info;
  cudaStream_t st = run.st;
  const int n = c->n, ld = c->ld, ldm = c->s_max;
  const int nl = c->nr;  // rows of the tall-skinny blocks held here (n unless row-sharded)
  const double sgn = side == PSDPROJ_SIDE_POS ? 1.0 : -1.0;
  const bool hard = c->prm.locking == PSDPROJ_LOCK_HARD;
  const int g = c->prm.guard;
  info->side = side;
  abort_direct = false;

  bool cold = !(c->warm && c->block_side == side);
  info->cold = cold;
  int m = cold ? c->m0 : c->m_warm;
  if (m > c->m_max) return set_err(PSDPROJ_E_CAPACITY, "block %d > m_max %d", m, c->m_max);
  // ---- start block X0 in S[:, :m] and B X0 in BS
  if (cold) {
    TRY(run.philox(m, c->S, ld, 0u));
  } else {
    TRY(run.copy_cols(nl, m, c->S, ld, c->Xw, ld));
  }
  TRY(run.amul(sgn, A, lda, c->S, ld, m, c->BS, ld));
  // ---- Alg. 3 line 2: Rayleigh-Ritz on span(X0): G = X0^T X0, H = X0^T B X0 (G is formed for a warm
  // block too: it is the previous call's block, orthonormal only up to that call's drift)
  TRY(run.gram(m, m, c->S, ld, c->S, ld, c->G, ldm));
  TRY(run.gram(m, m, c->S, ld, c->BS, ld, c->Hm, ldm));
  int rc = run.rr(m, 0, 0, c->d_thU, m);
  if (rc > 0 && !cold) {
    // the warm block lost rank (e.g. the previous input was 0): cold start (R28)
    cold = true;
    info->cold = 1;
    m = c->m0;
    TRY(run.philox(m, c->S, ld, 0u));
    TRY(run.amul(sgn, A, lda, c->S, ld, m, c->BS, ld));
    TRY(run.gram(m, m, c->S, ld, c->S, ld, c->G, ldm));
    TRY(run.gram(m, m, c->S, ld, c->BS, ld, c->Hm, ldm));
    rc = run.rr(m, 0, 0, c->d_thU, m);
  }
  if (rc > 0) return set_err(PSDPROJ_E_DEGENERATE, "start block rank deficient");
  TRY(rc);
  std::vector<double> thU(c->h_d, c->h_d + m);  // all m values (the initial RR keeps m of m)
  TRY(run.gemm(OP_N, OP_N, nl, m, m, 1.0, c->S, ld, c->Cp, ldm, 0.0, c->S2, ld));
  TRY(run.gemm(OP_N, OP_N, nl, m, m, 1.0, c->BS, ld, c->Cp, ldm, 0.0, c->BS2, ld));
  std::swap(c->S, c->S2);
  std::swap(c->BS, c->BS2);
  CK(cudaMemcpyAsync(c->d_thU, c->d_ths, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));

  int mU = m, nL = 0, qe = 0;
  // the hard-locked block X_L / B X_L: right-aligned in the prefix of the current S / BS (mirrored in
  // front of S2 / BS2), so that [X_L | X_U] is contiguous
  auto XLp = [&]() { return c->S - (size_t)nL * ld; };
  auto BXLp = [&]() { return c->BS - (size_t)nL * ld; };
  std::vector<double> rU(m, INFINITY), thL, rL;
  std::vector<char> hasP(m, 0);
  int status = PSDPROJ_NOT_CONVERGED;
  int k = 0;
  static int restart = getenv("PSDPROJ_RESTART") ? atoi(getenv("PSDPROJ_RESTART")) : 100;
  // R61: a restart also when the largest residual of the positive Ritz pairs has not improved for
  // `stall` iterations (>= 2 stall since the last restart): the rotated B X carries rounding that
  // leaves a residual floor near tol; the restart recomputes B X explicitly (PSDPROJ_STALL, 0 = off)
  static int stall = getenv("PSDPROJ_STALL") ? atoi(getenv("PSDPROJ_STALL")) : 0;
  // R61 (default): a restart when every unconverged positive pair has r < near_c * tol and the largest
  // of them has not improved by 5% for near_win iterations (at most once per 2 near_win iterations):
  // the warm calls otherwise sit just above tol until the next periodic restart (DESIGN R61)
  static double near_c = getenv("PSDPROJ_NEAR_RESTART") ? atof(getenv("PSDPROJ_NEAR_RESTART")) : 3.0;
  static int near_win = getenv("PSDPROJ_NEAR_WIN") ? atoi(getenv("PSDPROJ_NEAR_WIN")) : 5;
  bool force_restart = false;
  // residual norms of the current block already on the host (issued speculatively before the last
  // Rayleigh-Ritz sync, Run::spec_fn), in the pinned slot h_d + h_d_len / 2
  bool spec_ready = false;
  static const int spec_env = getenv("PSDPROJ_SPEC") ? atoi(getenv("PSDPROJ_SPEC")) : 1;
  const size_t rslot = c->h_d_len / 2;
  int k_restart = 0, k_best = 0;
  double best_rpos = INFINITY;
  for (;;) {
    // R47: restart every `restart` iterations -- X_U re-orthonormalised (against X_L, then by the
    // Cholesky-QR of the start-block RR), B X_U recomputed, Rayleigh-Ritz on span(X_U), P dropped.
    // The pencil takes X_U^T X_U = I and B X_U from the rotation; both drift (by ~u cond(G) and
    // ~u ||C'|| per step) on long runs that never meet the stopping rule.
    if (((restart > 0 && k > 0 && k % restart == 0) || force_restart) && mU > 0) {
      force_restart = false;
      spec_ready = false;
      k_restart = k;
      best_rpos = INFINITY;
      k_best = k;
      TRY(run.mark(0));
      if (hard && nL > 0) {
        TRY(run.gram(nL, mU, XLp(), ld, c->S, ld, c->Y, ldm));
        TRY(run.gemm(OP_N, OP_N, nl, mU, nL, -1.0, XLp(), ld, c->Y, ldm, 1.0, c->S, ld));
      }
      TRY(run.amul(sgn, A, lda, c->S, ld, mU, c->BS, ld));
      int rr0;
      for (;;) {
        TRY(run.gram(mU, mU, c->S, ld, c->S, ld, c->G, ldm));
        TRY(run.gram(mU, mU, c->S, ld, c->BS, ld, c->Hm, ldm));
        rr0 = run.rr(mU, 0, 0, c->d_thU, mU);
        if (rr0 <= 0 || mU <= 1) break;
        // a column that became dependent on the others (duplicated direction): drop it (R41)
        const int col = rr0 - 1, last = mU - 1;
        if (col != last) {
          swap_cols_kernel<<<grid1d((size_t)nl), 256, 0, st>>>(nl, c->S, ld, col, last);
          CKL();
          swap_cols_kernel<<<grid1d((size_t)nl), 256, 0, st>>>(nl, c->BS, ld, col, last);
          CKL();
        }
        --mU;
        info->dropped++;
      }
      if (rr0 > 0) return set_err(PSDPROJ_E_DEGENERATE, "restart block rank deficient");
      TRY(rr0);
      thU.assign(c->h_d, c->h_d + mU);
      TRY(run.gemm(OP_N, OP_N, nl, mU, mU, 1.0, c->S, ld, c->Cp, ldm, 0.0, c->S2, ld));
      TRY(run.gemm(OP_N, OP_N, nl, mU, mU, 1.0, c->BS, ld, c->Cp, ldm, 0.0, c->BS2, ld));
      std::swap(c->S, c->S2);
      std::swap(c->BS, c->BS2);
      CK(cudaMemcpyAsync(c->d_thU, c->d_ths, sizeof(double) * mU, cudaMemcpyDeviceToDevice, st));
      static const int soft_restart = getenv("PSDPROJ_SOFT_RESTART") ? atoi(getenv("PSDPROJ_SOFT_RESTART")) : 0;
      // soft: P (re-projected against X every iteration) is kept unless a column was dropped
      if (!soft_restart || (int)hasP.size() != mU) hasP.assign(mU, 0);
    }
    // ---- line 5: R = B X - X Theta, r_i = ||R_i|| (unlocked columns)
    TRY(run.mark(6));
    if (spec_ready) {
      rU.assign(c->h_d + rslot, c->h_d + rslot + mU);
      spec_ready = false;
    } else {
      TRY(launch_pdl(resid_norm_kernel<256>, dim3(mU), dim3(256), 0, st, nl, (const double*)c->S, ld,
                     (const double*)c->BS, ld, (const double*)c->d_thU, c->R, ld, c->d_r, c->sharded ? 1 : 0));
      if (c->sharded) {  // column sums of squares over the ranks' rows
        TRY(run.allreduce(c->d_r, mU));
        sqrt_inplace_kernel<<<cdiv(mU, 256), 256, 0, st>>>(mU, c->d_r);
        CKL();
      }
      CK(cudaMemcpyAsync(c->h_d, c->d_r, sizeof(double) * mU, cudaMemcpyDeviceToHost, st));
      TRY(run.sync());
      rU.assign(c->h_d, c->h_d + mU);
    }
    const int trace = getenv("PSDPROJ_TRACE") ? 1 : 0;  // debugging: per-iteration state on stderr
    if (trace) {
      double tmx = -INFINITY, tmn = INFINITY, rmx = 0, rpos = 0;
      int nun = 0;
      for (int j = 0; j < mU; ++j) {
        tmx = std::max(tmx, thU[j]);
        tmn = std::min(tmn, thU[j]);
        rmx = std::max(rmx, rU[j]);
        if (thU[j] > 0) {
          rpos = std::max(rpos, rU[j]);
          nun += rU[j] > tol;
        }
      }
      fprintf(stderr, "trace k=%d mU=%d nL=%d qe=%d theta[%g, %g] rmax %g rpos %g unconv+ %d tol %g dropped %d\n", k, mU, nL,
              qe, tmn, tmx, rmx, rpos, nun, tol, info->dropped);
    }
    if ((stall > 0 || near_c > 0.0) && mU > 0) {
      double rpos = 0.0;
      for (int j = 0; j < mU; ++j)
        if (thU[j] > 0 && rU[j] > tol) rpos = std::max(rpos, rU[j]);
      if (rpos > 0.0) {
        const int win = stall > 0 ? stall : near_win;
        if (rpos < 0.95 * best_rpos) {
          best_rpos = rpos;
          k_best = k;
        } else if (k - k_best >= win && k - k_restart >= 2 * win && (near_c <= 0.0 || rpos < near_c * tol)) {
          force_restart = true;
        }
      }
    }
    // ---- stopping rule (R12)
    int npos = nL;
    bool conv_pos = true;
    double g_th = -INFINITY, g_r = 0.0;
    bool has_guard = false;
    for (int j = 0; j < mU; ++j) {
      if (thU[j] > 0) {
        npos++;
        if (!(rU[j] <= tol)) conv_pos = false;
      } else if (!has_guard || thU[j] > g_th) {
        has_guard = true;
        g_th = thU[j];
        g_r = rU[j];
      }
    }
    int mtot = nL + mU;
    // guard certification theta_g + r_g <= tol (R52: its inclusion interval lies below tol) and
    // r_g <= max(tol, |theta_g| / 2) (R60): a guard whose residual exceeds both the tolerance and half
    // its distance to zero is too far from convergence to vouch for the block (a cold 2-column block
    // passed R52 at k = 1 with theta_g = -0.86, r_g = 0.83 and missed the only positive eigenvalue);
    // with the paper's loose schedule (10/k^1.01) both reduce to r_g <= tol-ish
    bool guard_ok = (mtot >= n) ? true
                                : (has_guard && g_th + g_r <= tol && g_r <= std::max(tol, 0.5 * std::fabs(g_th)));
    bool converged = conv_pos && guard_ok && qe == 0 && !(cold && k == 0);
    if (converged) {
      status = PSDPROJ_OK;
      break;
    }
    if (k >= c->prm.max_iter) break;
    // ---- hard locking (R35) at lock_tol = lock_factor * tol (R55: a locked vector is frozen with its
    // error ~ r / gap, which bounds the residual the columns kept orthogonal to it can reach)
    TRY(run.mark(7));
    const double lock_tol = (c->prm.lock_factor > 0.0 ? c->prm.lock_factor : 1.0) * tol;
    std::vector<int> keep, lock;
    for (int j = 0; j < mU; ++j) {
      if (hard && thU[j] > 0 && rU[j] <= lock_tol)
        lock.push_back(j);
      else
        keep.push_back(j);
    }
    if (!lock.empty()) {
      // the newly locked columns join X_L at its front (in both S prefixes and both BS prefixes)
      const size_t nw = (size_t)(nL + lock.size()) * ld;
      TRY(run.gather(nl, (int)lock.size(), c->S - nw, ld, c->S, ld, lock));
      TRY(run.gather(nl, (int)lock.size(), c->S2 - nw, ld, c->S, ld, lock));
      TRY(run.gather(nl, (int)lock.size(), c->BS - nw, ld, c->BS, ld, lock));
      TRY(run.gather(nl, (int)lock.size(), c->BS2 - nw, ld, c->BS, ld, lock));
      {
        std::vector<double> th0, r0;
        for (int j : lock) {
          th0.push_back(thU[j]);
          r0.push_back(rU[j]);
        }
        thL.insert(thL.begin(), th0.begin(), th0.end());
        rL.insert(rL.begin(), r0.begin(), r0.end());
      }
      nL += (int)lock.size();
      // compact U (X, BX, P, BP, theta)
      int nk = (int)keep.size();
      TRY(run.gather(nl, nk, c->T, ld, c->S, ld, keep));
      TRY(run.copy_cols(nl, nk, c->S, ld, c->T, ld));
      TRY(run.gather(nl, nk, c->T, ld, c->BS, ld, keep));
      TRY(run.copy_cols(nl, nk, c->BS, ld, c->T, ld));
      TRY(run.gather(nl, nk, c->T, ld, c->Pb, ld, keep));
      TRY(run.copy_cols(nl, nk, c->Pb, ld, c->T, ld));
      TRY(run.gather(nl, nk, c->T, ld, c->BPb, ld, keep));
      TRY(run.copy_cols(nl, nk, c->BPb, ld, c->T, ld));
      std::vector<double> th2, r2;
      std::vector<char> hp2;
      for (int j : keep) {
        th2.push_back(thU[j]);
        r2.push_back(rU[j]);
        hp2.push_back(hasP[j]);
      }
      thU = th2;
      rU = r2;
      hasP = hp2;
      mU = nk;
      for (int j = 0; j < mU; ++j) c->h_d[j] = thU[j];
      CK(cudaMemcpyAsync(c->d_thU, c->h_d, sizeof(double) * mU, cudaMemcpyHostToDevice, st));
      TRY(run.sync());
    }
    // ---- active set J (BLOPEX active mask): unlocked columns with r > tol
    std::vector<int> Jorig, Jnew, PJ;
    // R62: on warm calls only the top guard_active non-positive columns keep their W / P directions
    // (the guard test of R12 looks at the top guard only; measured on C3-R: +13% iterations at -20%
    // time per iteration); cold calls keep every unconverged column (Alg. 3's mask)
    static const char* ga_env = getenv("PSDPROJ_GUARD_ACTIVE");  // experiments: overrides the parameter
    const int ga_prm = ga_env ? atoi(ga_env) : c->prm.guard_active;
    const int guard_active = cold ? -1 : (ga_prm == 0 ? 2 : ga_prm);
    int nonpos_seen = 0;
    for (int jj = 0; jj < mU; ++jj) {
      int j0 = keep[jj];
      const bool guard_col = !(thU[jj] > 0);
      if (guard_col) ++nonpos_seen;
      if (guard_active >= 0 && guard_col && nonpos_seen > guard_active) continue;
      if (rU[jj] > tol) {
        Jorig.push_back(j0);
        Jnew.push_back(jj);
        if (hasP[jj]) PJ.push_back(jj);
      }
    }
    // experiment (PSDPROJ_S_CAP = +-cap, default off): on warm calls keep the basis within the
    // register tridiagonalisation's range (s <= cap) by giving directions only to the (cap - mU) / 2
    // active columns with the smallest (cap > 0) or largest (cap < 0) residuals
    static const int s_cap = getenv("PSDPROJ_S_CAP") ? atoi(getenv("PSDPROJ_S_CAP")) : 0;
    if (s_cap != 0 && !cold && mU + 2 * (int)Jorig.size() > std::abs(s_cap)) {
      const int keep_a = std::max(16, (std::abs(s_cap) - mU) / 2);
      if ((int)Jnew.size() > keep_a) {
        std::vector<int> ord(Jnew.size());
        for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
        std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
          return s_cap > 0 ? rU[Jnew[x]] < rU[Jnew[y]] : rU[Jnew[x]] > rU[Jnew[y]];
        });
        std::vector<char> sel(Jnew.size(), 0);
        for (int i = 0; i < keep_a; ++i) sel[ord[i]] = 1;
        std::vector<int> Jo2, Jn2, PJ2;
        for (size_t i = 0; i < Jnew.size(); ++i)
          if (sel[i]) {
            Jo2.push_back(Jorig[i]);
            Jn2.push_back(Jnew[i]);
            if (hasP[Jnew[i]]) PJ2.push_back(Jnew[i]);
          }
        Jorig.swap(Jo2);
        Jnew.swap(Jn2);
        PJ.swap(PJ2);
      }
    }
    int a = (int)Jorig.size();
    // experiment (PSDPROJ_WIDE_NO_P = a0, default off): iterations whose active set is wider than a0
    // leave dX out of the trial space (s = mU + a instead of mU + 2a; the Rayleigh-Ritz cost of the
    // few wide iterations at the start of a warm call is several times that of a late one)
    static const int wide_no_p = getenv("PSDPROJ_WIDE_NO_P") ? atoi(getenv("PSDPROJ_WIDE_NO_P")) : 0;
    if (wide_no_p > 0 && !cold && a > wide_no_p) PJ.clear();
    int ap = (int)PJ.size();
    if (mU + a + qe + ap == 0) {
      // every column is locked and no direction is left, but the guard test (R12) is not met: the
      // block has no non-positive column -- draw the expansion block now (Alg. 3 line 8, R8)
      const int mt = nL;
      if (mt >= n) {
        status = PSDPROJ_OK;
        break;
      }
      const int qq = std::min(c->q, n - mt);
      if (mt + qq > c->m_max) {
        if (c->sharded) return set_err(PSDPROJ_E_CAPACITY, "block %d exceeds m_max %d", mt + qq, c->m_max);
        abort_direct = true;
        return PSDPROJ_OK;
      }
      TRY(run.philox(qq, c->E, ld, (uint32_t)(k + 1) | 0x80000000u));
      for (int pass = 0; pass < 2 && nL > 0; ++pass) {
        TRY(run.gram(nL, qq, XLp(), ld, c->E, ld, c->Y, ldm));
        TRY(run.gemm(OP_N, OP_N, nl, qq, nL, -1.0, XLp(), ld, c->Y, ldm, 1.0, c->E, ld));
      }
      qe = qq;
      info->expansions++;
    }
    int offW = mU, offE = mU + a, offP = mU + a + qe;
    // R57 (krylov_depth d > 1): d - 1 block-Krylov directions B^k R_J follow P in the basis
    // R63: only while the active set is at most krylov_max_active columns wide (0: always)
    static const char* kma_env = getenv("PSDPROJ_KRYLOV_MAX_ACTIVE");  // experiments: overrides the parameter
    const int kma = kma_env ? atoi(kma_env) : c->prm.krylov_max_active;
    const int depth = (kma > 0 && a > kma) ? 1 : std::max(1, c->prm.krylov_depth);
    const int aK = depth > 1 ? a : 0;
    int s = offP + ap + (depth - 1) * aK;
    if (getenv("PSDPROJ_TRACE")) fprintf(stderr, "basis k=%d s=%d mU=%d a=%d ap=%d qe=%d nL=%d\n", k, s, mU, a, ap, qe, nL);
    if (s > c->s_max) return set_err(PSDPROJ_E_CAPACITY, "RR basis %d > s_max %d", s, c->s_max);
    // W = R_J (+ pending expansion E) and P_J sit contiguously in S: [W E P] at offW; both are
    // projected against the locked block and X_U in one pass (one Gram + one update GEMM each)
    TRY(run.mark(1));
    int aw = a + qe;
    double* W = c->S + (size_t)offW * ld;
    double* P = c->S + (size_t)offP * ld;
    double* BP = c->BS + (size_t)offP * ld;
    TRY(run.gather_multi(nl, {{W, ld, c->R, ld, a, &Jorig},
                              {c->S + (size_t)offE * ld, ld, c->E, ld, qe, nullptr},
                              {P, ld, c->Pb, ld, ap, &PJ},
                              {BP, ld, c->BPb, ld, ap, &PJ}}));
    const int wp = aw + ap;
    static int lock_reproj = getenv("PSDPROJ_LOCK_REPROJ") ? atoi(getenv("PSDPROJ_LOCK_REPROJ")) : 0;
    const int xr = (lock_reproj && hard && nL > 0) ? mU : 0;  // X_U columns included (R46)
    if (xr > 0) {
      // R46 (off by default): X_U (and B X_U) re-projected against X_L
      TRY(run.gram(nL, xr, XLp(), ld, c->S, ld, c->Y, ldm));
      TRY(run.gemm(OP_N, OP_N, nl, xr, nL, -1.0, XLp(), ld, c->Y, ldm, 1.0, c->S, ld));
      TRY(run.gemm(OP_N, OP_N, nl, xr, nL, -1.0, BXLp(), ld, c->Y, ldm, 1.0, c->BS, ld));
    }
    if (wp > 0) {
      // [W P] <- [W P] - [X_L X_U] ([X_L X_U]^T [W P]) in one pass over the contiguous block (B P
      // likewise with [B X_L, B X_U]): the pencil's X-block of G becomes [I 0]
      const int nX = (hard ? nL : 0) + mU;
      double* Xall = hard ? XLp() : c->S;
      double* BXall = hard ? BXLp() : c->BS;
      TRY(run.gram(nX, wp, Xall, ld, W, ld, c->Y, ldm));
      TRY(run.gemm(OP_N, OP_N, nl, wp, nX, -1.0, Xall, ld, c->Y, ldm, 1.0, W, ld));
      if (ap > 0) TRY(run.gemm(OP_N, OP_N, nl, ap, nX, -1.0, BXall, ld, c->Y + (size_t)aw * ldm, ldm, 1.0, BP, ld));
    }
    TRY(run.normalize(nl, aw, W, ld, nullptr, 0));
    if (ap > 0) TRY(run.normalize(nl, ap, P, ld, BP, ld));
    // ---- line 6: Rayleigh-Ritz on span(X, R, P) via the pencil (S^T BS, S^T S). Only the direction
    // block of G is needed (X^T X = I, X^T [W P] = 0 by construction); it does not depend on B W, so
    // its Gram and Cholesky run on the side stream, overlapping the block multiply (unsharded mode)
    static int ovl_env = getenv("PSDPROJ_NO_OVERLAP") ? 0 : 1;
    // (R57 / R63 iterations: the last Krylov block is known only after the multiply before it, so the
    // fork sits before the LAST block multiply of the iteration)
    const bool ovl = ovl_env && !c->sharded && s > mU;
    auto fork_chol = [&]() -> int {
      if (!c->st2) {
        // high priority: the 16-CTA cluster Cholesky is dispatched before the block multiply's
        // CTAs, which would otherwise occupy every SM until the multiply ends
        int lo_pr = 0, hi_pr = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo_pr, &hi_pr));
        CK(cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, hi_pr));
        CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        CK(cudaMalloc(&c->d_flag, sizeof(int)));
        CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), st));
        c->chol_seq = 0;
      }
      // the direction-block Gram first (on the main stream), then the Cholesky on the side stream
      TRY(run.gram(s - mU, s - mU, c->S + (size_t)mU * ld, ld, c->S + (size_t)mU * ld, ld, c->G + mU + (size_t)mU * ldm,
                   ldm));
      CK(cudaEventRecord(c->ev_fork, st));
      CK(cudaStreamWaitEvent(c->st2, c->ev_fork, 0));
      Run r2{c, c->st2, info};
      r2.part = c->part2;
      // the block multiply waits (on the device, bounded) until the Cholesky cluster is resident:
      // dispatched after the multiply's CTAs it finds no 8 free SMs and runs after the multiply
      static int hold = getenv("PSDPROJ_CHOL_HOLD") ? atoi(getenv("PSDPROJ_CHOL_HOLD")) : 1;
      const int seq = hold ? ++c->chol_seq : 0;
      TRY(r2.rr_factor(s, mU, hold ? c->d_flag : nullptr, seq));
      CK(cudaEventRecord(c->ev_join, c->st2));
      if (hold) {
        wait_flag_kernel<<<1, 32, 0, st>>>(c->d_flag, seq, 200000LL);
        CKL();
      }
      return 0;
    };
    const bool krylov_it = depth > 1 && aK > 0;
    if (ovl && !krylov_it) TRY(fork_chol());
    TRY(run.mark(0));
    static int hold_env = getenv("PSDPROJ_CHOL_HOLD") ? atoi(getenv("PSDPROJ_CHOL_HOLD")) : 1;
    static const int chol_sms = getenv("PSDPROJ_CHOL_CS") ? std::max(1, atoi(getenv("PSDPROJ_CHOL_CS"))) : 8;
    g_sm_reserve = (ovl && !krylov_it && hold_env) ? chol_sms : 0;  // the Cholesky cluster's CTAs (one SM each)
    rc = run.amul(sgn, A, lda, W, ld, aw, c->BS + (size_t)offW * ld, ld);
    g_sm_reserve = 0;
    TRY(rc);
    // R57: K_k = B K_{k-1} (K_1 = the normalised R_J block), each projected against X_L, X_U and R_J,
    // normalised, and multiplied by B (one more block multiply of a columns per depth level)
    if (depth > 1 && aK > 0) {
      TRY(run.mark(1));
      int offK = offP + ap;
      const double* BKprev = c->BS + (size_t)offW * ld;
      for (int dk = 2; dk <= depth; ++dk, offK += aK) {
        double* K = c->S + (size_t)offK * ld;
        double* BK = c->BS + (size_t)offK * ld;
        TRY(copy_block_pdl(st, nl, aK, K, ld, BKprev, ld));
        // K <- K - [X_L X_U R_J] ([X_L X_U R_J]^T K): the three blocks are contiguous in S and R_J is
        // orthogonal to X (projected above), so one Gram + one update equal the oracle's three
        // successive projections up to rounding
        const int nXW = ((hard && nL > 0) ? nL : 0) + mU + aK;
        const double* XW = (hard && nL > 0) ? XLp() : c->S;
        TRY(run.gram(nXW, aK, XW, ld, K, ld, c->Y, ldm));
        TRY(run.gemm(OP_N, OP_N, nl, aK, nXW, -1.0, XW, ld, c->Y, ldm, 1.0, K, ld));
        TRY(run.normalize(nl, aK, K, ld, nullptr, 0));
        const bool fork_here = ovl && dk == depth;
        if (fork_here) TRY(fork_chol());
        TRY(run.mark(0));
        g_sm_reserve = (fork_here && hold_env) ? chol_sms : 0;
        rc = run.amul(sgn, A, lda, K, ld, aK, BK, ld);
        g_sm_reserve = 0;
        TRY(rc);
        BKprev = BK;
      }
      TRY(run.mark(2));
    }
    TRY(run.mark(2));
    if (!ovl)
      TRY(run.gram(s - mU, s - mU, c->S + (size_t)mU * ld, ld, c->S + (size_t)mU * ld, ld, c->G + mU + (size_t)mU * ldm,
                   ldm));
    TRY(run.gram(s, s, c->S, ld, c->BS, ld, c->Hm, ldm));
    int sU = s;
    // the rotation (a8) and the next iteration's residual norms (a4) are issued before the Rayleigh-
    // Ritz sync, assuming it succeeds (they only read S, BS, C' and the new Ritz values): one host sync
    // per iteration; a failed pivot or a corrective eigensolver pass voids them (issued again below)
    const bool spec_arm = spec_env && !c->sharded;
    const int mUn_spec = std::min(mU + qe, s);
    if (spec_arm) {
      run.spec_fn = [&, mUn_spec, s]() -> int {
        TRY(run.mark(5));
        TRY(dgemm2(st, nl, mUn_spec, s, 1.0, c->S, c->BS, ld, c->Cp, ldm, 0.0, c->S2, c->BS2, ld, c->part,
                   c->part_elems));
        TRY(dgemm2(st, nl, mUn_spec, s - mU, 1.0, c->S + (size_t)mU * ld, c->BS + (size_t)mU * ld, ld, c->Cp + mU,
                   ldm, 0.0, c->Pb, c->BPb, ld, c->part, c->part_elems));
        TRY(run.mark(6));
        TRY(launch_pdl(resid_norm_kernel<256>, dim3(mUn_spec), dim3(256), 0, st, nl, (const double*)c->S2, ld,
                       (const double*)c->BS2, ld, (const double*)c->d_ths, c->R, ld, c->d_r, 0));
        CK(cudaMemcpyAsync(c->h_d + rslot, c->d_r, sizeof(double) * mUn_spec, cudaMemcpyDeviceToHost, st));
        return run.mark(7);
      };
    }
    rc = run.rr(s, mU, mU, c->d_thU, std::min(mU + qe, s), ovl);
    run.spec_fn = nullptr;
    const bool spec_done = spec_arm && rc == 0 && !run.spec_redo;
    // a failed attempt still ran the eigensolver, which uses G / Hm as scratch: a retry forms the
    // pencil again from S, BS
    auto regram = [&](int sr) -> int {
      TRY(run.gram(sr - mU, sr - mU, c->S + (size_t)mU * ld, ld, c->S + (size_t)mU * ld, ld,
                   c->G + mU + (size_t)mU * ldm, ldm));
      return run.gram(sr, sr, c->S, ld, c->BS, ld, c->Hm, ldm);
    };
    if (rc > 0 && s > offP) {
      sU = offP;  // drop P (and the Krylov blocks after it, R57) and retry (R20)
      TRY(regram(sU));
      rc = run.rr(sU, mU, mU, c->d_thU, std::min(mU + qe, sU));
    }
    // R41: still rank deficient -> truncate the basis at the failing pivot: the leading columns
    // (whose Cholesky factor is the leading block of the failed one) are kept, the direction at
    // the pivot and those after it wait for the next iteration (one retry instead of one per
    // dependent column; the oracle's Householder fallback drops near-dependent columns)
    while (rc > 0 && sU > mU) {
      const int col = rc - 1;  // failing column of the basis (index in S)
      if (col < mU || col >= sU) return set_err(PSDPROJ_E_DEGENERATE, "Cholesky-QR failed at pivot %d (s=%d)", rc, sU);
      info->dropped += sU - col;
      sU = col;
      TRY(regram(sU));
      rc = run.rr(sU, mU, mU, c->d_thU, std::min(mU + qe, sU));
    }
    if (rc > 0) return set_err(PSDPROJ_E_DEGENERATE, "Cholesky-QR failed at pivot %d (s=%d)", rc, sU);
    TRY(rc);
    int mUn = std::min(mU + qe, sU);
    std::vector<double> ths(c->h_d, c->h_d + mUn);
    const int rr_npos = run.rr_npos;
    // ---- rotation (a8): X <- S C', BX <- BS C', P <- S_[R P] C'_[R P], BP likewise
    TRY(run.mark(5));
    // X and BX (S C', BS C') in one launch, P and BP likewise (already issued when spec_done)
    if (!spec_done) {
      TRY(dgemm2(st, nl, mUn, sU, 1.0, c->S, c->BS, ld, c->Cp, ldm, 0.0, c->S2, c->BS2, ld, c->part, c->part_elems));
      TRY(dgemm2(st, nl, mUn, sU - mU, 1.0, c->S + (size_t)mU * ld, c->BS + (size_t)mU * ld, ld, c->Cp + mU, ldm,
                 0.0, c->Pb, c->BPb, ld, c->part, c->part_elems));
    }
    spec_ready = spec_done;
    info->flops += 8.0 * nl * (double)mUn * sU;
    std::swap(c->S, c->S2);
    std::swap(c->BS, c->BS2);
    if (getenv("PSDPROJ_TRACE")) {  // debugging: orthonormality of the new block
      std::vector<double> hY((size_t)ldm * std::max(mUn, 1));
      TRY(run.gram(mUn, mUn, c->S, ld, c->S, ld, c->Y, ldm));
      TRY(run.sync());
      CK(cudaMemcpy(hY.data(), c->Y, sizeof(double) * (size_t)ldm * mUn, cudaMemcpyDeviceToHost));
      double oU = 0;
      for (int j = 0; j < mUn; ++j)
        for (int i = 0; i < mUn; ++i) oU = std::max(oU, std::fabs(hY[(size_t)j * ldm + i] - (i == j)));
      double oL = 0;
      if (nL > 0) {
        TRY(run.gram(nL, mUn, XLp(), ld, c->S, ld, c->Y, ldm));
        TRY(run.sync());
        CK(cudaMemcpy(hY.data(), c->Y, sizeof(double) * (size_t)ldm * mUn, cudaMemcpyDeviceToHost));
        for (int j = 0; j < mUn; ++j)
          for (int i = 0; i < nL; ++i) oL = std::max(oL, std::fabs(hY[(size_t)j * ldm + i]));
      }
      fprintf(stderr, "   rotation: s=%d mUn=%d |XU'XU-I| %g |XL'XU| %g  theta %g..%g\n", sU, mUn, oU, oL,
              ths.empty() ? 0.0 : ths.back(), ths.empty() ? 0.0 : ths.front());
    }
    TRY(copy_block_pdl(st, mUn, 1, c->d_thU, mUn, c->d_ths, mUn));
    thU.assign(ths.begin(), ths.begin() + mUn);
    rU.assign(mUn, INFINITY);
    hasP.assign(mUn, 1);
    mU = mUn;
    qe = 0;
    ++k;
    // ---- line 8: expansion when fewer than g guards would remain (R8)
    TRY(run.mark(7));
    int p_rr = (hard ? nL : 0) + rr_npos;  // positive RR values among all sU (R8)
    int mt = nL + mU;
    if (p_rr >= mt - g + 1 && mt < n) {
      int qq = std::min(c->q, n - mt);
      if (mt + qq > c->m_max) {  // R18: the block reached the exact-eig regime (m_max = ceil(n/3)+1)
        if (c->sharded) return set_err(PSDPROJ_E_CAPACITY, "block %d exceeds m_max %d (no DIRECT in sharded mode)", mt + qq, c->m_max);
        abort_direct = true;
        return PSDPROJ_OK;
      }
      TRY(run.philox(qq, c->E, ld, (uint32_t)k));
      for (int pass = 0; pass < 2; ++pass) {
        if (nL > 0) {
          TRY(run.gram(nL, qq, XLp(), ld, c->E, ld, c->Y, ldm));
          TRY(run.gemm(OP_N, OP_N, nl, qq, nL, -1.0, XLp(), ld, c->Y, ldm, 1.0, c->E, ld));
        }
        TRY(run.gram(mU, qq, c->S, ld, c->E, ld, c->Y, ldm));
        TRY(run.gemm(OP_N, OP_N, nl, qq, mU, -1.0, c->S, ld, c->Y, ldm, 1.0, c->E, ld));
      }
      qe = qq;
      info->expansions++;
    }
  }
  TRY(run.mark(7));
  info->iters = k;
  info->status = status;
  info->locked = nL;
  // ---- kept pairs: theta > 0 over L and U
  std::vector<int> lpos, upos;
  std::vector<double> wts;
  double rs = 0.0, rmax = 0.0;
  for (int j = 0; j < nL; ++j)
    if (thL[j] > 0) { lpos.push_back(j); wts.push_back(thL[j]); rs += rL[j] * rL[j]; rmax = std::max(rmax, rL[j]); }
  for (int j = 0; j < mU; ++j)
    if (thU[j] > 0) { upos.push_back(j); wts.push_back(thU[j]); rs += rU[j] * rU[j]; rmax = std::max(rmax, rU[j]); }
  int p = (int)wts.size();
  double* V = c->T;
  double* BV = c->T2;
  TRY(run.gather(nl, (int)lpos.size(), V, ld, XLp(), ld, lpos));
  TRY(run.gather(nl, (int)upos.size(), V + (size_t)lpos.size() * ld, ld, c->S, ld, upos));
  for (int j = 0; j < p; ++j) c->h_d[j] = wts[j];
  CK(cudaMemcpyAsync(c->d_w, c->h_d, sizeof(double) * std::max(p, 1), cudaMemcpyHostToDevice, st));
  // ---- a10 (R16, R36, R53): certify the returned pairs with an explicit B V+ (one block multiply
  // of the p kept columns; B V+ of the rotation and of the frozen locked columns is not used)
  double thmax = 0.0, th2 = 0.0;
  for (double x : wts) {
    thmax = std::max(thmax, x);
    th2 += x * x;
  }
  info->pi_fro = std::sqrt(th2);  // ||V Theta+ V^T||_F (side +) -- of the computed side's part
  Cert ct;
  TRY(certify(run, sgn, A, lda, V, p, c->d_w, BV, c->Y, ldm, false, ct));
  rs = 0.0;
  rmax = 0.0;
  for (int j = 0; j < p; ++j) {
    rs += ct.r2[j];
    rmax = std::max(rmax, std::sqrt(ct.r2[j]));
  }
  // ---- f2 (R48): the perp term by projected Lanczos on (I - V V^T) B (I - V V^T), V = the kept
  // positive Ritz vectors: a randomized upper bound that holds with probability >= 1 - perp_delta
  // over the Philox start (0 unless perp_steps > 0: the paper ignores the term)
  double perp = 0.0;
  if (c->prm.perp_steps > 0) TRY(perp_estimate(run, sgn, A, lda, V, p, c->prm.perp_steps, &perp));
  info->perp_est = perp;
  // ---- Theorem 3 bound (R14-R16, R36, R53)
  info->resid_fro = std::sqrt(rs);
  info->resid_max = rmax;
  info->lock_defect = ct.defect;
  info->orth_defect = ct.orth;
  info->err_bound = theorem3_bound(n, rs, perp, ct.defect, ct.orth, thmax, run.anorm);
  info->npos = p;
  // ---- a11: Pi = V Theta+ V^T (side +) or A + V Theta+ V^T (side -, pairs of -A)
  if (sgn < 0 && Pi != A) {
    CK(cudaMemcpy2DAsync(Pi, (size_t)ldpi * 8, A, (size_t)lda * 8, (size_t)nl * 8, n, cudaMemcpyDeviceToDevice, st));
  }
  if (p > 0 && !c->sharded) {
    scale_copy_cols_kernel<<<grid1d((size_t)n * p), 256, 0, st>>>(n, p, c->E, ld, V, ld, c->d_w);
    CKL();
    TRY(run.gemm(OP_N, OP_T, n, n, p, 1.0, c->E, ld, V, ld, sgn < 0 ? 1.0 : 0.0, Pi, ldpi));
    symmetrize_kernel<<<grid1d((size_t)n * n), 256, 0, st>>>(n, Pi, ldpi);
    CKL();
  } else if (p > 0) {
    // row-sharded: Pi_local = W_local W^T with W = V diag(sqrt(theta+)) (each entry a sum of identical
    // products in the same order on both sides of the diagonal), W gathered from the ranks
    scale_sqrt_cols_kernel<<<grid1d((size_t)nl * p), 256, 0, st>>>(nl, p, c->E, ld, V, ld, c->d_w);
    CKL();
    TRY(run.gather_full(c->E, ld, p));
    TRY(run.gemm(OP_N, OP_T, nl, n, p, 1.0, c->E, ld, c->zfull, c->ldn, sgn < 0 ? 1.0 : 0.0, Pi, ldpi));
  } else if (sgn > 0) {
    CK(cudaMemset2DAsync(Pi, (size_t)ldpi * 8, 0, (size_t)nl * 8, n, st));
  }
  // ---- a12: warm block for the next call: all columns by theta desc, first p + extra
  struct Col { double th; int src; int j; };
  std::vector<Col> cols;
  for (int j = 0; j < nL; ++j) cols.push_back({thL[j], 0, j});
  for (int j = 0; j < mU; ++j) cols.push_back({thU[j], 1, j});
  std::stable_sort(cols.begin(), cols.end(), [](const Col& x, const Col& y) { return x.th > y.th; });
  int mtot = nL + mU;
  int keepn = std::min(keep_count(c, p, mtot), c->m_max);
  // gather L-sourced then U-sourced into Xw preserving the sorted order via T2 staging
  std::vector<int> li, ui, pos_l, pos_u;
  for (int i = 0; i < keepn; ++i) {
    if (cols[i].src == 0) { li.push_back(cols[i].j); pos_l.push_back(i); }
    else { ui.push_back(cols[i].j); pos_u.push_back(i); }
  }
  TRY(run.gather(nl, (int)li.size(), c->T2, ld, XLp(), ld, li));
  TRY(run.gather(nl, (int)ui.size(), c->T2 + (size_t)li.size() * ld, ld, c->S, ld, ui));
  std::vector<int> perm(keepn);  // Xw[:, pos] = T2[:, staged index]
  for (size_t i = 0; i < pos_l.size(); ++i) perm[pos_l[i]] = (int)i;
  for (size_t i = 0; i < pos_u.size(); ++i) perm[pos_u[i]] = (int)(li.size() + i);
  TRY(run.gather(nl, keepn, c->Xw, ld, c->T2, ld, perm));
  c->m_warm = keepn;
  c->th_warm.clear();
  for (int i = 0; i < keepn; ++i) c->th_warm.push_back(cols[i].th);
  c->block_side = side;
  c->warm = true;
  // ---- counts for the side rule (computed side p, other side n - p)
  if (side == PSDPROJ_SIDE_POS) { c->last_pos = p; c->last_neg = n - p; }
  else { c->last_neg = p; c->last_pos = n - p; }
  c->have_counts = true;
  info->m = mtot;
  info->bytes += 8.0 * n * (double)n * (sgn < 0 ? 2 : 1);
  info->flops += (double)n * (n + 1) * p;
  return status;
}

static int project_impl(psdproj_ctx c, const double* A, int lda, double* Pi, int ldpi, double tol, cudaStream_t st,
                        psdproj_info* info) {
  int n = c->n;
  // first pass: non-finite check and ||A||_F (deterministic partials, host sums in order)
  const int nl = c->nr;
  int nb = c->sharded ? sms() * 2 : std::min(sms() * 2, std::max(1, (int)(((size_t)nl * n + 255) / 256)));
  CK(cudaMemsetAsync(c->d_status + 8, 0, sizeof(int), st));
  nonfinite_kernel<<<nb, 256, 0, st>>>(nl, n, A, lda, c->d_status + 8);
  CKL();
  fro_partial_kernel<<<nb, 256, 0, st>>>(nl, n, A, lda, c->T2);
  CKL();
  if (c->sharded) {  // every rank needs the global ||A||_F and the non-finite flag
    int* flag = c->d_status + 8;
    double* fl = c->T2 + nb;
    i2d_kernel<<<1, 32, 0, st>>>(flag, fl);
    CKL();
    NK(g_nccl.allReduce(c->T2, c->T2, (size_t)nb + 1, ncclFloat64, ncclSum, c->comm, st));
    d2i_kernel<<<1, 32, 0, st>>>(fl, flag);
    CKL();
  }
  CK(cudaMemcpyAsync(c->h_d, c->T2, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c->h_i + c->h_i_len - 32, c->d_status + 8, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (c->h_i[c->h_i_len - 32]) return set_err(PSDPROJ_E_NONFINITE, "A contains inf/nan");
  double fro2 = 0.0;
  for (int i = 0; i < nb; ++i) fro2 += c->h_d[i];
  Run run{c, st, info};
  long long launches0 = g_launches - 2;  // count the two first-pass kernels
  run.anorm = std::sqrt(fro2);
  info->anorm_f = run.anorm;
  int mode = select_mode(c);
  int call = c->calls++;
  (void)call;
  if (mode != PSDPROJ_SIDE_DIRECT) {
    int mstart = (c->warm && c->block_side == mode) ? c->m_warm : c->m0;
    if (3 * mstart >= n) mode = PSDPROJ_SIDE_DIRECT;  // R18
  }
  if (mode == PSDPROJ_SIDE_DIRECT && c->sharded)
    return set_err(PSDPROJ_E_CAPACITY, "the one-third rule selects the exact eigensolver (PAPER.md:505), which the row-sharded mode does not provide");
  int rc;
  if (mode == PSDPROJ_SIDE_DIRECT) {
    rc = direct_path(run, A, lda, Pi, ldpi);
    info->status = rc;
  } else {
    bool abort_direct = false;
    rc = lobpcg_path(run, mode, A, lda, Pi, ldpi, tol, abort_direct);
    if (rc >= 0 && abort_direct) {
      rc = direct_path(run, A, lda, Pi, ldpi);
      info->status = rc;
    }
  }
  if (rc < 0) return rc;
  info->last_pos = c->last_pos;
  info->last_neg = c->last_neg;
  info->launches = (int)(g_launches - launches0);
  CK(cudaStreamSynchronize(st));
  if ((c->prm.profile & 2) && !run.marks.empty()) {
    TRY(run.mark(7));
    CK(cudaEventSynchronize(c->pev[run.marks.size() - 1]));
    for (size_t i = 0; i + 1 < run.marks.size(); ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->pev[i], c->pev[i + 1]));
      info->phase_ms[run.marks[i]] += ms;
    }
  }
  if ((c->prm.profile & 1) && run.nev > 0) {
    double tot = 0.0;
    for (int i = 0; i < run.nev; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]));
      tot += ms;
    }
    info->amul_ms = tot;
    info->amul_launches = run.nev;
  }
  if ((c->prm.profile & 4) && run.ntev > 0) {
    double tot = 0.0;
    for (int i = 0; i < run.ntev; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->tev[2 * i], c->tev[2 * i + 1]));
      tot += ms;
    }
    info->tri_ms = tot;
    info->tri_launches = run.ntev;
  }
  return rc;
}

extern "C" int psdproj_project(psdproj_ctx c, const double* A, int lda, double* Pi, int ldpi, double tol,
                               void* stream, psdproj_info* info) {
  psdproj_info local;
  if (!info) info = &local;
  std::memset(info, 0, sizeof(*info));
  if (!c) return info->status = set_err(PSDPROJ_E_INVALID, "ctx NULL");
  if (c->poisoned) return info->status = set_err(PSDPROJ_E_CUDA, "context poisoned by an earlier CUDA error");
  if (!A || !Pi || lda < c->nr || ldpi < c->nr || !(tol > 0.0) || !std::isfinite(tol))
    return info->status = set_err(PSDPROJ_E_INVALID, "invalid arguments (lda=%d ldpi=%d tol=%g)", lda, ldpi, tol);
  if ((const void*)Pi == (const void*)A && lda != ldpi)
    return info->status = set_err(PSDPROJ_E_INVALID, "aliased Pi needs ldpi == lda");
  const auto t0 = std::chrono::steady_clock::now();
  const double s0 = g_sync_s;
  const long n0 = g_nsync;
  int rc = project_impl(c, A, lda, Pi, ldpi, tol, (cudaStream_t)stream, info);
  if (g_hostprof) {
    // host-side time split of the call: blocked in stream syncs vs issuing work
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[psdproj hostprof] wall %.1f ms, in syncs %.1f ms (%ld), issuing %.1f ms, iters %d, launches %ld\n",
                 1e3 * wall, 1e3 * (g_sync_s - s0), g_nsync - n0, 1e3 * (wall - (g_sync_s - s0)), info->iters,
                 (long)info->launches);
  }
  if (rc == PSDPROJ_E_CUDA) c->poisoned = true;
  info->status = rc;
  return rc;
}

extern "C" int psdproj_project_host(psdproj_ctx c, const double* A_host, int lda, double* Pi_host, int ldpi,
                                    double tol, void* stream, psdproj_info* info) {
  psdproj_info local;
  if (!info) info = &local;
  std::memset(info, 0, sizeof(*info));
  if (!c || !c->stage || c->sharded) return info->status = set_err(PSDPROJ_E_INVALID, "ctx NULL, sharded, or created without host_io");
  if (!A_host || !Pi_host || lda < c->n || ldpi < c->n) return info->status = set_err(PSDPROJ_E_INVALID, "invalid arguments");
  cudaStream_t st = (cudaStream_t)stream;
  int n = c->n, ld = c->ld;
  CK(cudaMemcpy2DAsync(c->stage, (size_t)ld * 8, A_host, (size_t)lda * 8, (size_t)n * 8, n, cudaMemcpyHostToDevice, st));
  int rc = psdproj_project(c, c->stage, ld, c->stage, ld, tol, stream, info);
  if (rc < 0) return rc;
  CK(cudaMemcpy2DAsync(Pi_host, (size_t)ldpi * 8, c->stage, (size_t)ld * 8, (size_t)n * 8, n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return rc;
}

// ------------------------------------------------------------------ f4: many tiny cone blocks
extern "C" int psdproj_project_tiny_batched(int count, const int* n, const double* const* A, const int* lda,
                                            double* const* Pi, const int* ldpi, int* npos_host, void* stream) {
  if (count < 0 || (count > 0 && (!n || !A || !lda || !Pi || !ldpi)))
    return set_err(PSDPROJ_E_INVALID, "invalid tiny-batch arguments");
  if (count == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int nmax = 0;
  std::vector<TinyBlock> hb((size_t)count);
  for (int i = 0; i < count; ++i) {
    if (n[i] < 0 || n[i] > JAC_SMEM_MAX || (n[i] > 0 && (!A[i] || !Pi[i] || lda[i] < n[i] || ldpi[i] < n[i])))
      return set_err(n[i] > JAC_SMEM_MAX ? PSDPROJ_E_CAPACITY : PSDPROJ_E_INVALID,
                     "tiny block %d: n = %d (supported 0..%d)", i, n[i], JAC_SMEM_MAX);
    hb[i] = TinyBlock{A[i], Pi[i], n[i], lda[i], ldpi[i], 0};
    nmax = std::max(nmax, n[i]);
  }
  // per-thread device descriptor / count buffers, grown on demand (batched calls from threads)
  static thread_local TinyBlock* dblk = nullptr;
  static thread_local int* dnpos = nullptr;
  static thread_local int cap = 0;
  if (count > cap) {
    if (dblk) cudaFree(dblk);
    if (dnpos) cudaFree(dnpos);
    cap = std::max(count, 2 * cap);
    CK(cudaMalloc(&dblk, sizeof(TinyBlock) * cap));
    CK(cudaMalloc(&dnpos, sizeof(int) * cap));
  }
  CK(cudaMemcpyAsync(dblk, hb.data(), sizeof(TinyBlock) * count, cudaMemcpyHostToDevice, st));
  const int N = nmax + (nmax & 1);
  const size_t smem = (size_t)2 * N * (N + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(tiny_project_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  tiny_project_kernel<256><<<count, 256, smem, st>>>(dblk, 60, dnpos);
  CKL();
  if (npos_host) {
    CK(cudaMemcpyAsync(npos_host, dnpos, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int i = 0; i < count; ++i)
      if (npos_host[i] < 0) return set_err(PSDPROJ_E_DEGENERATE, "tiny block %d: Jacobi did not converge", i);
  } else {
    CK(cudaStreamSynchronize(st));  // the host descriptor array may be reused by the caller
  }
  return 0;
}

// ------------------------------------------------------------------ f4: one-CTA warm LOBPCG per tiny block
extern "C" size_t psdproj_tiny_lobpcg_ws_bytes(int count) {
  return count <= 0 ? 0 : (size_t)count * (sizeof(TinyLobBlock) + sizeof(TinyLobOut)) + 512;
}

extern "C" int psdproj_project_tiny_lobpcg(int count, const int* n, const double* const* A, const int* lda,
                                           double* const* Pi, const int* ldpi, double* const* Xw, int* m_state,
                                           double tol, int max_iter, int guard, int m0, uint64_t seed, uint32_t call,
                                           void* ws, size_t ws_bytes, int* status, int* iters, int* npos,
                                           double* bound, void* stream) {
  if (count < 0 || (count > 0 && (!n || !A || !lda || !Pi || !ldpi || !Xw || !m_state || !ws || !status || !iters ||
                                   !npos || !bound)) ||
      !(tol > 0.0) || max_iter < 0 || guard < 1 || m0 < 1)
    return set_err(PSDPROJ_E_INVALID, "invalid tiny-LOBPCG arguments");
  if (count == 0) return 0;
  if (ws_bytes < psdproj_tiny_lobpcg_ws_bytes(count) || ((uintptr_t)ws & 15))
    return set_err(PSDPROJ_E_WORKSPACE, "tiny-LOBPCG workspace too small / misaligned");
  cudaStream_t st = (cudaStream_t)stream;
  int nmax = 1;
  std::vector<TinyLobBlock> hb((size_t)count);
  std::vector<TinyLobOut> ho((size_t)count);
  for (int i = 0; i < count; ++i) {
    if (n[i] < 1 || n[i] > TL_NMAX || !A[i] || !Pi[i] || !Xw[i] || lda[i] < n[i] || ldpi[i] < n[i])
      return set_err(n[i] > TL_NMAX ? PSDPROJ_E_CAPACITY : PSDPROJ_E_INVALID, "tiny block %d: n = %d (1..%d)", i, n[i],
                     TL_NMAX);
    static const int dbg = getenv("PSDPROJ_TINY_DEBUG") ? atoi(getenv("PSDPROJ_TINY_DEBUG")) : -1;
    hb[i] = TinyLobBlock{A[i], Pi[i], Xw[i], n[i], lda[i], ldpi[i], i == dbg ? 1 : 0};
    ho[i] = TinyLobOut{0.0, 0.0, 0, 0, 0, std::max(0, std::min(m_state[i], TL_MCAP))};
    nmax = std::max(nmax, n[i]);
  }
  TinyLobBlock* dblk = reinterpret_cast<TinyLobBlock*>(ws);
  TinyLobOut* dout = reinterpret_cast<TinyLobOut*>(
      (char*)ws + (((size_t)count * sizeof(TinyLobBlock) + 255) / 256) * 256);
  CK(cudaMemcpyAsync(dblk, hb.data(), sizeof(TinyLobBlock) * count, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dout, ho.data(), sizeof(TinyLobOut) * count, cudaMemcpyHostToDevice, st));
  const size_t smem = tiny_lob_smem_doubles(nmax) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(tiny_lobpcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(tiny_lob_smem_doubles(TL_NMAX) * sizeof(double))));
    attr = true;
  }
  tiny_lobpcg_kernel<<<count, TL_NT, smem, st>>>(dblk, dout, tol, max_iter, guard, m0, seed, call);
  CKL();
  CK(cudaMemcpyAsync(ho.data(), dout, sizeof(TinyLobOut) * count, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // blocks the one-CTA LOBPCG hands back (capacity / singular pencil): the exact one-CTA path (R50)
  std::vector<int> xn, xl, xp, xi;
  std::vector<const double*> xa;
  std::vector<double*> xpi;
  for (int i = 0; i < count; ++i) {
    status[i] = ho[i].status;
    iters[i] = ho[i].iters;
    npos[i] = ho[i].npos;
    bound[i] = ho[i].bound;
    m_state[i] = ho[i].m;
    if (ho[i].status == TL_NEEDS_EXACT) {
      xi.push_back(i);
      xn.push_back(n[i]);
      xa.push_back(A[i]);
      xl.push_back(lda[i]);
      xpi.push_back(Pi[i]);
      xp.push_back(ldpi[i]);
    }
  }
  if (!xi.empty()) {
    std::vector<int> np(xi.size());
    TRY(psdproj_project_tiny_batched((int)xi.size(), xn.data(), xa.data(), xl.data(), xpi.data(), xp.data(), np.data(),
                                     stream));
    for (size_t k = 0; k < xi.size(); ++k) {
      npos[xi[k]] = np[k];
      status[xi[k]] = 3;  // computed by the exact path (no LOBPCG bound; Jacobi to rounding level)
      bound[xi[k]] = 0.0;
      m_state[xi[k]] = 0;
    }
  }
  return 0;
}

extern "C" int psdproj_project_batched(psdproj_ctx* ctxs, int count, const double* const* A, const int* lda,
                                       double* const* Pi, const int* ldpi, const double* tol, void* stream,
                                       psdproj_info* infos) {
  if (count < 0 || (count > 0 && (!ctxs || !A || !lda || !Pi || !ldpi || !tol || !infos)))
    return set_err(PSDPROJ_E_INVALID, "invalid batched arguments");
  if (count == 0) return PSDPROJ_OK;
  for (int i = 0; i < count; ++i)
    for (int k = 0; k < i && k < 64; ++k)
      if (ctxs[k] == ctxs[i]) return set_err(PSDPROJ_E_INVALID, "batched contexts must be distinct");
  // Independent blocks are driven by up to PSDPROJ_BATCH_THREADS host threads (default 8); every item
  // runs on its own context's stream (created once, destroyed with the context), forked from and
  // joined back to the caller's stream by the context's events, so the latency-bound per-iteration
  // work of different blocks overlaps on the GPU and no stream or event is created per call.
  int nth = 8;
  if (const char* e = getenv("PSDPROJ_BATCH_THREADS")) nth = std::max(1, atoi(e));
  nth = std::min(nth, count);
  cudaStream_t st = (cudaStream_t)stream;
  if (nth == 1) {
    int worst = PSDPROJ_OK;
    for (int i = 0; i < count; ++i) {
      int rc = psdproj_project(ctxs[i], A[i], lda[i], Pi[i], ldpi[i], tol[i], stream, &infos[i]);
      if (rc < 0) return rc;
      worst = std::max(worst, rc);
    }
    return worst;
  }
  for (int i = 0; i < count; ++i) {
    psdproj_ctx c = ctxs[i];
    if (!c) return set_err(PSDPROJ_E_INVALID, "ctx NULL in batch");
    if (!c->bst) {
      CK(cudaStreamCreateWithFlags(&c->bst, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->bev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->bev_join, cudaEventDisableTiming));
    }
  }
  CK(cudaEventRecord(ctxs[0]->bev_fork, st));
  for (int i = 0; i < count; ++i) CK(cudaStreamWaitEvent(ctxs[i]->bst, ctxs[0]->bev_fork, 0));
  std::vector<int> rcs(nth, PSDPROJ_OK);
  std::vector<std::string> errs(nth);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::vector<std::thread> th;
  for (int t = 0; t < nth; ++t) {
    th.emplace_back([&, t]() {
      cudaSetDevice(dev);
      int worst = PSDPROJ_OK;
      for (int i = t; i < count; i += nth) {
        int rc = psdproj_project(ctxs[i], A[i], lda[i], Pi[i], ldpi[i], tol[i], ctxs[i]->bst, &infos[i]);
        if (rc < 0) {
          worst = rc;
          errs[t] = g_err;
          break;
        }
        worst = std::max(worst, rc);
      }
      rcs[t] = worst;
    });
  }
  for (auto& x : th) x.join();
  int worst = PSDPROJ_OK;
  for (int i = 0; i < count; ++i) {
    CK(cudaEventRecord(ctxs[i]->bev_join, ctxs[i]->bst));
    CK(cudaStreamWaitEvent(st, ctxs[i]->bev_join, 0));
  }
  for (int t = 0; t < nth; ++t) {
    if (rcs[t] < 0 && worst >= 0) {
      worst = rcs[t];
      g_err = errs[t];
    } else if (worst >= 0) {
      worst = std::max(worst, rcs[t]);
    }
  }
  return worst;
}

extern "C" int psdproj_get_ritz(psdproj_ctx c, double* vals_host, int cap, double* vecs_dev, int ldv) {
  if (!c) return set_err(PSDPROJ_E_INVALID, "ctx NULL");
  if (!c->warm) return 0;
  int k = std::min(cap, c->m_warm);
  if (vals_host)
    for (int i = 0; i < k; ++i) vals_host[i] = c->th_warm[i];
  if (vecs_dev && k > 0) {
    if (ldv < c->nr) return set_err(PSDPROJ_E_INVALID, "ldv < rows held by this context");
    CK(cudaMemcpy2D(vecs_dev, (size_t)ldv * 8, c->Xw, (size_t)c->ld * 8, (size_t)c->nr * 8, k, cudaMemcpyDeviceToDevice));
  }
  return k;
}

// ------------------------------------------------------------------ kernel-level entry points
extern "C" int psdproj_dgemm(int opA, int opB, int M, int N, int K, double alpha, const double* A, int lda,
                             const double* B, int ldb, double beta, double* C, int ldc, double* ws, size_t ws_elems,
                             void* stream) {
  if (M < 0 || N < 0 || K < 0 || (opA != 0 && opA != 1) || (opB != 0 && opB != 1))
    return set_err(PSDPROJ_E_INVALID, "invalid gemm arguments");
  if (lda < std::max(1, opA == OP_N ? M : K) || ldb < std::max(1, opB == OP_N ? K : N) || ldc < std::max(1, M))
    return set_err(PSDPROJ_E_INVALID, "invalid leading dimension");
  int rc = dgemm((cudaStream_t)stream, opA, opB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws ? ws_elems : 0);
  return rc;
}

extern "C" int psdproj_symm_multiply(int n, int k, double alpha, const double* A, int lda, const double* Z, int ldz,
                                     double* Y, int ldy, double* ws, size_t ws_elems, void* stream) {
  if (n <= 0 || k <= 0 || lda < n || ldz < n || ldy < n || !A || !Z || !Y)
    return set_err(PSDPROJ_E_INVALID, "invalid symm_multiply arguments");
  if (lda % 2 || ldz % 2 || ((uintptr_t)A & 15) || ((uintptr_t)Z & 15))
    return set_err(PSDPROJ_E_INVALID, "symm_multiply needs even leading dimensions and 16-byte aligned A, Z");
  return a3_multiply_tma((cudaStream_t)stream, n, k, alpha, A, lda, Z, ldz, Y, ldy, ws, ws ? ws_elems : 0);
}

extern "C" size_t psdproj_jacobi_ws_elems(int s) {
  size_t N = (size_t)(s + (s & 1));
  return 3 * N * N + 256;
}

extern "C" int psdproj_jacobi(int s, const double* A, int lda, double* w, double* V, int ldv, double* ws,
                              void* stream) {
  if (s <= 0 || lda < s || ldv < s || !A || !w || !V || !ws) return set_err(PSDPROJ_E_INVALID, "invalid jacobi args");
  cudaStream_t st = (cudaStream_t)stream;
  size_t N = (size_t)(s + (s & 1));
  double* M = ws;
  double* M2 = ws + N * N;
  double* Q = ws + 2 * N * N;
  int* d_info = (int*)(ws + 3 * N * N);
  int* d_cnt = d_info + 8;
  double* d_fro = ws + 3 * N * N + 128;
  TRY(jacobi_run(st, s, A, lda, w, V, ldv, M, M2, Q, d_info, d_cnt, d_fro));
  int hinfo = 0;
  CK(cudaMemcpyAsync(&hinfo, d_info, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hinfo < 0) return set_err(PSDPROJ_E_DEGENERATE, "Jacobi did not converge");
  // ascending order for the kernel-level API
  return hinfo;
}

extern "C" int psdproj_philox_raw(int count, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                                  uint32_t* out, void* stream) {
  if (count < 0 || (count > 0 && !out)) return set_err(PSDPROJ_E_INVALID, "invalid philox args");
  if (count == 0) return 0;
  philox_raw_kernel<<<grid1d(count), 256, 0, (cudaStream_t)stream>>>(count, c1, c2, c3, k0, k1, out);
  CKL();
  return 0;
}

extern "C" int psdproj_philox_gauss(int n, int q, double* out, int ld, uint64_t seed, uint32_t stream_id, uint32_t ctx,
                                    uint32_t tag, void* stream) {
  if (n < 0 || q < 0 || ld < n || (n * (size_t)q > 0 && !out)) return set_err(PSDPROJ_E_INVALID, "invalid gauss args");
  if ((size_t)n * q == 0) return 0;
  philox_gauss_kernel<<<grid1d(((size_t)n * q + 1) / 2), 256, 0, (cudaStream_t)stream>>>(n, q, out, ld, seed,
                                                                                           stream_id, ctx, tag);
  CKL();
  return 0;
}

extern "C" size_t psdproj_eigh_ws_elems(int s, int m) {
  size_t mm = (size_t)std::max(m, 1);
  return (size_t)5 * s + 64 + (size_t)6 * s * mm + 2 * (size_t)s * s + 16 * (size_t)s + 2048 + 2 * mm * mm + (size_t)s * mm + 64;
}

extern "C" int psdproj_eigh(int s, const double* A, int lda, int m, double* w, double* V, int ldv, int* npos,
                            double* ws, void* stream) {
  if (s <= 0 || m < 0 || m > s || lda < s || ldv < s || !A || !w || !V || !npos || !ws)
    return set_err(PSDPROJ_E_INVALID, "invalid eigh args");
  cudaStream_t st = (cudaStream_t)stream;
  size_t mm = (size_t)std::max(m, 1);
  EighScratch e;
  e.td = ws;
  e.te = e.td + s;
  e.ttau = e.te + s;
  e.te2 = e.ttau + s;
  e.tbounds = e.te2 + s + 8;
  e.dev = reinterpret_cast<unsigned long long*>(e.tbounds + 16);
  e.tscr = e.tbounds + 56;
  e.tscr_elems = (size_t)6 * s * mm;
  e.tG = e.tscr + e.tscr_elems;
  e.ldg = s;
  e.Vh = e.tG + (size_t)s * s + 16 * (size_t)s + 2048;
  e.ldv = s;
  e.nsM = e.Vh + (size_t)s * s;
  e.nsZ = e.nsM + mm * mm;
  e.nsY = e.nsZ + mm * mm;
  // the side stream and its events live for this call only
  CK(cudaStreamCreateWithFlags(&e.side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&e.ev_f, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&e.ev_j, cudaEventDisableTiming));
  auto release = [&]() {
    cudaStreamSynchronize(e.side);
    cudaEventDestroy(e.ev_f);
    cudaEventDestroy(e.ev_j);
    cudaStreamDestroy(e.side);
  };
  int rc = eigh_top(st, s, A, lda, m, w, V, ldv, npos, e, nullptr, 0, false);
  double dev = 0.0;
  if (rc >= 0 && cudaMemcpyAsync(&dev, e.dev, sizeof(double), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
      cudaStreamSynchronize(st) == cudaSuccess) {
    if (!(dev <= 1e-7)) {
      rc = eigh_top(st, s, A, lda, m, w, V, ldv, npos, e, nullptr, 0, true);
      if (rc >= 0 && cudaStreamSynchronize(st) != cudaSuccess) rc = set_err(PSDPROJ_E_CUDA, "psdproj_eigh sync");
    }
  } else if (rc >= 0) {
    rc = set_err(PSDPROJ_E_CUDA, "psdproj_eigh sync");
  }
  release();
  return rc < 0 ? rc : 0;
}

extern "C" int psdproj_cholesky(int t, double* G, int ld, void* stream) {
  if (t <= 0 || ld < t || !G) return set_err(PSDPROJ_E_INVALID, "invalid cholesky args");
  cudaStream_t st = (cudaStream_t)stream;
  int* d_status = nullptr;
  CK(cudaMallocAsync(&d_status, sizeof(int), st));
  CK(cudaMemsetAsync(d_status, 0, sizeof(int), st));
  const size_t gel = (size_t)16 * chol_local_cols(t, 16) * t;
  double* gs = nullptr;
  CK(cudaMallocAsync(&gs, gel * sizeof(double), st));
  int rc = cholesky_run(st, t, G, ld, d_status, gs, gel);
  int h = 0;
  if (rc == 0) CK(cudaMemcpyAsync(&h, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(d_status, st));
  CK(cudaFreeAsync(gs, st));
  CK(cudaStreamSynchronize(st));
  return rc < 0 ? rc : h;
}

// ------------------------------------------------------------------ f1/f3: approximate ADMM (diagonal SDP)
extern "C" int psdproj_admm_maxcut_step1(int n, double* X, const double* Zp, const double* Yp, const double* ye,
                                         const double* Q, int ld, double sigma, double rho, double alpha, double* Zh,
                                         double* V, double* zeh, const double* b, const double* w, void* stream) {
  if (n <= 0 || ld < n || !X || !Zp || !Yp || !ye || !Q || !Zh || !V || !zeh || !(rho > 0.0) || !(sigma >= 0.0) ||
      !(alpha > 0.0 && alpha < 2.0))
    return set_err(PSDPROJ_E_INVALID, "invalid admm step1 arguments");
  admm_maxcut_step1_kernel<<<grid1d((size_t)n * n), 256, 0, (cudaStream_t)stream>>>(n, X, Zp, Yp, ye, Q, sigma, rho,
                                                                                     alpha, Zh, V, zeh, ld, b, w);
  CKL();
  return 0;
}

extern "C" int psdproj_admm_certificate_terms(int n, const double* X, const double* X0, const double* ye,
                                              const double* ye0, const double* Yp, const double* Yp0, const double* Q,
                                              int ld, const double* b, const double* w, double* dY_sym,
                                              double* mdX_sym, double* work, size_t work_elems, double* terms_host,
                                              void* stream) {
  if (n <= 0 || ld < n || !X || !X0 || !ye || !ye0 || !Yp || !Yp0 || !Q || !dY_sym || !mdX_sym || !work ||
      !terms_host)
    return set_err(PSDPROJ_E_INVALID, "invalid certificate arguments");
  cudaStream_t st = (cudaStream_t)stream;
  int nb = std::min(sms() * 2, std::max(1, (int)(((size_t)n * n + 255) / 256)));
  if (work_elems < (size_t)CERT_TERMS * (nb + 1)) nb = (int)(work_elems / CERT_TERMS) - 1;
  if (nb < 1) return set_err(PSDPROJ_E_WORKSPACE, "certificate work buffer too small");
  admm_cert_partial_kernel<<<nb, 256, 0, st>>>(n, X, X0, ye, ye0, Yp, Yp0, Q, ld, b, w, dY_sym, mdX_sym, work);
  CKL();
  admm_cert_final_kernel<<<1, 32, 0, st>>>(nb, work, work + (size_t)CERT_TERMS * nb);
  CKL();
  CK(cudaMemcpyAsync(terms_host, work + (size_t)CERT_TERMS * nb, CERT_TERMS * sizeof(double), cudaMemcpyDeviceToHost,
                     st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

extern "C" int psdproj_admm_maxcut_step2(int n, const double* X, const double* Zp, const double* Zh, double* Yp,
                                         double* ye, const double* zeh, const double* Q, int ld, double rho,
                                         double* res_host, const double* b, const double* w, void* stream) {
  if (n <= 0 || ld < n || !X || !Zp || !Zh || !Yp || !ye || !zeh || !Q || !res_host || !(rho > 0.0))
    return set_err(PSDPROJ_E_INVALID, "invalid admm step2 arguments");
  cudaStream_t st = (cudaStream_t)stream;
  static thread_local unsigned long long* dres = nullptr;
  if (!dres) CK(cudaMalloc(&dres, 4 * sizeof(unsigned long long)));
  CK(cudaMemsetAsync(dres, 0, 3 * sizeof(unsigned long long), st));
  admm_maxcut_step2_kernel<<<grid1d((size_t)n * n), 256, 0, st>>>(n, X, Zp, Zh, Yp, ye, zeh, Q, rho, ld, dres, b, w);
  CKL();
  CK(cudaMemcpyAsync(res_host, dres, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}
