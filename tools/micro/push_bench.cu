// Microbenchmark: push-style DSMEM communication inside a 16-CTA cluster on B200 (sm_100a):
// st.async / cp.async.bulk (shared::cta -> shared::cluster) completing on the receiver's mbarrier,
// against the barrier.cluster + remote-load (pull) pattern. Cycles per broadcast / all-gather hop.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ unsigned crank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void bulk_s2c(uint32_t rdst, const void* src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
               "r"(smem_u32(src)), "r"(bytes), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// NB doubles broadcast / all-gathered per hop
__global__ void k_push(int iters, int mode, int NB, double* out) {
  __shared__ __align__(16) double src[2][512];
  __shared__ __align__(16) double dst[2][2048];
  __shared__ __align__(8) uint64_t bar[2];
  const unsigned r = crank(), cs = gridDim.x;
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int i = tid; i < 2 * 512; i += NT) (&src[0][0])[i] = r + i;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  csync();
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int par = it & 1;
    const uint32_t ph = (it >> 1) & 1;
    const unsigned prod = it % cs;
    if (mode <= 3) {
      // broadcast of NB doubles from CTA prod to all CTAs (incl. itself)
      const uint32_t bytes = (mode == 0) ? 8u : (uint32_t)NB * 8u;
      if (tid == 0) mbar_expect(&bar[par], bytes);
      if (r == prod) {
        if (mode == 0) {
          if (tid < (int)cs) st_async(mapa(smem_u32(&dst[par][0]), tid), acc + it, mapa(smem_u32(&bar[par]), tid));
        } else if (mode == 1) {  // one bulk copy per destination, lanes 0..cs-1 of warp 0
          src[par][tid & 511] += acc;  // generic writes to the source
          __syncthreads();
          if (tid < (int)cs) {
            fence_async_smem();
            bulk_s2c(mapa(smem_u32(&dst[par][0]), tid), &src[par][0], bytes, mapa(smem_u32(&bar[par]), tid));
          }
        } else if (mode == 2) {  // st.async v2 from all threads of the producer
          for (int q = tid; q < (int)cs * NB / 2; q += NT) {
            const int d = q / (NB / 2), e = 2 * (q - d * (NB / 2));
            st_async2(mapa(smem_u32(&dst[par][e]), d), src[par][e] + acc, src[par][e + 1],
                      mapa(smem_u32(&bar[par]), d));
          }
        } else {  // mode 3: producer warp 0 only, one bulk copy per destination, no CTA barrier
          if (tid < 32) {
            src[par][tid] += acc;
            __syncwarp();
            if (tid < (int)cs) {
              fence_async_smem();
              bulk_s2c(mapa(smem_u32(&dst[par][0]), tid), &src[par][0], bytes, mapa(smem_u32(&bar[par]), tid));
            }
          }
        }
      }
      mbar_wait(&bar[par], ph);
      acc += dst[par][tid % NB];
    } else if (mode == 4 || mode == 5) {
      // all-gather: every CTA sends NB doubles to every CTA (slot r); expect cs * NB * 8 bytes
      const uint32_t bytes = (uint32_t)NB * 8u;
      if (tid == 0) mbar_expect(&bar[par], bytes * cs);
      if (mode == 4) {
        src[par][tid & 511] += acc;
        __syncthreads();
        if (tid < (int)cs) {
          fence_async_smem();
          bulk_s2c(mapa(smem_u32(&dst[par][r * NB]), tid), &src[par][0], bytes, mapa(smem_u32(&bar[par]), tid));
        }
      } else {
        for (int q = tid; q < (int)cs * NB; q += NT) {
          const int d = q / NB, e = q - d * NB;
          st_async(mapa(smem_u32(&dst[par][r * NB + e]), d), src[par][e] + acc, mapa(smem_u32(&bar[par]), d));
        }
      }
      mbar_wait(&bar[par], ph);
      acc += dst[par][tid % (NB * cs)];
    } else if (mode == 6) {
      // pull reference: barrier.cluster, then every thread loads NB doubles from the producer
      if (r == prod) src[par][tid % NB] += acc;
      csync();
      {
        // generic DSMEM load through the mapped pointer
        double* p;
        asm volatile("mapa.u64 %0, %1, %2;" : "=l"(p) : "l"(&src[par][0]), "r"(prod));
        for (int q = tid; q < NB; q += NT) dst[par][q] = p[q];
      }
      __syncthreads();
      acc += dst[par][tid % NB];
    } else if (mode == 7) {
      // pull all-gather reference: barrier.cluster, every thread loads its share of cs * NB doubles
      src[par][tid % NB] += acc;
      csync();
      for (int q = tid; q < (int)cs * NB; q += NT) {
        const int d = q / NB, e = q - d * NB;
        double* p;
        asm volatile("mapa.u64 %0, %1, %2;" : "=l"(p) : "l"(&src[par][e]), "r"(d));
        dst[par][q] = *p;
      }
      __syncthreads();
      acc += dst[par][tid % (NB * cs)];
    }
  }
  long long t1 = clock64();
  csync();
  if (tid == 0 && r == 0) out[0] = (double)(t1 - t0) / iters;
  if (acc == 12345.0) out[1] = acc;
}

int main() {
  double* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k_push, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"bcast st.async 1 dbl", "bcast bulk (CTA bar)", "bcast st.async.v2 all thr", "bcast bulk (warp 0)",
                         "allgather bulk", "allgather st.async", "pull bcast (cluster bar)", "pull allgather (cluster bar)"};
  for (int mode = 0; mode < 8; ++mode)
    for (int nb : {32, 128, 512})
      for (int nt : {256, 512}) {
        if ((mode == 0) && nb != 32) continue;
        if ((mode == 4 || mode == 5 || mode == 7) && nb > 128) continue;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(nt);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_push, 2000, mode, nb, d);
        cudaError_t e = cudaDeviceSynchronize();
        double h[2] = {0, 0};
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%-30s nb=%4d nt=%4d: %8.1f cycles/hop %s\n", names[mode], nb, nt, h[0], e ? cudaGetErrorString(e) : "");
        if (e) return 1;
      }
  return 0;
}
