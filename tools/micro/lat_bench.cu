// Microbenchmark: dependent-chain latency of DFMA, SHFL.BFLY(f64) and LDS.64 on B200 (sm_100a).
#include <cstdio>
__global__ void k(int iters, double* out, int mode) {
  __shared__ double sm[1024];
  sm[threadIdx.x] = threadIdx.x * 1e-3;
  __syncthreads();
  double a = threadIdx.x * 1e-3 + 1.0, b = 0.999999, c = 1e-9;
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
    else if (mode == 1) { a += __shfl_xor_sync(0xffffffffu, a, 1); a += __shfl_xor_sync(0xffffffffu, a, 2); a += __shfl_xor_sync(0xffffffffu, a, 4); a += __shfl_xor_sync(0xffffffffu, a, 8); }
    else { a = sm[(idx + (int)a) & 1023]; a = sm[((int)a + 1) & 1023]; a = sm[((int)a + 2) & 1023]; a = sm[((int)a + 3) & 1023]; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[mode] = (double)(t1 - t0) / (4.0 * iters);
  if (a == 12345.0) out[3] = a;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  const char* nm[] = {"DFMA dependent", "SHFL+DADD dependent", "LDS dependent"};
  for (int m = 0; m < 3; ++m) {
    k<<<1, 32>>>(10000, d, m);
    double h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("%-22s %.1f cycles\n", nm[m], h[m]);
  }
  return 0;
}
