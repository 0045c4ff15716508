// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) and DFMA peak on this GPU.
// Used once to fix the FP64 roofline denominator (bench/peaks_fp64.json).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  double a = 1.0000001, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int wpb : {4, 8, 16, 32}) {
      int blocks = sms * 2, iters = 20000;
      dmma_loop<<<blocks, wpb * 32>>>(d, 100);
      cudaEventRecord(e0);
      dmma_loop<<<blocks, wpb * 32>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * wpb;
      printf("DMMA m8n8k4 warps/blk=%d: %.2f TFLOP/s (%.3f ms)\n", wpb, flops / ms / 1e9, ms);
      dfma_loop<<<blocks, wpb * 32>>>(d, 100);
      cudaEventRecord(e0);
      dfma_loop<<<blocks, wpb * 32>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8.0 * iters * (double)blocks * wpb * 32;
      printf("DFMA warps/blk=%d: %.2f TFLOP/s (%.3f ms)\n", wpb, flops / ms / 1e9, ms);
    }
  }
  printf("SMs=%d\n", sms);
  return 0;
}
