// Microbenchmark: fp64 DFMA pipe vs fp64 tensor (mma.sync m8n8k4 f64 -> DMMA) vs both interleaved.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
  double acc[4][2];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE & 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    if (MODE & 2) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(acc[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[0] = s;
}

template <int MODE>
double run(double* d, int blocks) {
  const int threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fma_flops = (MODE & 1) ? 2.0 * 8 * iters * (double)blocks * threads : 0;
  // m8n8k4: 8*8*4 MACs per warp-instruction = 256 MAC = 512 flop per warp
  double mma_flops = (MODE & 2) ? 512.0 * 4 * iters * (double)blocks * (threads / 32) : 0;
  printf("{\"mode\": %d, \"ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"total_tflops\": %.2f}\n", MODE, ms,
         fma_flops / (ms * 1e-3) / 1e12, mma_flops / (ms * 1e-3) / 1e12, (fma_flops + mma_flops) / (ms * 1e-3) / 1e12);
  return ms;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  run<1>(d, sm * 8);
  run<2>(d, sm * 8);
  run<3>(d, sm * 8);
  return 0;
}
