// DFMA latency / ILP microbenchmark: TF/s for C independent FMA chains per thread with W warps
// per SM (one CTA of 32*W threads per SM, 148 CTAs), plus the dependent-chain latency in cycles,
// MUFU.RSQ64H/RCP64H-seeded Newton latency, and shared-memory 64-bit CAS throughput.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k_ilp(double* out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int i = 0; i < C; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}

__global__ void k_cas(double* out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned long long* p = reinterpret_cast<unsigned long long*>(s + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    unsigned long long o = *p;
    atomicCAS(p, o, __double_as_longlong(__longlong_as_double(o) + 1.0));
  }
  __syncthreads();
  if (s[threadIdx.x] == -1.0) out[0] = 1;
}

template <int C>
void run(double* d, int W) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  k_ilp<C><<<148, 32 * W>>>(d, 10, 0.999999, 1e-7);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    k_ilp<C><<<148, 32 * W>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("{\"chains\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", C, W,
         2.0 * C * iters * 148.0 * 32 * W / (best * 1e-3) / 1e12);
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8);
  for (int W : {4, 8, 12, 16, 32}) {
    run<1>(d, W);
    run<2>(d, W);
    run<4>(d, W);
    run<8>(d, W);
  }
  k_lat<<<1, 32>>>(d, c, 10000, 0.999999, 1e-7);
  long long cyc;
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"dfma_dependent_latency_cycles\": %.2f}\n", cyc / 10000.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int W : {8, 16, 32}) {
    k_cas<<<148, 32 * W>>>(d, 10);
    cudaEventRecord(e0);
    k_cas<<<148, 32 * W>>>(d, 2000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"smem_cas64_per_sm_per_clk\": %.3f, \"warps_per_sm\": %d}\n",
           2000.0 * 32 * W / (ms * 1e-3 * 1.965e9), W);
  }
  return 0;
}
