// DFMA throughput microbenchmark for the fp64 roofline denominator (B200 has no fp64 entry in
// MEASURED_PEAKS.json).  8 independent FMA chains per thread, 148*8 blocks x 256 threads.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 5;
  double* d;
  cudaMalloc(&d, 8);
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sm * 8, threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
  double best = 0;
  std::vector<double> all;
  for (int rep = 0; rep < reps; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double tf = 2.0 * 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
    all.push_back(tf);
  }
  std::sort(all.begin(), all.end());
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dfma_tflops_median\": %.3f, \"reps\": %d, \"sms\": %d}\n", best,
         all[all.size() / 2], reps, sm);
  return 0;
}
