// Device helpers shared by several kernel files (interface-group sums, per-node BC projection).
#pragma once
#include <cstdio>

#include "hhg_internal.h"

namespace hhg {

// Bounds checks of our own (compute-sanitizer is closed on this pool): built with -DHHG_CHECKED, every
// global index of the element kernels, interface sums and transfers is checked against its vector length
// and a violation prints the kernel, index and bound and traps.  Compiled out otherwise.
#ifdef HHG_CHECKED
#define HHG_CHECK(cond, what, idx, bound)                                                                    \
  do {                                                                                                      \
    if (!(cond)) {                                                                                          \
      printf("HHG_CHECKED: %s out of range: %lld (bound %lld) block (%d,%d) thread %d\n", what,            \
             (long long)(idx), (long long)(bound), (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);     \
      __trap();                                                                                             \
    }                                                                                                       \
  } while (0)
#else
#define HHG_CHECK(cond, what, idx, bound) \
  do {                                    \
  } while (0)
#endif

// Sum of the copies of group gi (copies gathered in chunks of 4 independent loads: macro vertices
// have up to ~20 copies and a sequential dependent walk made coarse levels latency-bound).
template <int NC>
__device__ __forceinline__ void group_sum(int64_t b, int64_t e, const int64_t* __restrict__ copy, int64_t cstride,
                                          const double* __restrict__ v, double (&val)[NC]) {
  constexpr int CH = 4;
#pragma unroll
  for (int c = 0; c < NC; ++c) val[c] = 0.0;
  for (int64_t k0 = b; k0 < e; k0 += CH) {
    int64_t idx[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) idx[j] = (k0 + j < e) ? copy[k0 + j] : -1;
#pragma unroll
    for (int j = 0; j < CH; ++j) HHG_CHECK(idx[j] < cstride || NC == 1, "group copy", idx[j], cstride);
    double x[CH][NC];
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int c = 0; c < NC; ++c) x[j][c] = idx[j] >= 0 ? v[c * cstride + idx[j]] : 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (idx[j] >= 0) val[c] += x[j][c];
  }
}
template <int NC>
__device__ __forceinline__ void group_store(int64_t b, int64_t e, const int64_t* __restrict__ copy, int64_t cstride,
                                            const double (&val)[NC], double* __restrict__ v) {
  constexpr int CH = 4;
  for (int64_t k0 = b; k0 < e; k0 += CH) {
    int64_t idx[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) idx[j] = (k0 + j < e) ? copy[k0 + j] : -1;
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (idx[j] >= 0)
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c * cstride + idx[j]] = val[c];
  }
}
template <int NC>
__device__ __forceinline__ void group_bc(int kd, const double* __restrict__ nrm, double (&val)[NC]) {
  if (kd == HHG_BC_DIRICHLET0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) val[c] = 0.0;
  } else if (kd == HHG_BC_FREESLIP && NC == 3) {
    const double n0 = nrm[0], n1 = nrm[1], n2 = nrm[2];
    const double un = val[0] * n0 + val[1 % NC] * n1 + val[2 % NC] * n2;
    val[0] -= un * n0;
    val[1 % NC] -= un * n1;
    val[2 % NC] -= un * n2;
  }
}

__device__ __forceinline__ void bc_project(int b, const double* __restrict__ nrm, double& v0, double& v1, double& v2) {
  if (b == -1) return;
  if (b == -2) {
    v0 = v1 = v2 = 0.0;
    return;
  }
  const double n0 = nrm[3 * b], n1 = nrm[3 * b + 1], n2 = nrm[3 * b + 2];
  const double un = v0 * n0 + v1 * n1 + v2 * n2;
  v0 -= un * n0;
  v1 -= un * n1;
  v2 -= un * n2;
}

}  // namespace hhg
