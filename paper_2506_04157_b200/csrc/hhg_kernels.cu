// sm_100a kernels of the hot path (fp64 DFMA; the operator is not a dense contraction).
//
//  k_elem      element loop over micro tets of the structured macro lattices: gathers the 30
//              velocity dofs (+4 eta, +4 p), evaluates the blending Jacobian at the 4 quadrature
//              points on the fly, and accumulates A u, B^T p, (B+C) u
//               or diag(A).
//  k_fixup     sums replicated interface copies (HHG interface communication analogue) and
//              applies the Dirichlet mask / free-slip projection P_v.
//  k_prolong / k_restrict   P2 nodal interpolation between nested lattices and its transpose.
//  k_dot*      deterministic two-pass reductions over unique dofs.
#include <cstdio>

#include "hhg_internal.h"
#include "hhg_device.cuh"

namespace hhg {

// Q4 rule (R6): barycentric (a,b,b,b) and permutations, weights 1/24.
constexpr double QA = 0.58541019662496845446;  // (5 + 3 sqrt 5)/20
constexpr double QB = 0.13819660112501051518;  // (5 - sqrt 5)/20

// ------------------------------------------------------------------ interface sum + BC
template <int NC, bool BC>
__global__ void k_fixup(int64_t ng, const int64_t* __restrict__ ptr, const int64_t* __restrict__ copy,
                        const uint8_t* __restrict__ kind, const double* __restrict__ normal, int64_t cstride,
                        bool sum, double* __restrict__ v) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= ng) return;
  const int64_t b = ptr[gi], e = ptr[gi + 1];
  double val[NC];
  if (sum) {
    group_sum<NC>(b, e, copy, cstride, v, val);
  } else {
    const int64_t i0 = copy[b];
#pragma unroll
    for (int c = 0; c < NC; ++c) val[c] = v[c * cstride + i0];
  }
  if (BC) group_bc<NC>(kind[gi], normal + 3 * gi, val);
  if (!sum && !BC) return;
  group_store<NC>(b, e, copy, cstride, val, v);
}

// local partial sums of the groups shared with other ranks -> send buffer [slot][NC]
template <int NC>
__global__ void k_halo_pack(int64_t nslots, const int64_t* __restrict__ slot_group, const int64_t* __restrict__ ptr,
                            const int64_t* __restrict__ copy, int64_t cstride, const double* __restrict__ v,
                            double* __restrict__ sbuf) {
  const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= nslots) return;
  const int64_t g = slot_group[sl], b = ptr[g], e = ptr[g + 1];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double s = 0.0;
    for (int64_t k = b; k < e; ++k) {
      HHG_CHECK(NC == 1 || copy[k] < cstride, "halo pack copy", copy[k], cstride);
      s += v[c * cstride + copy[k]];
    }
    sbuf[sl * NC + c] = s;
  }
}

// interface sum including the partial sums received from other ranks, then BC, scattered to copies
template <int NC, bool BC>
__global__ void k_fixup_remote(int64_t ng, const int64_t* __restrict__ ptr, const int64_t* __restrict__ copy,
                               const uint8_t* __restrict__ kind, const double* __restrict__ normal, int64_t cstride,
                               const int64_t* __restrict__ gs_ptr, const int64_t* __restrict__ gs_idx,
                               const double* __restrict__ rbuf, double* __restrict__ v) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= ng) return;
  const int64_t b = ptr[gi], e = ptr[gi + 1];
  double val[NC];
  group_sum<NC>(b, e, copy, cstride, v, val);
  for (int64_t k = gs_ptr[gi]; k < gs_ptr[gi + 1]; ++k)
#pragma unroll
    for (int c = 0; c < NC; ++c) val[c] += rbuf[gs_idx[k] * NC + c];
  if (BC) group_bc<NC>(kind[gi], normal + 3 * gi, val);
  group_store<NC>(b, e, copy, cstride, val, v);
}

static const Groups& groups_of(const Level& L, int space) { return space == HHG_P1 ? L.g1 : L.g2; }

int launch_halo_pack(const Mesh* m, const Level& L, int space, const double* v, double* sbuf, cudaStream_t s) {
  const Groups& G = groups_of(L, space);
  const Halo& H = G.halo;
  if (H.nslots == 0) return HHG_OK;
  const int64_t nm = macro_count(m);
  const unsigned nb = (unsigned)((H.nslots + 255) / 256);
  if (space == HHG_P2VEC)
    k_halo_pack<3><<<nb, 256, 0, s>>>(H.nslots, H.slot_group, G.ptr, G.copy, nm * L.npts2, v, sbuf);
  else
    k_halo_pack<1><<<nb, 256, 0, s>>>(H.nslots, H.slot_group, G.ptr, G.copy, 0, v, sbuf);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

int launch_fixup_remote(const Mesh* m, const Level& L, int space, bool bc, const double* rbuf, double* v,
                        cudaStream_t s) {
  const Groups& G = groups_of(L, space);
  const Halo& H = G.halo;
  if (G.n == 0) return HHG_OK;
  const int64_t nm = macro_count(m);
  const unsigned nb = (unsigned)((G.n + 255) / 256);
  if (space == HHG_P2VEC) {
    if (bc)
      k_fixup_remote<3, true><<<nb, 256, 0, s>>>(G.n, G.ptr, G.copy, G.kind, G.normal, nm * L.npts2, H.gs_ptr,
                                                 H.gs_idx, rbuf, v);
    else
      k_fixup_remote<3, false><<<nb, 256, 0, s>>>(G.n, G.ptr, G.copy, G.kind, G.normal, nm * L.npts2, H.gs_ptr,
                                                  H.gs_idx, rbuf, v);
  } else {
    k_fixup_remote<1, false><<<nb, 256, 0, s>>>(G.n, G.ptr, G.copy, nullptr, nullptr, 0, H.gs_ptr, H.gs_idx, rbuf, v);
  }
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

int launch_fixup(const Mesh* m, const Level& L, int space, bool sum, bool bc, double* v, cudaStream_t s) {
  // multi-rank interface sum: pack shared partial sums, NCCL exchange, local + remote sum (+BC)
  if (sum && m->comm && m->nranks > 1 && groups_of(L, space).halo.nslots > 0) {
    const Halo& H = groups_of(L, space).halo;
    const int nc = space == HHG_P2VEC ? 3 : 1;
    HHG_TRY(launch_halo_pack(m, L, space, v, H.sbuf, s));
    HHG_TRY(comm_exchange(m->comm, H, nc, H.sbuf, H.rbuf, s));
    return launch_fixup_remote(m, L, space, bc && space == HHG_P2VEC, H.rbuf, v, s);
  }
  const int64_t nm = macro_count(m);
  if (space == HHG_P2VEC) {
    // BC-only passes visit just the groups carrying a BC (they are sorted first)
    const int64_t ng = sum ? L.g2.n : (bc ? L.g2.nbc : 0);
    if (ng == 0) return HHG_OK;
    const unsigned nb = (unsigned)((ng + 255) / 256);
    if (bc)
      k_fixup<3, true><<<nb, 256, 0, s>>>(ng, L.g2.ptr, L.g2.copy, L.g2.kind, L.g2.normal, nm * L.npts2, sum, v);
    else
      k_fixup<3, false><<<nb, 256, 0, s>>>(ng, L.g2.ptr, L.g2.copy, L.g2.kind, L.g2.normal, nm * L.npts2, sum, v);
  } else if (space == HHG_P2) {
    if (L.g2.n == 0) return HHG_OK;
    const unsigned nb = (unsigned)((L.g2.n + 255) / 256);
    k_fixup<1, false><<<nb, 256, 0, s>>>(L.g2.n, L.g2.ptr, L.g2.copy, nullptr, nullptr, 0, sum, v);
  } else {
    if (L.g1.n == 0) return HHG_OK;
    const unsigned nb = (unsigned)((L.g1.n + 255) / 256);
    k_fixup<1, false><<<nb, 256, 0, s>>>(L.g1.n, L.g1.ptr, L.g1.copy, nullptr, nullptr, 0, sum, v);
  }
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// ------------------------------------------------------------------ dot products
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k_dot_partial(int64_t nstored, int nc, int64_t cstride, const uint8_t* __restrict__ own,
                              const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nstored; i += (int64_t)gridDim.x * blockDim.x) {
    if (!own[i]) continue;
    for (int c = 0; c < nc; ++c) s += x[c * cstride + i] * y[c * cstride + i];
  }
  __shared__ double sh[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

__global__ void k_dot_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out = v;
  }
}

// one-launch dot: block partials + last-block (fixed-order) finalisation; partials and counter live in
// the caller's reduction scratch `red` (one per solver object, so dots of different objects never share
// it; the counter is reset by the last block, so graph replays stay valid)
__global__ void k_dot_fused(int64_t nstored, int nc, int64_t cstride, const uint8_t* __restrict__ own,
                            const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ part,
                            unsigned* __restrict__ counter, double* __restrict__ out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nstored; i += (int64_t)gridDim.x * blockDim.x) {
    if (!own[i]) continue;
    for (int c = 0; c < nc; ++c) s += x[c * cstride + i] * y[c * cstride + i];
  }
  __shared__ double sh[32];
  __shared__ bool last;
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      part[blockIdx.x] = v;
      __threadfence();
      last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += ((volatile double*)part)[i];
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      *out = v;
      *counter = 0u;
    }
  }
}

int launch_dot_fused(const Mesh* m, const Level& L, int space, const double* x, const double* y, double* out,
                     cudaStream_t s, double* red) {
  const int64_t nm = macro_count(m);
  const bool p1 = space == HHG_P1;
  const int64_t nst = nm * (p1 ? L.npts1 : L.npts2);
  const int nc = space == HHG_P2VEC ? 3 : 1;
  int64_t nb = (nst + 255) / 256;
  nb = nb < 1 ? 1 : (nb > kRedBlocks ? kRedBlocks : nb);
  k_dot_fused<<<(unsigned)nb, 256, 0, s>>>(nst, nc, nst, p1 ? L.own1 : L.own2, x, y, red,
                                          reinterpret_cast<unsigned*>(red + kRedBlocks + 4), out);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  if (m->comm && m->nranks > 1) HHG_TRY(comm_allreduce_sum(m->comm, out, 1, s));
  return HHG_OK;
}

int red_alloc(double** red) {
  if (cudaMalloc(red, kRedScratch * sizeof(double)) != cudaSuccess) return fail(HHG_ENOMEM, "reduction scratch");
  HHG_CUDA(cudaMemset(*red, 0, kRedScratch * sizeof(double)));
  return HHG_OK;
}

int launch_dot(const Mesh* m, const Level& L, int space, const double* x, const double* y, double* out,
               cudaStream_t s, double* red) {
  const int64_t nm = macro_count(m);
  const bool p1 = space == HHG_P1;
  const int64_t nst = nm * (p1 ? L.npts1 : L.npts2);
  const int nc = space == HHG_P2VEC ? 3 : 1;
  k_dot_partial<<<kRedBlocks, 256, 0, s>>>(nst, nc, nst, p1 ? L.own1 : L.own2, x, y, red);
  k_dot_final<<<1, 256, 0, s>>>(red, kRedBlocks, out);
  count_launch(2);
  HHG_CUDA(cudaGetLastError());
  if (m->comm && m->nranks > 1) HHG_TRY(comm_allreduce_sum(m->comm, out, 1, s));
  return HHG_OK;
}

// ------------------------------------------------------------------ lattice walkers
// warp per (j,k) row of a lattice of resolution N; grid.y = macro
struct RowCtx {
  int i0, j, k, len;
};

__device__ __forceinline__ bool row_of(const int32_t* rows, int64_t nrows, int N, RowCtx& rc) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nrows) return false;
  const int32_t pk = rows[r];
  rc.j = pk & 0xffff;
  rc.k = pk >> 16;
  rc.len = N - rc.j - rc.k + 1;
  return true;
}

// ------------------------------------------------------------------ P2 transfers (stencil tables)
// Prolongation = nodal interpolation of the coarse P2 function at the fine P2 nodes (DESIGN.md
// R14); restriction = its transpose.  Both are gathers driven by host-built tables:
//  * prolong: fine node F (fine P2 lattice index) lies in coarse cube F>>2 at offset o = F&3; the
//    64 offset classes carry <= 10 (coarse node offset dC in [0,2]^3 from 2(F>>2), weight) pairs
//    of the coarse tet containing the point (weights lambda(2 lambda - 1), 4 lambda_p lambda_q);
//  * restrict: coarse node C gathers sum_F w(F,C) own(F) r(F) over the transposed stencil of its
//    parity class (8 classes: coarse vertex or one of the 7 lattice edge directions), clipped to
//    the macro's lattice.  No atomics; each output written once.
constexpr int kPMax = 10, kRMax = 128;
__device__ int gPn[64];
__device__ int gPd[64][kPMax];        // dx + 3 dy + 9 dz
__device__ double gPw[64][kPMax];
__device__ int gRn[8];
__device__ int gRd[8][kRMax];         // (dx+8) | (dy+8) << 5 | (dz+8) << 10
__device__ double gRw[8][kRMax];

static bool g_tabs_ready = false;
static int ensure_transfer_tabs() {
  if (g_tabs_ready) return HHG_OK;
  const int TV[6][4][3] = {
      {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}}};
  const int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  static int pn[64], pd[64][kPMax];
  static double pw[64][kPMax];
  for (int cls = 0; cls < 64; ++cls) {
    const int o[3] = {cls & 3, (cls >> 2) & 3, cls >> 4};
    pn[cls] = 0;
    if (((o[0] | o[1] | o[2]) & 1) == 0) {
      pd[cls][0] = o[0] / 2 + 3 * (o[1] / 2) + 9 * (o[2] / 2);
      pw[cls][0] = 1.0;
      pn[cls] = 1;
      continue;
    }
    // coarse tet of the cube containing the point o/4 (Freudenthal split, sorted-coordinate rule)
    const int S = o[0] + o[1] + o[2];
    int t;
    if (S <= 4) t = 0;
    else if (S > 8) t = 5;
    else {
      const bool xy = o[0] + o[1] >= 4, yz = o[1] + o[2] >= 4;
      t = xy ? (yz ? 3 : 1) : (yz ? 4 : 2);
    }
    // barycentric coordinates (exact multiples of 1/4): o = 4 V0 + sum_v b_v (V_v - V0)
    double E[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) E[3 * r + c] = TV[t][c + 1][r] - TV[t][0][r];
    const double det = E[0] * (E[4] * E[8] - E[5] * E[7]) - E[1] * (E[3] * E[8] - E[5] * E[6]) +
                       E[2] * (E[3] * E[7] - E[4] * E[6]);
    const double adj[9] = {E[4] * E[8] - E[5] * E[7], E[2] * E[7] - E[1] * E[8], E[1] * E[5] - E[2] * E[4],
                           E[5] * E[6] - E[3] * E[8], E[0] * E[8] - E[2] * E[6], E[2] * E[3] - E[0] * E[5],
                           E[3] * E[7] - E[4] * E[6], E[1] * E[6] - E[0] * E[7], E[0] * E[4] - E[1] * E[3]};
    const double q[3] = {o[0] - 4.0 * TV[t][0][0], o[1] - 4.0 * TV[t][0][1], o[2] - 4.0 * TV[t][0][2]};
    double lam[4];
    for (int r = 0; r < 3; ++r) lam[r + 1] = 0.25 * (adj[3 * r] * q[0] + adj[3 * r + 1] * q[1] + adj[3 * r + 2] * q[2]) / det;
    lam[0] = 1.0 - lam[1] - lam[2] - lam[3];
    for (int v = 0; v < 4; ++v) {
      const double w = lam[v] * (2.0 * lam[v] - 1.0);
      if (w != 0.0) {
        pd[cls][pn[cls]] = 2 * TV[t][v][0] + 3 * 2 * TV[t][v][1] + 9 * 2 * TV[t][v][2];
        pw[cls][pn[cls]++] = w;
      }
    }
    for (int e = 0; e < 6; ++e) {
      const int p = ep[e][0], r = ep[e][1];
      const double w = 4.0 * lam[p] * lam[r];
      if (w != 0.0) {
        pd[cls][pn[cls]] = (TV[t][p][0] + TV[t][r][0]) + 3 * (TV[t][p][1] + TV[t][r][1]) + 9 * (TV[t][p][2] + TV[t][r][2]);
        pw[cls][pn[cls]++] = w;
      }
    }
  }
  // transpose: representative coarse node C = 8 + parity per dimension; scan fine nodes around 2C
  static int rn[8], rd[8][kRMax];
  static double rw[8][kRMax];
  for (int pc = 0; pc < 8; ++pc) {
    const int C[3] = {8 + (pc & 1), 8 + ((pc >> 1) & 1), 8 + (pc >> 2)};
    rn[pc] = 0;
    for (int dz = -8; dz <= 8; ++dz)
      for (int dy = -8; dy <= 8; ++dy)
        for (int dx = -8; dx <= 8; ++dx) {
          const int F[3] = {2 * C[0] + dx, 2 * C[1] + dy, 2 * C[2] + dz};
          const int cls = (F[0] & 3) + 4 * (F[1] & 3) + 16 * (F[2] & 3);
          for (int e = 0; e < pn[cls]; ++e) {
            const int d = pd[cls][e];
            const int Cn[3] = {2 * (F[0] >> 2) + d % 3, 2 * (F[1] >> 2) + (d / 3) % 3, 2 * (F[2] >> 2) + d / 9};
            if (Cn[0] == C[0] && Cn[1] == C[1] && Cn[2] == C[2]) {
              if (rn[pc] >= kRMax) return fail(HHG_EINVAL, "restriction stencil table overflow");
              rd[pc][rn[pc]] = (dx + 8) | ((dy + 8) << 5) | ((dz + 8) << 10);
              rw[pc][rn[pc]++] = pw[cls][e];
            }
          }
        }
  }
  HHG_CUDA(cudaMemcpyToSymbol(gPn, pn, sizeof(pn)));
  HHG_CUDA(cudaMemcpyToSymbol(gPd, pd, sizeof(pd)));
  HHG_CUDA(cudaMemcpyToSymbol(gPw, pw, sizeof(pw)));
  HHG_CUDA(cudaMemcpyToSymbol(gRn, rn, sizeof(rn)));
  HHG_CUDA(cudaMemcpyToSymbol(gRd, rd, sizeof(rd)));
  HHG_CUDA(cudaMemcpyToSymbol(gRw, rw, sizeof(rw)));
  g_tabs_ready = true;
  return HHG_OK;
}

__device__ __forceinline__ int rowstart_i32(int N, int j, int k) {
  const int M = N - k;
  return ((N + 1) * (N + 2) * (N + 3) - (M + 1) * (M + 2) * (M + 3)) / 6 + (j * (2 * M + 3 - j)) / 2;
}

// x_f += P x_c on every stored fine node (per macro; consistent copies stay consistent).
// Warp per fine row (J,K): the 9 coarse rows a stencil can touch are the same for the whole row,
// so their starts are computed once per warp (shared memory); tables read through L1.
__global__ void k_prolong(const int32_t* __restrict__ rowsf, int64_t nrowsf, int Nf, int64_t nptsf, int64_t nptsc,
                          int64_t cstridef, int64_t cstridec, const double* __restrict__ xc, double* __restrict__ xf) {
  __shared__ int srs[8][9];
  RowCtx rc;
  if (!row_of(rowsf, nrowsf, Nf, rc)) return;
  const int mac = blockIdx.y;
  const int Nc = Nf / 2;
  const int J = rc.j, K = rc.k, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int by = 2 * (J >> 2), bz = 2 * (K >> 2);
  if (lane < 9) srs[w][lane] = rowstart_i32(Nc, by + lane % 3, bz + lane / 3);
  __syncwarp();
  double* fr = xf + (int64_t)mac * nptsf + rowstart_i32(Nf, J, K);
  const double* cm = xc + (int64_t)mac * nptsc;
  const int cls0 = 4 * (J & 3) + 16 * (K & 3);
  // 4 passes over I mod 4 so that all lanes of a pass share one stencil class (no divergence)
  for (int it = lane; it < 4 * ((rc.len + 3) / 4); it += 32) {
    const int o = it / ((rc.len + 3) / 4), I = 4 * (it % ((rc.len + 3) / 4)) + o;
    if (I >= rc.len) continue;
    const int cls = o + cls0;
    const int bx = 2 * (I >> 2);
    const int n = __ldg(gPn + cls);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int e = 0; e < kPMax; ++e) {  // fully unrolled, predicated: all gathers in flight at once
      if (e < n) {
        const int d = __ldg(&gPd[cls][e]);
        const int ci = srs[w][d / 3] + bx + d % 3;
        HHG_CHECK(ci >= 0 && ci < nptsc, "prolong gather", ci, nptsc);
        const double wt = __ldg(&gPw[cls][e]);
        s0 += wt * __ldg(cm + ci);
        s1 += wt * __ldg(cm + cstridec + ci);
        s2 += wt * __ldg(cm + 2 * cstridec + ci);
      }
    }
    fr[I] += s0;
    fr[cstridef + I] += s1;
    fr[2 * cstridef + I] += s2;
  }
}

// r_c = P^T r_f over owned fine copies (per macro), written (not accumulated) on every coarse node.
// Warp per coarse row (J,K): starts of the 17x17 fine rows (2J-8..2J+8, 2K-8..2K+8) the stencils
// can touch are computed once per warp.
__global__ void k_restrict(const int32_t* __restrict__ rowsc, int64_t nrowsc, int Nc, int64_t nptsf, int64_t nptsc,
                           int64_t cstridef, int64_t cstridec, const uint8_t* __restrict__ ownf,
                           const double* __restrict__ rf, double* __restrict__ rc_out) {
  __shared__ int srs[8][289];
  RowCtx rc;
  if (!row_of(rowsc, nrowsc, Nc, rc)) return;
  const int mac = blockIdx.y;
  const int Nf = 2 * Nc;
  const int J = rc.j, K = rc.k, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = lane; r < 289; r += 32) {
    const int fy = 2 * J + r % 17 - 8, fz = 2 * K + r / 17 - 8;
    srs[w][r] = (fy >= 0 && fz >= 0 && fy + fz <= Nf) ? rowstart_i32(Nf, fy, fz) : -1;
  }
  __syncwarp();
  const int64_t fb = (int64_t)mac * nptsf;
  const uint8_t* om = ownf + fb;
  const double* rm = rf + fb;
  double* cr = rc_out + (int64_t)mac * nptsc + rowstart_i32(Nc, J, K);
  const int pc0 = ((J & 1) << 1) | ((K & 1) << 2);
  // 2 passes over I mod 2 so that all lanes of a pass share one stencil class (no divergence)
  const int half = (rc.len + 1) / 2;
  for (int it = lane; it < 2 * half; it += 32) {
    const int ph = it / half, I = 2 * (it % half) + ph;
    if (I >= rc.len) continue;
    const int pc = ph | pc0;
    const int n = __ldg(gRn + pc);
    const int lim = Nf - 2 * J - 2 * K;  // fx + (fy - 2J) + (fz - 2K) <= lim
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll 4
    for (int e = 0; e < n; ++e) {  // branch-free body: out-of-lattice / non-owned entries get weight 0
      const int d = __ldg(&gRd[pc][e]);
      const int dx = (d & 31) - 8, dy = ((d >> 5) & 31) - 8, dz = (d >> 10) - 8;
      const int fx = 2 * I + dx;
      const int rs = srs[w][(dy + 8) + 17 * (dz + 8)];
      const bool in = fx >= 0 && rs >= 0 && fx + dy + dz <= lim;
      const int fi = in ? rs + fx : 0;
      HHG_CHECK(fi >= 0 && fi < nptsf, "restrict gather", fi, nptsf);
      const double wt = (in && om[fi]) ? __ldg(&gRw[pc][e]) : 0.0;
      s0 += wt * __ldg(rm + fi);
      s1 += wt * __ldg(rm + cstridef + fi);
      s2 += wt * __ldg(rm + 2 * cstridef + fi);
    }
    cr[I] = s0;
    cr[cstridec + I] = s1;
    cr[2 * cstridec + I] = s2;
  }
}

int transfer_prepare() { return ensure_transfer_tabs(); }

int launch_prolong(const Mesh* m, const Level& Lc, const Level& Lf, const double* xc, double* xf, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;
  HHG_TRY(ensure_transfer_tabs());
  const int64_t nm = macro_count(m);
  dim3 grid((unsigned)((Lf.nrows2 + 7) / 8), (unsigned)nm);
  k_prolong<<<grid, 256, 0, s>>>(Lf.rows2, Lf.nrows2, Lf.n2, Lf.npts2, Lc.npts2, nm * Lf.npts2, nm * Lc.npts2, xc, xf);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

int launch_restrict(const Mesh* m, const Level& Lc, const Level& Lf, const double* rf, double* rc, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;
  HHG_TRY(ensure_transfer_tabs());
  const int64_t nm = macro_count(m);
  dim3 grid((unsigned)((Lc.nrows2 + 7) / 8), (unsigned)nm);
  k_restrict<<<grid, 256, 0, s>>>(Lc.rows2, Lc.nrows2, Lc.n2, Lf.npts2, Lc.npts2, nm * Lf.npts2, nm * Lc.npts2,
                                  Lf.own2, rf, rc);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// ------------------------------------------------------------------ P1 transfers (w-BFBT K multigrid)
// Nested P1 spaces: a fine node F (res 2 Nc) with odd-coordinate pattern o != 0 is the midpoint of the
// coarse lattice edge F -/+ d(o) (the 7 edge directions of the Freudenthal split); linear interpolation
// x_f(F) = 1/2 (x_c((F - d)/2) + x_c((F + d)/2)), x_f(2C) = x_c(C).  Restriction = the transpose over
// owned fine copies, then the interface sum of the coarse copies.
__device__ __forceinline__ void p1_dir(int o, int& dx, int& dy, int& dz) {
  // o = ox | oy << 1 | oz << 2  ->  d with |d_r| = o_r: (1,-1,0), (1,0,-1), (0,1,-1), (1,-1,1) for pairs/triple
  dx = o & 1;
  dy = (o >> 1) & 1;
  dz = (o >> 2) & 1;
  if (dx && dy) dy = -1;
  else if (dz && (dx || dy)) dz = -1;
  if (o == 7) dz = 1;
}

__global__ void k_p1_prolong(const int32_t* __restrict__ rowsf, int64_t nrowsf, int Nf, int64_t nptsf, int64_t nptsc,
                             const double* __restrict__ xc, double* __restrict__ xf) {
  RowCtx rc;
  if (!row_of(rowsf, nrowsf, Nf, rc)) return;
  const int mac = blockIdx.y, Nc = Nf / 2, lane = threadIdx.x & 31;
  const double* cm = xc + (int64_t)mac * nptsc;
  double* fr = xf + (int64_t)mac * nptsf + rowstart_i32(Nf, rc.j, rc.k);
  for (int I = lane; I < rc.len; I += 32) {
    const int o = (I & 1) | ((rc.j & 1) << 1) | ((rc.k & 1) << 2);
    if (o == 0) {
      fr[I] += __ldg(cm + rowstart_i32(Nc, rc.j >> 1, rc.k >> 1) + (I >> 1));
      continue;
    }
    int dx, dy, dz;
    p1_dir(o, dx, dy, dz);
    const int a = rowstart_i32(Nc, (rc.j - dy) >> 1, (rc.k - dz) >> 1) + ((I - dx) >> 1);
    const int b = rowstart_i32(Nc, (rc.j + dy) >> 1, (rc.k + dz) >> 1) + ((I + dx) >> 1);
    fr[I] += 0.5 * (__ldg(cm + a) + __ldg(cm + b));
  }
}

__global__ void k_p1_restrict(const int32_t* __restrict__ rowsc, int64_t nrowsc, int Nc, int64_t nptsf, int64_t nptsc,
                              const uint8_t* __restrict__ ownf, const double* __restrict__ rf, double* __restrict__ rc_out) {
  RowCtx rc;
  if (!row_of(rowsc, nrowsc, Nc, rc)) return;
  const int mac = blockIdx.y, Nf = 2 * Nc, lane = threadIdx.x & 31;
  const int64_t fb = (int64_t)mac * nptsf;
  const uint8_t* om = ownf + fb;
  const double* rm = rf + fb;
  double* cr = rc_out + (int64_t)mac * nptsc + rowstart_i32(Nc, rc.j, rc.k);
  const int FY = 2 * rc.j, FZ = 2 * rc.k;
  for (int I = lane; I < rc.len; I += 32) {
    const int FX = 2 * I;
    int c = rowstart_i32(Nf, FY, FZ) + FX;
    double s = om[c] ? rm[c] : 0.0;
#pragma unroll
    for (int o = 1; o < 8; ++o) {
      int dx, dy, dz;
      p1_dir(o, dx, dy, dz);
#pragma unroll
      for (int sg = -1; sg <= 1; sg += 2) {
        const int x = FX + sg * dx, y = FY + sg * dy, z = FZ + sg * dz;
        if (x < 0 || y < 0 || z < 0 || x + y + z > Nf) continue;
        c = rowstart_i32(Nf, y, z) + x;
        if (om[c]) s += 0.5 * rm[c];
      }
    }
    cr[I] = s;
  }
}

int launch_p1_prolong(const Mesh* m, const Level& Lc, const Level& Lf, const double* xc, double* xf, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;
  const int64_t nm = macro_count(m);
  dim3 grid((unsigned)((Lf.nrows1 + 7) / 8), (unsigned)nm);
  k_p1_prolong<<<grid, 256, 0, s>>>(Lf.rows1, Lf.nrows1, Lf.n1, Lf.npts1, Lc.npts1, xc, xf);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

int launch_p1_restrict(const Mesh* m, const Level& Lc, const Level& Lf, const double* rf, double* rc, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;
  const int64_t nm = macro_count(m);
  dim3 grid((unsigned)((Lc.nrows1 + 7) / 8), (unsigned)nm);
  k_p1_restrict<<<grid, 256, 0, s>>>(Lc.rows1, Lc.nrows1, Lc.n1, Lf.npts1, Lc.npts1, Lf.own1, rf, rc);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// ------------------------------------------------------------------ coordinates
__global__ void k_coords(const MacroGeo* __restrict__ mgeo, const int32_t* __restrict__ rows, int64_t nrows, int N,
                         int64_t npts, bool blend, double* __restrict__ xyz) {
  RowCtx rc;
  if (!row_of(rows, nrows, N, rc)) return;
  const int mac = blockIdx.y;
  const MacroGeo& g = mgeo[mac];
  const int64_t base = (int64_t)mac * npts + lidx(0, rc.j, rc.k, N);
  for (int i = threadIdx.x & 31; i < rc.len; i += 32) {
    const double a = (double)i / N, b = (double)rc.j / N, c = (double)rc.k / N;
    double x[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) x[r] = g.X0[r] + g.Jm[3 * r] * a + g.Jm[3 * r + 1] * b + g.Jm[3 * r + 2] * c;
    if (blend) {
      const double rr = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
      const double f = g.cK * (g.nhat[0] * x[0] + g.nhat[1] * x[1] + g.nhat[2] * x[2]) / rr;
      x[0] *= f;
      x[1] *= f;
      x[2] *= f;
    }
    double* o = xyz + 3 * (base + i);
    o[0] = x[0];
    o[1] = x[1];
    o[2] = x[2];
  }
}

int launch_coords(const Mesh* m, const Level& L, int space, double* xyz, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;
  const int64_t nm = macro_count(m);
  const bool p1 = space == HHG_P1;
  const int64_t nrows = p1 ? L.nrows1 : L.nrows2;
  dim3 grid((unsigned)((nrows + 7) / 8), (unsigned)nm);
  k_coords<<<grid, 256, 0, s>>>(m->dgeo, p1 ? L.rows1 : L.rows2, nrows, p1 ? L.n1 : L.n2, p1 ? L.npts1 : L.npts2,
                                m->blend == HHG_BLEND_SHELL, xyz);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// ------------------------------------------------------------------ canonical gather / scatter
__global__ void k_canon(int64_t nstored, int nc, int64_t ncanon_nodes, const int64_t* __restrict__ map,
                        const double* __restrict__ v, double* __restrict__ c, bool to) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nstored; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ci = map[i];
    for (int k = 0; k < nc; ++k) {
      if (to) c[ci * nc + k] = v[k * nstored + i];
      else c[k * nstored + i] = v[ci * nc + k];
    }
  }
}

int launch_gather_canon(const Level& L, int space, int64_t nstored, const double* v, double* c, bool to,
                        cudaStream_t s) {
  const bool p1 = space == HHG_P1;
  const int nc = space == HHG_P2VEC ? 3 : 1;
  k_canon<<<1184, 256, 0, s>>>(nstored, nc, p1 ? L.ncanon1 : L.ncanon2, p1 ? L.canon1 : L.canon2, v, c, to);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// ------------------------------------------------------------------ vector kernels
#define GRID_STRIDE(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)
static inline unsigned vgrid(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  GRID_STRIDE(i, n) y[i] = a * x[i] + b * y[i];
}
// first Chebyshev step: r = f - t (t = A x, or x = 0 when t == nullptr), d = D^-1 r / theta
__global__ void k_cheb0(int64_t n, const double* __restrict__ f, const double* __restrict__ t,
                        const double* __restrict__ dinv, double it, double* __restrict__ r, double* __restrict__ d) {
  GRID_STRIDE(i, n) {
    const double ri = t ? f[i] - t[i] : f[i];
    r[i] = ri;
    d[i] = dinv[i] * ri * it;
  }
}
// degree-1 sweep fused: x += D^-1 (f - t) / theta   (t == nullptr: x = 0 on entry)
__global__ void k_cheb_deg1(int64_t n, const double* __restrict__ f, const double* __restrict__ t,
                            const double* __restrict__ dinv, double it, double* __restrict__ x) {
  GRID_STRIDE(i, n) {
    const double ri = t ? f[i] - t[i] : f[i];
    x[i] = (t ? x[i] : 0.0) + dinv[i] * ri * it;
  }
}
// last Chebyshev step fused with the final update: x += d + (c1 d + c2 D^-1 (r - t)); r, d dead after
__global__ void k_chebk_last(int64_t n, const double* __restrict__ t, const double* __restrict__ dinv, double c1,
                             double c2, const double* __restrict__ r, const double* __restrict__ d,
                             double* __restrict__ x) {
  GRID_STRIDE(i, n) {
    const double di = d[i];
    x[i] += di + (c1 * di + c2 * dinv[i] * (r[i] - t[i]));
  }
}
__global__ void k_chebk(int64_t n, const double* __restrict__ t, const double* __restrict__ dinv, double c1, double c2,
                        double* __restrict__ x, double* __restrict__ r, double* __restrict__ d) {
  GRID_STRIDE(i, n) {
    const double di = d[i];
    x[i] += di;
    const double ri = r[i] - t[i];
    r[i] = ri;
    d[i] = c1 * di + c2 * dinv[i] * ri;
  }
}

__global__ void k_fill(int64_t n, double v, double* __restrict__ y) { GRID_STRIDE(i, n) y[i] = v; }
__global__ void k_recip(int64_t n, double* __restrict__ y) { GRID_STRIDE(i, n) y[i] = 1.0 / y[i]; }
__global__ void k_scale(int64_t n, const double* __restrict__ d, const double* __restrict__ x, double* __restrict__ y) {
  GRID_STRIDE(i, n) y[i] = d[i] * x[i];
}
int launch_fill(int64_t n, double v, double* y, cudaStream_t s) {
  k_fill<<<vgrid(n), 256, 0, s>>>(n, v, y);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_recip(int64_t n, double* y, cudaStream_t s) {
  k_recip<<<vgrid(n), 256, 0, s>>>(n, y);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_pcg_scale(int64_t n, const double* d, const double* x, double* y, cudaStream_t s) {
  k_scale<<<vgrid(n), 256, 0, s>>>(n, d, x, y);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s) {
  k_axpby<<<vgrid(n), 256, 0, s>>>(n, a, x, b, y);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_cheb0(int64_t n, const double* f, const double* t, const double* dinv, double inv_theta, double* r,
                 double* d, cudaStream_t s) {
  k_cheb0<<<vgrid(n), 256, 0, s>>>(n, f, t, dinv, inv_theta, r, d);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_cheb_deg1(int64_t n, const double* f, const double* t, const double* dinv, double inv_theta, double* x,
                     cudaStream_t s) {
  k_cheb_deg1<<<vgrid(n), 256, 0, s>>>(n, f, t, dinv, inv_theta, x);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_chebk_last(int64_t n, const double* t, const double* dinv, double c1, double c2, const double* r,
                      const double* d, double* x, cudaStream_t s) {
  k_chebk_last<<<vgrid(n), 256, 0, s>>>(n, t, dinv, c1, c2, r, d, x);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_chebk(int64_t n, const double* t, const double* dinv, double c1, double c2, double* x, double* r,
                 double* d, cudaStream_t s) {
  k_chebk<<<vgrid(n), 256, 0, s>>>(n, t, dinv, c1, c2, x, r, d);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// ---- node-major variants: i over stored P2 nodes, the 3 components at i, i+cs, i+2cs; the BC
// projection P_v M of the new direction is applied per node (Dirichlet: 0; free slip: remove the
// normal component with the node group's normal) -- identical to a BC-only interface pass on a
// consistent vector.
__global__ void k_cheb0_bc(int64_t ns, int64_t cs, const double* __restrict__ f, const double* __restrict__ t,
                           const double* __restrict__ dinv, double it, double* __restrict__ r, double* __restrict__ d,
                           const int32_t* __restrict__ bcn, const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    double dv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      const double ri = t ? f[j] - t[j] : f[j];
      r[j] = ri;
      dv[c] = dinv[j] * ri * it;
    }
    bc_project(bcn[i], nrm, dv[0], dv[1], dv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) d[i + c * cs] = dv[c];
  }
}
__global__ void k_cheb_deg1_bc(int64_t ns, int64_t cs, const double* __restrict__ f, const double* __restrict__ t,
                               const double* __restrict__ dinv, double it, double* __restrict__ x,
                               const int32_t* __restrict__ bcn, const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    double dv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      dv[c] = dinv[j] * (t ? f[j] - t[j] : f[j]) * it;
    }
    bc_project(bcn[i], nrm, dv[0], dv[1], dv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      x[j] = (t ? x[j] : 0.0) + dv[c];
    }
  }
}
__global__ void k_chebk_bc(int64_t ns, int64_t cs, const double* __restrict__ t, const double* __restrict__ dinv,
                           double c1, double c2, double* __restrict__ x, double* __restrict__ r, double* __restrict__ d,
                           const int32_t* __restrict__ bcn, const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    double dv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      const double di = d[j];
      x[j] += di;
      const double ri = r[j] - t[j];
      r[j] = ri;
      dv[c] = c1 * di + c2 * dinv[j] * ri;
    }
    bc_project(bcn[i], nrm, dv[0], dv[1], dv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) d[i + c * cs] = dv[c];
  }
}
__global__ void k_chebk_last_bc(int64_t ns, int64_t cs, const double* __restrict__ t, const double* __restrict__ dinv,
                                double c1, double c2, const double* __restrict__ r, const double* __restrict__ d,
                                double* __restrict__ x, const int32_t* __restrict__ bcn,
                                const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    double dn[3], dold[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      dold[c] = d[j];
      dn[c] = c1 * dold[c] + c2 * dinv[j] * (r[j] - t[j]);
    }
    bc_project(bcn[i], nrm, dn[0], dn[1], dn[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) x[i + c * cs] += dold[c] + dn[c];
  }
}
__global__ void k_pcg_update_bc(int64_t ns, int64_t cs, const double* __restrict__ rzp, const double* __restrict__ pqp,
                                double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                                const double* __restrict__ q, const double* __restrict__ dinv, double* __restrict__ z,
                                const int32_t* __restrict__ bcn, const double* __restrict__ nrm) {
  const double rz = *rzp, pq = *pqp;
  const double alpha = (rz > 1e-300 && pq != 0.0) ? rz / pq : 0.0;
  GRID_STRIDE(i, ns) {
    double zv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      x[j] += alpha * p[j];
      const double ri = r[j] - alpha * q[j];
      r[j] = ri;
      zv[c] = dinv[j] * ri;
    }
    bc_project(bcn[i], nrm, zv[0], zv[1], zv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) z[i + c * cs] = zv[c];
  }
}
// p = z + beta p, beta = rz_new / rz_old (0 once converged to the zero-rhs guard); q = 0 for the
// next operator application
__global__ void k_pcg_dir_zero(int64_t n, const double* __restrict__ rzo, const double* __restrict__ rzn,
                               const double* __restrict__ z, double* __restrict__ p, double* __restrict__ q) {
  const double a = *rzo, b = *rzn;
  const double beta = a > 1e-300 ? b / a : 0.0;
  GRID_STRIDE(i, n) {
    p[i] = z[i] + beta * p[i];
    q[i] = 0.0;
  }
}

static inline unsigned ngrid(int64_t ns) {
  int64_t b = (ns + 255) / 256;
  return (unsigned)(b < 148 * 8 ? (b < 1 ? 1 : b) : 148 * 8);
}
#define NODE_ARGS(m, L) (macro_count(m) * (L).npts2), (macro_count(m) * (L).npts2)
int launch_cheb0_bc(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                    double inv_theta, double* r, double* d, cudaStream_t s) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_cheb0_bc<<<ngrid(ns), 256, 0, s>>>(NODE_ARGS(m, L), f, t, dinv, inv_theta, r, d, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_cheb_deg1_bc(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                        double inv_theta, double* x, cudaStream_t s) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_cheb_deg1_bc<<<ngrid(ns), 256, 0, s>>>(NODE_ARGS(m, L), f, t, dinv, inv_theta, x, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_chebk_bc(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2, double* x,
                    double* r, double* d, cudaStream_t s) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_chebk_bc<<<ngrid(ns), 256, 0, s>>>(NODE_ARGS(m, L), t, dinv, c1, c2, x, r, d, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_chebk_last_bc(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2,
                         const double* r, const double* d, double* x, cudaStream_t s) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_chebk_last_bc<<<ngrid(ns), 256, 0, s>>>(NODE_ARGS(m, L), t, dinv, c1, c2, r, d, x, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_pcg_update_bc(const Mesh* m, const Level& L, int it, const double* scal, double* x, double* r,
                         const double* p, const double* q, const double* dinv, double* z, cudaStream_t s) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_pcg_update_bc<<<ngrid(ns), 256, 0, s>>>(NODE_ARGS(m, L), scal + ((it & 1) ? 2 : 0), scal + 1, x, r, p, q, dinv,
                                            z, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_pcg_dir_zero(int64_t n, int it, const double* scal, const double* z, double* p, double* q_zero,
                        cudaStream_t s) {
  k_pcg_dir_zero<<<vgrid(n), 256, 0, s>>>(n, scal + ((it & 1) ? 2 : 0), scal + ((it & 1) ? 0 : 2), z, p, q_zero);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// PCG scalars live on the device: scal[0] = r.z (old), scal[1] = p.q, scal[2] = r.z (new)
// op 0: alpha-step done in k_pcg_update; op 1: beta = new/old, old = new
__global__ void k_pcg_update(int64_t n, const double* __restrict__ scal, double* __restrict__ x,
                             double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ q,
                             const double* __restrict__ dinv, double* __restrict__ z) {
  const double rz = scal[0], pq = scal[1];
  const double alpha = (rz > 1e-300 && pq != 0.0) ? rz / pq : 0.0;
  GRID_STRIDE(i, n) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    z[i] = dinv[i] * ri;
  }
}
int launch_pcg_update(int64_t n, const double* scal, double* x, double* r, const double* p, const double* q,
                      const double* dinv, double* z, cudaStream_t s) {
  k_pcg_update<<<vgrid(n), 256, 0, s>>>(n, scal, x, r, p, q, dinv, z);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
// p = z + beta p, beta = scal[2]/scal[0] (0 if stopped); then scal[0] = scal[2]
__global__ void k_pcg_dir(int64_t n, double* __restrict__ scal, const double* __restrict__ z, double* __restrict__ p) {
  const double rz = scal[0], rzn = scal[2];
  const double beta = rz > 1e-300 ? rzn / rz : 0.0;
  GRID_STRIDE(i, n) p[i] = z[i] + beta * p[i];
}
__global__ void k_pcg_roll(double* scal) {
  if (threadIdx.x == 0 && blockIdx.x == 0) scal[0] = scal[0] > 1e-300 ? scal[2] : scal[0];
}
int launch_pcg_dir(int64_t n, double* scal, const double* z, double* p, cudaStream_t s) {
  k_pcg_dir<<<vgrid(n), 256, 0, s>>>(n, scal, z, p);
  k_pcg_roll<<<1, 32, 0, s>>>(scal);
  count_launch(2);
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

}  // namespace hhg

namespace hhg {
// ------------------------------------------------------------------ fused interface sum + BC consumers
// t is the raw element-kernel output (per-copy partial sums).  tval() returns, for stored node i, the value
// k_fixup<3, true> would have written: the sum of its group's copies (fixed copy order -> every copy gets
// the bitwise same value) with the group's BC applied, or t[i] for nodes in no group.
struct FxArgs {
  const int32_t* __restrict__ gmap;
  const int64_t* __restrict__ ptr;
  const int64_t* __restrict__ copy;
  const uint8_t* __restrict__ kind;
  const double* __restrict__ normal;
  const uint8_t* __restrict__ skip;  // nodes already updated by the fused element-kernel epilogue (or nullptr)
};
__device__ __forceinline__ void tval(const FxArgs& a, int64_t i, int64_t cs, const double* __restrict__ t,
                                     double (&v)[3]) {
  const int g = a.gmap[i];
  if (g < 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) v[c] = t[i + c * cs];
    return;
  }
  group_sum<3>(a.ptr[g], a.ptr[g + 1], a.copy, cs, t, v);
  group_bc<3>(a.kind[g], a.normal + 3 * g, v);
}
static FxArgs fx_args(const Level& L, const uint8_t* skip) {
  return FxArgs{L.gmap2, L.g2.ptr, L.g2.copy, L.g2.kind, L.g2.normal, skip};
}
#define FX_SKIP(a, i) \
  if ((a).skip && (a).skip[i]) continue;

__global__ void k_cheb0_fx(int64_t ns, int64_t cs, FxArgs a, const double* __restrict__ f, const double* __restrict__ t,
                           const double* __restrict__ dinv, double it, double* __restrict__ r, double* __restrict__ d,
                           const int32_t* __restrict__ bcn, const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    FX_SKIP(a, i)
    double tv[3], dv[3];
    tval(a, i, cs, t, tv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      const double ri = f[j] - tv[c];
      r[j] = ri;
      dv[c] = dinv[j] * ri * it;
    }
    bc_project(bcn[i], nrm, dv[0], dv[1], dv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) d[i + c * cs] = dv[c];
  }
}
__global__ void k_cheb_deg1_fx(int64_t ns, int64_t cs, FxArgs a, const double* __restrict__ f,
                               const double* __restrict__ t, const double* __restrict__ dinv, double it,
                               double* __restrict__ x, const int32_t* __restrict__ bcn, const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    FX_SKIP(a, i)
    double tv[3], dv[3];
    tval(a, i, cs, t, tv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      dv[c] = dinv[j] * (f[j] - tv[c]) * it;
    }
    bc_project(bcn[i], nrm, dv[0], dv[1], dv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) x[i + c * cs] += dv[c];
  }
}
__global__ void k_chebk_fx(int64_t ns, int64_t cs, FxArgs a, const double* __restrict__ t,
                           const double* __restrict__ dinv, double c1, double c2, double* __restrict__ x,
                           double* __restrict__ r, double* __restrict__ d, const int32_t* __restrict__ bcn,
                           const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    FX_SKIP(a, i)
    double tv[3], dv[3];
    tval(a, i, cs, t, tv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      const double di = d[j];
      x[j] += di;
      const double ri = r[j] - tv[c];
      r[j] = ri;
      dv[c] = c1 * di + c2 * dinv[j] * ri;
    }
    bc_project(bcn[i], nrm, dv[0], dv[1], dv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) d[i + c * cs] = dv[c];
  }
}
__global__ void k_chebk_last_fx(int64_t ns, int64_t cs, FxArgs a, const double* __restrict__ t,
                                const double* __restrict__ dinv, double c1, double c2, const double* __restrict__ r,
                                const double* __restrict__ d, double* __restrict__ x, const int32_t* __restrict__ bcn,
                                const double* __restrict__ nrm) {
  GRID_STRIDE(i, ns) {
    FX_SKIP(a, i)
    double tv[3], dn[3], dold[3];
    tval(a, i, cs, t, tv);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      dold[c] = d[j];
      dn[c] = c1 * dold[c] + c2 * dinv[j] * (r[j] - tv[c]);
    }
    bc_project(bcn[i], nrm, dn[0], dn[1], dn[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) x[i + c * cs] += dold[c] + dn[c];
  }
}
__global__ void k_sub_fx(int64_t ns, int64_t cs, FxArgs a, const double* __restrict__ f, const double* __restrict__ t,
                         double* __restrict__ r) {
  GRID_STRIDE(i, ns) {
    FX_SKIP(a, i)
    double tv[3];
    tval(a, i, cs, t, tv);
#pragma unroll
    for (int c = 0; c < 3; ++c) r[i + c * cs] = f[i + c * cs] - tv[c];
  }
}
int launch_cheb0_fx(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                    double inv_theta, double* r, double* d, cudaStream_t s, const uint8_t* skip) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_cheb0_fx<<<ngrid(ns), 256, 0, s>>>(ns, ns, fx_args(L, skip), f, t, dinv, inv_theta, r, d, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_cheb_deg1_fx(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                        double inv_theta, double* x, cudaStream_t s) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_cheb_deg1_fx<<<ngrid(ns), 256, 0, s>>>(ns, ns, fx_args(L, nullptr), f, t, dinv, inv_theta, x, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_chebk_fx(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2, double* x,
                    double* r, double* d, cudaStream_t s, const uint8_t* skip) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_chebk_fx<<<ngrid(ns), 256, 0, s>>>(ns, ns, fx_args(L, skip), t, dinv, c1, c2, x, r, d, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_chebk_last_fx(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2,
                         const double* r, const double* d, double* x, cudaStream_t s, const uint8_t* skip) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_chebk_last_fx<<<ngrid(ns), 256, 0, s>>>(ns, ns, fx_args(L, skip), t, dinv, c1, c2, r, d, x, L.bcn2, L.g2.normal);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
int launch_sub_fx(const Mesh* m, const Level& L, const double* f, const double* t, double* r, cudaStream_t s, const uint8_t* skip) {
  const int64_t ns = macro_count(m) * L.npts2;
  k_sub_fx<<<ngrid(ns), 256, 0, s>>>(ns, ns, fx_args(L, skip), f, t, r);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// PCG step x += a p, r -= a q, z = P_v M D^-1 r fused with the new r.z (owner-weighted, block partials in
// `red`, the last block sums them in fixed order -- the same reduction as k_dot_fused) into rz_out; single
// rank only (a multi-rank dot needs an allreduce after the kernel)
__global__ void k_pcg_update_bc_dot(int64_t ns, int64_t cs, const double* __restrict__ rzp,
                                    const double* __restrict__ pqp, double* __restrict__ x, double* __restrict__ r,
                                    const double* __restrict__ p, const double* __restrict__ q,
                                    const double* __restrict__ dinv, double* __restrict__ z,
                                    const int32_t* __restrict__ bcn, const double* __restrict__ nrm,
                                    const uint8_t* __restrict__ own, double* __restrict__ part,
                                    unsigned* __restrict__ counter, double* __restrict__ rz_out) {
  const double rz = *rzp, pq = *pqp;
  const double alpha = (rz > 1e-300 && pq != 0.0) ? rz / pq : 0.0;
  double acc = 0.0;
  GRID_STRIDE(i, ns) {
    double zv[3], rv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      x[j] += alpha * p[j];
      rv[c] = r[j] - alpha * q[j];
      r[j] = rv[c];
      zv[c] = dinv[j] * rv[c];
    }
    bc_project(bcn[i], nrm, zv[0], zv[1], zv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) z[i + c * cs] = zv[c];
    if (own[i]) acc += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
  }
  __shared__ double sh[32];
  __shared__ bool last;
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      part[blockIdx.x] = v;
      __threadfence();
      last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += ((volatile double*)part)[i];
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      *rz_out = v;
      *counter = 0u;
    }
  }
}
int launch_pcg_update_bc_dot(const Mesh* m, const Level& L, int it, double* scal, double* x, double* r, const double* p,
                             const double* q, const double* dinv, double* z, double* red, cudaStream_t s) {
  const int64_t ns = macro_count(m) * L.npts2;
  int64_t nb = (ns + 255) / 256;
  nb = nb < 1 ? 1 : (nb > kRedBlocks ? kRedBlocks : nb);
  k_pcg_update_bc_dot<<<(unsigned)nb, 256, 0, s>>>(ns, ns, scal + ((it & 1) ? 2 : 0), scal + 1, x, r, p, q, dinv, z,
                                                   L.bcn2, L.g2.normal, L.own2, red,
                                                   reinterpret_cast<unsigned*>(red + kRedBlocks + 4),
                                                   scal + ((it & 1) ? 0 : 2));
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
}  // namespace hhg
