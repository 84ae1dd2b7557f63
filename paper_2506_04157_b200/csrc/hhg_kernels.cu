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

namespace hhg {

// Q4 rule (R6): barycentric (a,b,b,b) and permutations, weights 1/24.
constexpr double QA = 0.58541019662496845446;  // (5 + 3 sqrt 5)/20
constexpr double QB = 0.13819660112501051518;  // (5 - sqrt 5)/20
constexpr double QAB = QA - QB;
constexpr double WQ = 1.0 / 24.0;

__constant__ int cTV[6][4][3] = {
    {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
    {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}},
    {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}},
    {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}},
};
// integer inverse of E_t (columns V1-V0, V2-V0, V3-V0), row-major, for the 6 types
__constant__ int cEinv[6][9];

// local P2 numbering: 0..3 vertices, 4..9 edges 01,02,03,12,13,23
#define EI(m, j) (((m) == 0) ? (3 + (j)) : (((m) == 1) ? (((j) == 0) ? 4 : 5 + (j)) : (((m) == 2) ? (((j) == 0) ? 5 : ((j) == 1 ? 7 : 9)) : (((j) == 0) ? 6 : ((j) == 1 ? 8 : 9)))))

__device__ __forceinline__ int64_t d_lidx(int i, int j, int k, int N) { return lidx(i, j, k, N); }

static bool g_einv_ready = false;
static int ensure_einv() {
  if (g_einv_ready) return HHG_OK;
  int h[6][9];
  const int TV[6][4][3] = {
      {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}}};
  for (int t = 0; t < 6; ++t) {
    int E[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) E[3 * r + c] = TV[t][c + 1][r] - TV[t][0][r];
    int det = E[0] * (E[4] * E[8] - E[5] * E[7]) - E[1] * (E[3] * E[8] - E[5] * E[6]) + E[2] * (E[3] * E[7] - E[4] * E[6]);
    int adj[9] = {E[4] * E[8] - E[5] * E[7], E[2] * E[7] - E[1] * E[8], E[1] * E[5] - E[2] * E[4],
                  E[5] * E[6] - E[3] * E[8], E[0] * E[8] - E[2] * E[6], E[2] * E[3] - E[0] * E[5],
                  E[3] * E[7] - E[4] * E[6], E[1] * E[6] - E[0] * E[7], E[0] * E[4] - E[1] * E[3]};
    for (int i = 0; i < 9; ++i) h[t][i] = adj[i] * det;  // det = +-1 -> inverse = adj/det = adj*det
  }
  HHG_CUDA(cudaMemcpyToSymbol(cEinv, h, sizeof(h)));
  g_einv_ready = true;
  return HHG_OK;
}

// ------------------------------------------------------------------ interface sum + BC
template <int NC, bool BC>
__global__ void k_fixup(int64_t ng, const int64_t* __restrict__ ptr, const int64_t* __restrict__ copy,
                        const uint8_t* __restrict__ kind, const double* __restrict__ normal, int64_t cstride,
                        bool sum, double* __restrict__ v) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= ng) return;
  const int64_t b = ptr[gi], e = ptr[gi + 1];
  double val[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double s = v[c * cstride + copy[b]];
    if (sum)
      for (int64_t k = b + 1; k < e; ++k) s += v[c * cstride + copy[k]];
    val[c] = s;
  }
  if (BC) {
    const int kd = kind[gi];
    if (kd == HHG_BC_DIRICHLET0) {
#pragma unroll
      for (int c = 0; c < NC; ++c) val[c] = 0.0;
    } else if (kd == HHG_BC_FREESLIP && NC == 3) {
      const double n0 = normal[3 * gi], n1 = normal[3 * gi + 1], n2 = normal[3 * gi + 2];
      const double un = val[0] * n0 + val[1] * n1 + val[2 % NC] * n2;
      val[0] -= un * n0;
      val[1 % NC] -= un * n1;
      val[2 % NC] -= un * n2;
    }
  }
  if (!sum && !BC) return;
  for (int64_t k = b; k < e; ++k)
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c * cstride + copy[k]] = val[c];
}

int launch_fixup(const Mesh* m, const Level& L, int space, bool sum, bool bc, double* v, cudaStream_t s) {
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

int launch_dot(const Mesh* m, const Level& L, int space, const double* x, const double* y, double* out,
               cudaStream_t s) {
  const int64_t nm = macro_count(m);
  const bool p1 = space == HHG_P1;
  const int64_t nst = nm * (p1 ? L.npts1 : L.npts2);
  const int nc = space == HHG_P2VEC ? 3 : 1;
  k_dot_partial<<<kRedBlocks, 256, 0, s>>>(nst, nc, nst, p1 ? L.own1 : L.own2, x, y, L.red);
  k_dot_final<<<1, 256, 0, s>>>(L.red, kRedBlocks, out);
  count_launch(2);
  HHG_CUDA(cudaGetLastError());
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

// P2 prolongation: x_f += P x_c on every stored fine node (per macro, consistent copies)
template <bool RESTRICT>
__global__ void k_transfer(const int32_t* __restrict__ rowsf, int64_t nrowsf, int Nf, int64_t nptsf, int64_t nptsc,
                           int64_t cstridef, int64_t cstridec, const uint8_t* __restrict__ ownf,
                           const double* __restrict__ src, double* __restrict__ dst) {
  RowCtx rc;
  if (!row_of(rowsf, nrowsf, Nf, rc)) return;
  const int mac = blockIdx.y;
  const int Nc = Nf / 2;
  const int64_t fb = (int64_t)mac * nptsf + lidx(0, rc.j, rc.k, Nf);
  const int64_t cb = (int64_t)mac * nptsc;
  for (int i = threadIdx.x & 31; i < rc.len; i += 32) {
    const int I = i, J = rc.j, K = rc.k;
    const int64_t f = fb + i;
    double w[10];
    int64_t cid[10];
    int nn;
    if (((I | J | K) & 1) == 0) {
      nn = 1;
      w[0] = 1.0;
      cid[0] = cb + lidx(I >> 1, J >> 1, K >> 1, Nc);
    } else {
      const int a0 = I >> 2, a1 = J >> 2, a2 = K >> 2;
      const int F0 = I & 3, F1 = J & 3, F2 = K & 3;
      const int S = F0 + F1 + F2;
      int t;
      if (S <= 4) t = 0;
      else if (S > 8) t = 5;
      else {
        const bool xy = F0 + F1 >= 4, yz = F1 + F2 >= 4;
        t = xy ? (yz ? 3 : 1) : (yz ? 4 : 2);
      }
      int V[4][3];
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int r = 0; r < 3; ++r) V[v][r] = cTV[t][v][r];
      const int q0 = F0 - 4 * V[0][0], q1 = F1 - 4 * V[0][1], q2 = F2 - 4 * V[0][2];
      int b[4];
      b[1] = cEinv[t][0] * q0 + cEinv[t][1] * q1 + cEinv[t][2] * q2;
      b[2] = cEinv[t][3] * q0 + cEinv[t][4] * q1 + cEinv[t][5] * q2;
      b[3] = cEinv[t][6] * q0 + cEinv[t][7] * q1 + cEinv[t][8] * q2;
      b[0] = 4 - b[1] - b[2] - b[3];
      double lam[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) lam[v] = 0.25 * b[v];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        w[v] = lam[v] * (2.0 * lam[v] - 1.0);
        cid[v] = cb + lidx(2 * (a0 + V[v][0]), 2 * (a1 + V[v][1]), 2 * (a2 + V[v][2]), Nc);
      }
      const int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        const int p = ep[e][0], q = ep[e][1];
        w[4 + e] = 4.0 * lam[p] * lam[q];
        cid[4 + e] = cb + lidx(2 * a0 + V[p][0] + V[q][0], 2 * a1 + V[p][1] + V[q][1], 2 * a2 + V[p][2] + V[q][2], Nc);
      }
      nn = 10;
    }
    if (!RESTRICT) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int a = 0; a < nn; ++a) s += w[a] * src[c * cstridec + cid[a]];
        dst[c * cstridef + f] += s;
      }
    } else {
      if (!ownf[f]) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double r = src[c * cstridef + f];
        for (int a = 0; a < nn; ++a)
          if (w[a] != 0.0) atomicAdd(dst + c * cstridec + cid[a], w[a] * r);
      }
    }
  }
}

int launch_prolong(const Mesh* m, const Level& Lc, const Level& Lf, const double* xc, double* xf, cudaStream_t s) {
  HHG_TRY(ensure_einv());
  const int64_t nm = macro_count(m);
  dim3 grid((unsigned)((Lf.nrows2 + 7) / 8), (unsigned)nm);
  k_transfer<false><<<grid, 256, 0, s>>>(Lf.rows2, Lf.nrows2, Lf.n2, Lf.npts2, Lc.npts2, nm * Lf.npts2,
                                         nm * Lc.npts2, Lf.own2, xc, xf);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

int launch_restrict(const Mesh* m, const Level& Lc, const Level& Lf, const double* rf, double* rc, cudaStream_t s) {
  HHG_TRY(ensure_einv());
  const int64_t nm = macro_count(m);
  dim3 grid((unsigned)((Lf.nrows2 + 7) / 8), (unsigned)nm);
  k_transfer<true><<<grid, 256, 0, s>>>(Lf.rows2, Lf.nrows2, Lf.n2, Lf.npts2, Lc.npts2, nm * Lf.npts2,
                                        nm * Lc.npts2, Lf.own2, rf, rc);
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
__global__ void k_cheb0(int64_t n, const double* __restrict__ f, const double* __restrict__ t,
                        const double* __restrict__ dinv, double it, double* __restrict__ r, double* __restrict__ d) {
  GRID_STRIDE(i, n) {
    const double ri = f[i] - t[i];
    r[i] = ri;
    d[i] = dinv[i] * ri * it;
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
int launch_chebk(int64_t n, const double* t, const double* dinv, double c1, double c2, double* x, double* r,
                 double* d, cudaStream_t s) {
  k_chebk<<<vgrid(n), 256, 0, s>>>(n, t, dinv, c1, c2, x, r, d);
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
