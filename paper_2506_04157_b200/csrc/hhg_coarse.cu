// Coarse-grid solve of the V-cycle ("the coarse grid problem is solved by a Jacobi-preconditioned
// CG" with a fixed iteration count, R15) as ONE kernel resident on one thread-block cluster.
//
// The coarsest level is tiny (shell(3,2) L1: 1 920 micro tets, 8 400 stored P2 nodes), so the generic path
// -- element kernel, interface sum, fused dot, update, direction: five launches per iteration -- is bound by
// launch gaps and tails (~36 us per iteration, ~1.8 ms of a 26 ms V-cycle).  Here every PCG iteration runs
// inside one kernel on ONE cluster of kCl CTAs (compile-time cluster shape: it is part of the function, so a
// CUDA-graph capture of the launch cannot lose it), phases separated by hardware cluster barriers:
//   A  q_e = A_e p'  per micro tet (tet_body, the same arithmetic as the brick kernel), p' = z + beta p
//      formed on the fly; the 30 element outputs go to a buffer E ordered by unique node (no atomics);
//   B  per UNIQUE node u (an interface/BC group of g2, or a stored node in no group): q_u = the sum of u's
//      contiguous E segment (the outputs of every tet of every copy, fixed host-built order) + the group's BC
//      (= element kernel + k_fixup(sum, BC)); p = z + beta p; both written to every copy; partial p.q;
//   C  alpha = r.z / p.q; x += alpha p, r -= alpha q, z = P_v M D^-1 r on every copy; partial r.z;
// three cluster barriers per iteration; vectors stay consistent, so each scalar step runs once per unique node
// and the dots need no owner mask; the dots are reduced in fixed order by every CTA (deterministic, identical
// scalars everywhere).  Data written inside the kernel is read with ld.global.cg (L2), never through the
// non-coherent L1.  Semantics = mg_pcg (hhg_mg.cu) with the brick element kernel.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hhg_internal.h"
#include "hhg_device.cuh"
#include "hhg_tet.cuh"

namespace cg = cooperative_groups;

namespace hhg {

constexpr int kCT = 256;   // threads per CTA
constexpr int kCl = 8;     // CTAs per cluster (compile-time __cluster_dims__: kept by CUDA-graph capture)
constexpr int kClMax = kCl;

struct CoarseArgs {
  int64_t ns;               // stored P2 nodes (= component stride)
  int ntet, n1;
  double inv_n1;
  int64_t npts1, npts2;
  const MacroGeo* mgeo;
  const double* lgeo;
  const int32_t* node;      // [10][ntet] stored P2 index of local node a
  const int32_t* p1;        // [4][ntet] stored P1 index of vertex v
  const int32_t* info;      // [ntet] macro | type << 24
  const int32_t* anc;       // [ntet] cube anchor i | j << 10 | k << 20
  const int32_t* pos;       // [10][ntet] slot of element output (tet, a) in the node-ordered buffer E
  int nu, ng;               // unique nodes; the first ng are the interface/BC groups of g2 (same ids)
  const int32_t* ucp;       // [nu+1] CSR of the stored copies of u
  const int32_t* ucopy;     // stored copies (the first is the representative)
  const int32_t* urep;      // [nu] representative copy of u
  const int32_t* ub;        // [kCl+1] unique nodes of CTA b: [ub[b], ub[b+1])
  const int32_t* ib;        // [kCl+1] items of CTA b: [ib[b], ib[b+1])
  const int32_t* item;      // [nitems+1] E range of item k: [item[k], item[k+1]) (<= kIt entries, one node each)
  const int32_t* uitem;     // [nu+1] items of unique node u: [uitem[u], uitem[u+1])
  // shared-memory-resident variant (k_coarse_pcg_sm): owner CTA | local index of every tet node's unique node and
  // of every element output's E slot, the CTAs' E starts, and the per-CTA capacities (array strides)
  const int32_t* onode;     // [10][ntet]
  const int32_t* opos;      // [10][ntet]
  const int32_t* eb;        // [kCl+1]
  int NL, NE, NI;
  unsigned long long* dbg;  // HHG_CCL_TIMING=1: accumulated globaltimer ns per phase (CTA 0, thread 0)
  const uint8_t* kind;      // group BC kind
  const double* normal;     // group normals [3]
  const int32_t* bcn;       // per node BC for P_v M on directions
  const double* eta;        // P1 viscosity (nullptr: 1)
  const double* T2;         // P2 temperature (quadrature-point viscosity tier)
  EtaQ eq;
  const double* dinv;
  const double* f;
  double *x, *r, *z, *p, *q, *E, *part;
  int iters;
  double tol2;              // stop when r.z <= tol2 r0.z0 (0: exactly `iters` iterations)
  int* it_out;              // iterations taken (device)
};

__device__ __forceinline__ double ldcg(const double* a) { return __ldcg(a); }

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kCT / 32; ++w) t += sh[w];
  __syncthreads();
  return t;  // valid in thread 0
}
// cluster-wide sum: block partial -> part[blockIdx.x], barrier, every thread sums the partials in fixed order
__device__ __forceinline__ double cluster_sum(double v, double* part, double* sh, cg::cluster_group& cl) {
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  cl.sync();
  double s = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) s += ldcg(part + b);
  return s;
}

struct GU {  // p' = z + beta p at the tet's 10 nodes, gathered into registers
  double u[10][3];
  __device__ __forceinline__ double operator()(int a, int c) const { return u[a][c]; }
};
struct GT {
  double t[10];
  __device__ __forceinline__ double operator()(int a) const { return t[a]; }
};

// element outputs of micro tet e for the gathered p' (everything but the gather and the scatter)
template <bool BLEND, bool FULL, bool ETAQ>
__device__ __forceinline__ void coarse_tet(const CoarseArgs& a, int e, const GU& uu, double (&accE)[10][3]) {
  const int nt = a.ntet;
  const int inf = __ldg(a.info + e), an = __ldg(a.anc + e);
  const int mac = inf & 0xffffff, t = inf >> 24;
  GT tt;
  if (ETAQ) {
#pragma unroll
    for (int k = 0; k < 10; ++k) tt.t[k] = __ldg(a.T2 + __ldg(a.node + k * nt + e));
  }
  double et[4], pp[4] = {0, 0, 0, 0};
#pragma unroll
  for (int v = 0; v < 4; ++v) et[v] = a.eta ? __ldg(a.eta + __ldg(a.p1 + v * nt + e)) : 1.0;
  const MacroGeo& g = a.mgeo[mac];
  double nh[3] = {0, 0, 0}, cK = 1.0;
  if (BLEND) {
    nh[0] = g.nhat[0];
    nh[1] = g.nhat[1];
    nh[2] = g.nhat[2];
    cK = g.cK;
  }
  const double fa = (an & 1023) * a.inv_n1, fb = ((an >> 10) & 1023) * a.inv_n1, fc = (an >> 20) * a.inv_n1;
  double xa[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) xa[r] = g.X0[r] + g.Jm[3 * r] * fa + g.Jm[3 * r + 1] * fb + g.Jm[3 * r + 2] * fc;
  const double* Gm = a.lgeo + (int64_t)mac * kLevelGeo;
  double G[kTypeGeo];
#pragma unroll
  for (int k = 0; k < kTypeGeo; ++k) G[k] = __ldg(Gm + t * kTypeGeo + k);
  const double wdet = EWQ * __ldg(Gm + 6 * kTypeGeo);
  double gy[4];
  tet_body<BLEND, ELEM_A, FULL, GU, ETAQ, GT>(G, wdet, xa, nh, cK, 0.0, uu, et, pp, accE, gy, tt, a.eq);
}

constexpr int kIt = 16;   // E entries per work item (one load round trip)
constexpr int kNP = 4;    // unique nodes per thread per pass (their loads issued together)

template <bool BLEND, bool FULL, bool ETAQ>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kCT, 1) k_coarse_pcg(CoarseArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double sh[kCT / 32];
  extern __shared__ double dsm[];
  const int nthr = gridDim.x * blockDim.x;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, tid = threadIdx.x;
  const int64_t cs = a.ns;
  double* part = a.part;  // [3][kClMax] ping-pong partials (each buffer reused two barriers later)
  int pb = 0;
  auto next_part = [&]() {
    double* P = part + pb * kClMax;
    pb = (pb + 1) % 3;
    return P;
  };
  // this CTA's unique nodes [u0, u1) and items [i0, i1); shared: item partials [3][ni], q [3][nl]
  const int u0 = a.ub[blockIdx.x], u1 = a.ub[blockIdx.x + 1], nl = u1 - u0;
  const int i0 = a.ib[blockIdx.x], i1 = a.ib[blockIdx.x + 1], ni = i1 - i0;
  double* ps = dsm;             // [3][ni]
  double* qs = dsm + 3 * ni;    // [3][nl]
  auto store_all = [&](int u, double* v, const double (&val)[3]) {
    for (int k = __ldg(a.ucp + u), ke = __ldg(a.ucp + u + 1); k < ke; ++k) {
      const int64_t i = __ldg(a.ucopy + k);
#pragma unroll
      for (int c = 0; c < 3; ++c) v[i + c * cs] = val[c];
    }
  };

  // x = 0, r = f, z = P_v M D^-1 r, p = z (x, r at the representative; z, p on every copy); rz = r.z
  double acc = 0.0;
  for (int l = tid; l < nl; l += kCT) {
    const int u = u0 + l;
    const int64_t i = __ldg(a.urep + u);
    double rv[3], zv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      rv[c] = a.f[i + c * cs];
      zv[c] = __ldg(a.dinv + i + c * cs) * rv[c];
      a.x[i + c * cs] = 0.0;
      a.r[i + c * cs] = rv[c];
    }
    bc_project(__ldg(a.bcn + i), a.normal, zv[0], zv[1], zv[2]);
    store_all(u, a.z, zv);
    store_all(u, a.p, zv);
    acc += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
  }
  double rz = cluster_sum(acc, next_part(), sh, cl);
  const double rz_stop = a.tol2 * rz;  // every thread holds the same rz: the exit below is uniform
  double beta = 0.0;

  const int nt = a.ntet;
  const int64_t ne = 10 * (int64_t)nt;  // component stride of E
  int it = 0;
  for (; it < a.iters; ++it) {
    if (a.tol2 > 0.0 && (rz <= rz_stop || rz <= 1e-300)) break;
    // ---- A: element outputs of p' = z + beta p
    for (int e = gt; e < nt; e += nthr) {
      GU uu;
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int64_t j = __ldg(a.node + k * nt + e);
#pragma unroll
        for (int c = 0; c < 3; ++c) uu.u[k][c] = fma(beta, ldcg(a.p + j + c * cs), ldcg(a.z + j + c * cs));
      }
      double accE[10][3];
      coarse_tet<BLEND, FULL, ETAQ>(a, e, uu, accE);
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int64_t ps_ = __ldg(a.pos + k * nt + e);
#pragma unroll
        for (int c = 0; c < 3; ++c) a.E[c * ne + ps_] = accE[k][c];
      }
    }
    cl.sync();
    // ---- B1: item partial sums (<= kIt contiguous E entries of one node, summed in order) into shared memory
    for (int k = tid; k < ni; k += kCT) {
      const int e0 = __ldg(a.item + i0 + k), e1 = __ldg(a.item + i0 + k + 1);
      double v[kIt][3];
#pragma unroll
      for (int j = 0; j < kIt; ++j)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[j][c] = (e0 + j < e1) ? ldcg(a.E + c * ne + e0 + j) : 0.0;
      double sv[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < kIt; ++j)
#pragma unroll
        for (int c = 0; c < 3; ++c) sv[c] += v[j][c];
#pragma unroll
      for (int c = 0; c < 3; ++c) ps[c * ni + k] = sv[c];
    }
    __syncthreads();
    // ---- B2: q_u = sum of u's item partials (in order) + the group's BC (= element kernel + k_fixup(sum, BC));
    // p = z + beta p on every copy; partial p.q
    acc = 0.0;
    for (int l0 = tid; l0 < nl; l0 += kCT * kNP) {
      double zr[kNP][3], pr[kNP][3];
#pragma unroll
      for (int n = 0; n < kNP; ++n) {
        const int l = l0 + n * kCT;
        const int64_t i = l < nl ? __ldg(a.urep + u0 + l) : 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          zr[n][c] = l < nl ? ldcg(a.z + i + c * cs) : 0.0;
          pr[n][c] = l < nl ? ldcg(a.p + i + c * cs) : 0.0;
        }
      }
#pragma unroll
      for (int n = 0; n < kNP; ++n) {
        const int l = l0 + n * kCT;
        if (l >= nl) break;
        const int u = u0 + l;
        double qv[3] = {0.0, 0.0, 0.0}, pv[3];
        for (int k = __ldg(a.uitem + u) - i0, ke = __ldg(a.uitem + u + 1) - i0; k < ke; ++k)
#pragma unroll
          for (int c = 0; c < 3; ++c) qv[c] += ps[c * ni + k];
        if (u < a.ng) group_bc<3>(__ldg(a.kind + u), a.normal + 3 * u, qv);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pv[c] = fma(beta, pr[n][c], zr[n][c]);
          qs[c * nl + l] = qv[c];
        }
        store_all(u, a.p, pv);
        acc += pv[0] * qv[0] + pv[1] * qv[1] + pv[2] * qv[2];
      }
    }
    const double pq = cluster_sum(acc, next_part(), sh, cl);
    const double alpha = (rz > 1e-300 && pq != 0.0) ? rz / pq : 0.0;
    // ---- C: x += alpha p, r -= alpha q (representative), z = P_v M D^-1 r (every copy); partial r.z
    acc = 0.0;
    for (int l0 = tid; l0 < nl; l0 += kCT * kNP) {
      double pr[kNP][3], xr[kNP][3], rr[kNP][3];
      int64_t ir[kNP];
#pragma unroll
      for (int n = 0; n < kNP; ++n) {
        const int l = l0 + n * kCT;
        ir[n] = l < nl ? __ldg(a.urep + u0 + l) : 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          pr[n][c] = l < nl ? ldcg(a.p + ir[n] + c * cs) : 0.0;
          xr[n][c] = l < nl ? ldcg(a.x + ir[n] + c * cs) : 0.0;
          rr[n][c] = l < nl ? ldcg(a.r + ir[n] + c * cs) : 0.0;
        }
      }
#pragma unroll
      for (int n = 0; n < kNP; ++n) {
        const int l = l0 + n * kCT;
        if (l >= nl) break;
        const int64_t i = ir[n];
        double zv[3], rv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          a.x[i + c * cs] = fma(alpha, pr[n][c], xr[n][c]);
          rv[c] = fma(-alpha, qs[c * nl + l], rr[n][c]);
          a.r[i + c * cs] = rv[c];
          zv[c] = __ldg(a.dinv + i + c * cs) * rv[c];
        }
        bc_project(__ldg(a.bcn + i), a.normal, zv[0], zv[1], zv[2]);
        store_all(u0 + l, a.z, zv);
        acc += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
      }
    }
    const double rzn = cluster_sum(acc, next_part(), sh, cl);
    beta = rz > 1e-300 ? rzn / rz : 0.0;
    rz = rzn;
  }
  // x lives at the representatives during the iteration: broadcast to every copy
  for (int l = tid; l < nl; l += kCT) {
    const int u = u0 + l;
    const int64_t i = __ldg(a.urep + u);
    const double xv[3] = {ldcg(a.x + i), ldcg(a.x + i + cs), ldcg(a.x + i + 2 * cs)};
    store_all(u, a.x, xv);
  }
  if (gt == 0) *a.it_out = it;
}


// Shared-memory-resident variant (coarse levels whose per-CTA working set fits: shell(3,2) L1): every vector of a
// unique node lives in its owner CTA's shared memory for the whole solve; the tet phase reads p, z and writes its
// element outputs through distributed shared memory (DSMEM) of the owner CTAs; nothing but f, D^-1 and the final x
// touches global memory.  Same arithmetic and summation order as k_coarse_pcg.
template <bool BLEND, bool FULL, bool ETAQ>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kCT, 1) k_coarse_pcg_sm(CoarseArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double sh[kCT / 32];
  __shared__ double spart[3];
  extern __shared__ double dsm[];
  const int NL = a.NL, NE = a.NE, NI = a.NI;
  double* xs = dsm;
  double* rs = xs + 3 * NL;
  double* zs = rs + 3 * NL;
  double* ps = zs + 3 * NL;
  double* qs = ps + 3 * NL;
  double* ds = qs + 3 * NL;
  double* Es = ds + 3 * NL;
  double* pi = Es + 3 * NE;
  const int nthr = gridDim.x * blockDim.x;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, tid = threadIdx.x;
  const int b = blockIdx.x;
  const int64_t cs = a.ns;
  const int u0 = a.ub[b], nl = a.ub[b + 1] - u0;
  const int i0 = a.ib[b], ni = a.ib[b + 1] - i0;
  const int e0 = a.eb[b];
  int pb = 0;
  auto csum = [&](double v) {  // cluster sum through DSMEM, partials added in CTA order (identical everywhere)
    const double t = block_sum(v, sh);
    if (tid == 0) spart[pb] = t;
    cl.sync();
    double s = 0.0;
    for (int r = 0; r < kCl; ++r) s += *cl.map_shared_rank(spart + pb, r);
    pb = (pb + 1) % 3;
    return s;
  };
  // x = 0, r = f, z = P_v M D^-1 r, p = z; rz = r.z
  double acc = 0.0;
  for (int l = tid; l < nl; l += kCT) {
    const int64_t i = __ldg(a.urep + u0 + l);
    double rv[3], zv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      rv[c] = a.f[i + c * cs];
      ds[c * NL + l] = __ldg(a.dinv + i + c * cs);
      zv[c] = ds[c * NL + l] * rv[c];
    }
    bc_project(__ldg(a.bcn + i), a.normal, zv[0], zv[1], zv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xs[c * NL + l] = 0.0;
      rs[c * NL + l] = rv[c];
      zs[c * NL + l] = zv[c];
      ps[c * NL + l] = zv[c];
    }
    acc += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
  }
  double rz = csum(acc);
  const double rz_stop = a.tol2 * rz;
  double beta = 0.0;
  const int nt = a.ntet;
  int it = 0;
  unsigned long long tA = 0;
  auto tick = [&](int ph) {
    if (a.dbg && gt == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (ph >= 0) a.dbg[ph] += t - tA;
      tA = t;
    }
  };
  for (; it < a.iters; ++it) {
    if (a.tol2 > 0.0 && (rz <= rz_stop || rz <= 1e-300)) break;
    tick(-1);
    // ---- A: p' = z + beta p gathered from the owners (DSMEM), element outputs scattered to the owners' E
    for (int e = gt; e < nt; e += nthr) {
      GU uu;
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int o = __ldg(a.onode + k * nt + e);
        const double* rp = cl.map_shared_rank(ps, o >> 24);
        const double* rzz = cl.map_shared_rank(zs, o >> 24);
        const int loc = o & 0xffffff;
#pragma unroll
        for (int c = 0; c < 3; ++c) uu.u[k][c] = fma(beta, rp[c * NL + loc], rzz[c * NL + loc]);
      }
      double accE[10][3];
      coarse_tet<BLEND, FULL, ETAQ>(a, e, uu, accE);
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int o = __ldg(a.opos + k * nt + e);
        double* rE = cl.map_shared_rank(Es, o >> 24);
        const int loc = o & 0xffffff;
#pragma unroll
        for (int c = 0; c < 3; ++c) rE[c * NE + loc] = accE[k][c];
      }
    }
    tick(0);
    cl.sync();
    tick(1);
    // ---- B1: item partials (<= kIt E entries of one node, in order)
    for (int k = tid; k < ni; k += kCT) {
      const int ea = __ldg(a.item + i0 + k) - e0, eb_ = __ldg(a.item + i0 + k + 1) - e0;
      double sv[3] = {0.0, 0.0, 0.0};
      for (int j = ea; j < eb_; ++j)
#pragma unroll
        for (int c = 0; c < 3; ++c) sv[c] += Es[c * NE + j];
#pragma unroll
      for (int c = 0; c < 3; ++c) pi[c * NI + k] = sv[c];
    }
    __syncthreads();
    // ---- B2: q = sum of the node's item partials + group BC; p = z + beta p; partial p.q
    acc = 0.0;
    for (int l = tid; l < nl; l += kCT) {
      const int u = u0 + l;
      double qv[3] = {0.0, 0.0, 0.0}, pv[3];
      for (int k = __ldg(a.uitem + u) - i0, ke = __ldg(a.uitem + u + 1) - i0; k < ke; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) qv[c] += pi[c * NI + k];
      if (u < a.ng) group_bc<3>(__ldg(a.kind + u), a.normal + 3 * u, qv);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        pv[c] = fma(beta, ps[c * NL + l], zs[c * NL + l]);
        ps[c * NL + l] = pv[c];
        qs[c * NL + l] = qv[c];
      }
      acc += pv[0] * qv[0] + pv[1] * qv[1] + pv[2] * qv[2];
    }
    tick(2);
    const double pq = csum(acc);
    tick(3);
    const double alpha = (rz > 1e-300 && pq != 0.0) ? rz / pq : 0.0;
    // ---- C: x += alpha p, r -= alpha q, z = P_v M D^-1 r; partial r.z
    acc = 0.0;
    for (int l = tid; l < nl; l += kCT) {
      double rv[3], zv[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xs[c * NL + l] = fma(alpha, ps[c * NL + l], xs[c * NL + l]);
        rv[c] = fma(-alpha, qs[c * NL + l], rs[c * NL + l]);
        rs[c * NL + l] = rv[c];
        zv[c] = ds[c * NL + l] * rv[c];
      }
      bc_project(__ldg(a.bcn + __ldg(a.urep + u0 + l)), a.normal, zv[0], zv[1], zv[2]);
#pragma unroll
      for (int c = 0; c < 3; ++c) zs[c * NL + l] = zv[c];
      acc += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
    }
    tick(4);
    const double rzn = csum(acc);
    tick(5);
    beta = rz > 1e-300 ? rzn / rz : 0.0;
    rz = rzn;
  }
  // x to every copy
  for (int l = tid; l < nl; l += kCT) {
    const int u = u0 + l;
    for (int k = __ldg(a.ucp + u), ke = __ldg(a.ucp + u + 1); k < ke; ++k) {
      const int64_t i = __ldg(a.ucopy + k);
#pragma unroll
      for (int c = 0; c < 3; ++c) a.x[i + c * cs] = xs[c * NL + l];
    }
  }
  if (gt == 0) *a.it_out = it;
  cl.sync();  // no CTA may exit while others still read its shared memory
}

struct CoarseSolver {
  CoarseArgs a{};
  size_t smem = 0;
  bool sm = false;  // shared-memory-resident variant
  bool blend = false, full = true, etaq = false;
  std::vector<void*> bufs;
  ~CoarseSolver() {
    for (void* b : bufs) cudaFree(b);
  }
};

template <class T>
static int upload(CoarseSolver* c, const std::vector<T>& h, const T** d) {
  void* p = nullptr;
  HHG_CUDA(cudaMalloc(&p, std::max<size_t>(h.size(), 1) * sizeof(T)));
  c->bufs.push_back(p);
  if (!h.empty()) HHG_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *d = static_cast<const T*>(p);
  return HHG_OK;
}

// Build the coarse solver of level `level` (single-rank mesh; tables on the host, once).
int coarse_create(const Mesh* m, int level, int form, const double* eta, const double* T2, double lnC, double jump,
                  double rjump, const double* dinv, CoarseSolver** out) {
  *out = nullptr;
  if (m->nranks != 1 || m->comm) return fail(HHG_EINVAL, "coarse solver: single-rank meshes only");
  const Level& L = m->levels[level];
  const int64_t nm = macro_count(m);
  const int n1 = L.n1, n2 = L.n2;
  const int64_t ns = nm * L.npts2;
  auto* c = new CoarseSolver();
  auto bail = [&](int r) {
    delete c;
    return r;
  };
  // micro tets (same type tables as the brick kernel: Bey/Freudenthal types)
  const int TV[6][4][3] = {
      {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}}};
  const int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  std::vector<int32_t> node, p1v, info, anc;
  std::vector<std::array<int32_t, 10>> tn;
  std::vector<std::array<int32_t, 4>> tp;
  for (int64_t mc = 0; mc < nm; ++mc)
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j + k < n1; ++j)
        for (int i = 0; i + j + k < n1; ++i) {
          const int s = i + j + k;
          const int ntp = (s <= n1 - 3) ? 6 : ((s == n1 - 2) ? 5 : 1);
          for (int t = 0; t < ntp; ++t) {
            std::array<int32_t, 10> nd;
            std::array<int32_t, 4> pv;
            int off[10][3];
            for (int v = 0; v < 4; ++v)
              for (int r = 0; r < 3; ++r) off[v][r] = 2 * TV[t][v][r];
            for (int e = 0; e < 6; ++e)
              for (int r = 0; r < 3; ++r) off[4 + e][r] = TV[t][ep[e][0]][r] + TV[t][ep[e][1]][r];
            for (int q = 0; q < 10; ++q)
              nd[q] = (int32_t)(mc * L.npts2 + lidx(2 * i + off[q][0], 2 * j + off[q][1], 2 * k + off[q][2], n2));
            for (int v = 0; v < 4; ++v)
              pv[v] = (int32_t)(mc * L.npts1 + lidx(i + TV[t][v][0], j + TV[t][v][1], k + TV[t][v][2], n1));
            tn.push_back(nd);
            tp.push_back(pv);
            info.push_back((int32_t)(mc | (int64_t)t << 24));
            anc.push_back(i | j << 10 | k << 20);
          }
        }
  const int nt = (int)tn.size();
  node.resize(10 * (size_t)nt);
  p1v.resize(4 * (size_t)nt);
  for (int e = 0; e < nt; ++e) {
    for (int q = 0; q < 10; ++q) node[(size_t)q * nt + e] = tn[e][q];
    for (int v = 0; v < 4; ++v) p1v[(size_t)v * nt + e] = tp[e][v];
  }
  // unique nodes: the g2 groups (interface and/or BC, ids 0..ng-1), then every stored node in no group
  std::vector<int32_t> gmap(ns);
  HHG_CUDA(cudaMemcpy(gmap.data(), L.gmap2, ns * sizeof(int32_t), cudaMemcpyDeviceToHost));
  const int64_t ng = L.g2.n;
  std::vector<int64_t> gptr(ng + 1, 0), gcopy(L.g2.ncopy);
  if (ng > 0) {
    HHG_CUDA(cudaMemcpy(gptr.data(), L.g2.ptr, gptr.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
    HHG_CUDA(cudaMemcpy(gcopy.data(), L.g2.copy, gcopy.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
  }
  std::vector<int32_t> uof(ns), ucp(1, 0), ucopy;
  for (int64_t g = 0; g < ng; ++g) {
    for (int64_t k = gptr[g]; k < gptr[g + 1]; ++k) ucopy.push_back((int32_t)gcopy[k]);
    ucp.push_back((int32_t)ucopy.size());
  }
  int64_t nu = ng;
  for (int64_t i = 0; i < ns; ++i) {
    if (gmap[i] >= 0) {
      uof[i] = gmap[i];
    } else {
      uof[i] = (int32_t)nu++;
      ucopy.push_back((int32_t)i);
      ucp.push_back((int32_t)ucopy.size());
    }
  }
  // E segments: element outputs grouped by unique node, in (tet, local node) order within a segment
  std::vector<int32_t> useg(nu + 1, 0), pos(10 * (size_t)nt);
  for (int e = 0; e < nt; ++e)
    for (int q = 0; q < 10; ++q) ++useg[uof[tn[e][q]] + 1];
  for (int64_t u = 0; u < nu; ++u) useg[u + 1] += useg[u];
  {
    std::vector<int32_t> fill(useg.begin(), useg.end() - 1);
    for (int e = 0; e < nt; ++e)
      for (int q = 0; q < 10; ++q) pos[(size_t)q * nt + e] = fill[uof[tn[e][q]]]++;
  }
  // CTA partition of the unique nodes (contiguous ranges, balanced by E entries + copies) and work items
  std::vector<int32_t> urep(nu), ub(kCl + 1, 0), ib(kCl + 1, 0), item(1, 0), uitem(nu + 1, 0);
  for (int64_t u = 0; u < nu; ++u) urep[u] = ucopy[ucp[u]];
  {
    std::vector<double> wcum(nu + 1, 0.0);
    for (int64_t u = 0; u < nu; ++u) wcum[u + 1] = wcum[u] + (useg[u + 1] - useg[u]) + (ucp[u + 1] - ucp[u]);
    for (int b = 1; b < kCl; ++b)
      ub[b] = (int32_t)(std::lower_bound(wcum.begin(), wcum.end(), wcum[nu] * b / kCl) - wcum.begin());
    ub[kCl] = (int32_t)nu;
    for (int b = 1; b <= kCl; ++b) ub[b] = std::max(ub[b], ub[b - 1]);
  }
  size_t smem_max = 0;
  for (int b = 0; b < kCl; ++b) {
    ib[b] = (int32_t)(item.size() - 1);
    for (int64_t u = ub[b]; u < ub[b + 1]; ++u) {
      uitem[u] = (int32_t)(item.size() - 1);
      for (int32_t e0 = useg[u]; e0 < useg[u + 1]; e0 += kIt) item.push_back(std::min(e0 + kIt, useg[u + 1]));
      uitem[u + 1] = (int32_t)(item.size() - 1);
    }
    ib[b + 1] = (int32_t)(item.size() - 1);
    smem_max = std::max(smem_max, (size_t)3 * sizeof(double) * ((ib[b + 1] - ib[b]) + (ub[b + 1] - ub[b])));
  }
  if (smem_max > 200 * 1024) return bail(fail(HHG_ENOMEM, "coarse solver: coarse level too large for one cluster"));
  c->smem = smem_max;
  // shared-memory-resident layout: owner CTA | local index of each tet node's unique node and E slot
  std::vector<int32_t> onode(10 * (size_t)nt), opos(10 * (size_t)nt), eb(kCl + 1);
  int NL = 0, NE = 0, NI = 0;
  {
    std::vector<int32_t> cta_of(nu);
    for (int b = 0; b < kCl; ++b) {
      for (int64_t u = ub[b]; u < ub[b + 1]; ++u) cta_of[u] = b;
      eb[b] = useg[ub[b]];
      NL = std::max(NL, ub[b + 1] - ub[b]);
      NE = std::max(NE, useg[ub[b + 1]] - useg[ub[b]]);
      NI = std::max(NI, ib[b + 1] - ib[b]);
    }
    eb[kCl] = useg[nu];
    for (int e = 0; e < nt; ++e)
      for (int q = 0; q < 10; ++q) {
        const int u = uof[tn[e][q]], b = cta_of[u];
        onode[(size_t)q * nt + e] = b << 24 | (u - ub[b]);
        opos[(size_t)q * nt + e] = b << 24 | (pos[(size_t)q * nt + e] - eb[b]);
      }
  }
  const size_t smem_sm = sizeof(double) * (18 * (size_t)NL + 3 * (size_t)NE + 3 * (size_t)NI);
  {
    const char* e = getenv("HHG_CCL_GLOBAL");  // A/B switch: force the global-memory variant
    c->sm = smem_sm <= 200 * 1024 && !(e && e[0] == '1');
  }
  if (c->sm) c->smem = smem_sm;
  CoarseArgs& a = c->a;
  a.ns = ns;
  a.ntet = nt;
  a.n1 = n1;
  a.inv_n1 = 1.0 / n1;
  a.npts1 = L.npts1;
  a.npts2 = L.npts2;
  a.mgeo = m->dgeo;
  a.lgeo = L.geo;
  int r;
  a.nu = (int)nu;
  a.ng = (int)ng;
  a.NL = NL;
  a.NE = NE;
  a.NI = NI;
  if ((r = upload(c, node, &a.node)) || (r = upload(c, p1v, &a.p1)) || (r = upload(c, info, &a.info)) ||
      (r = upload(c, anc, &a.anc)) || (r = upload(c, pos, &a.pos)) || (r = upload(c, ucp, &a.ucp)) ||
      (r = upload(c, ucopy, &a.ucopy)) || (r = upload(c, urep, &a.urep)) || (r = upload(c, ub, &a.ub)) ||
      (r = upload(c, ib, &a.ib)) || (r = upload(c, item, &a.item)) || (r = upload(c, uitem, &a.uitem)) ||
      (r = upload(c, onode, &a.onode)) || (r = upload(c, opos, &a.opos)) || (r = upload(c, eb, &a.eb)))
    return bail(r);
  a.kind = L.g2.kind;
  a.normal = L.g2.normal;
  a.bcn = L.bcn2;
  a.eta = eta;
  a.T2 = T2;
  a.eq = EtaQ{lnC, jump, rjump};
  a.dinv = dinv;
  void* E = nullptr;
  if (cudaMalloc(&E, (size_t)30 * std::max(nt, 1) * sizeof(double) + 3 * kClMax * sizeof(double) + 8) != cudaSuccess)
    return bail(fail(HHG_ENOMEM, "coarse solver buffers"));
  c->bufs.push_back(E);
  a.E = static_cast<double*>(E);
  a.part = a.E + (size_t)30 * std::max(nt, 1);
  a.it_out = reinterpret_cast<int*>(a.part + 3 * kClMax);
  HHG_CUDA(cudaMemset(a.it_out, 0, sizeof(int)));
  {
    const char* e = getenv("HHG_CCL_TIMING");
    if (e && e[0] == '1') {
      void* d = nullptr;
      HHG_CUDA(cudaMalloc(&d, 6 * sizeof(unsigned long long)));
      c->bufs.push_back(d);
      HHG_CUDA(cudaMemset(d, 0, 6 * sizeof(unsigned long long)));
      a.dbg = static_cast<unsigned long long*>(d);
    }
  }
  c->blend = m->blend == HHG_BLEND_SHELL;
  c->full = form == HHG_VISC_FULL;
  c->etaq = T2 != nullptr;
  if (c->etaq && !c->full) return bail(fail(HHG_EINVAL, "coarse solver: quadrature-point viscosity needs the full form"));
#define HHG_CSMEM(B, F, Q)                                                                                    \
  r = cudaFuncSetAttribute(c->sm ? k_coarse_pcg_sm<B, F, Q> : k_coarse_pcg<B, F, Q>,                         \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem) == cudaSuccess        \
          ? HHG_OK                                                                                          \
          : fail(HHG_ECUDA, "coarse solver: shared memory attribute");
  if (c->etaq) {
    if (c->blend) HHG_CSMEM(true, true, true) else HHG_CSMEM(false, true, true)
  } else if (c->blend) {
    if (c->full) HHG_CSMEM(true, true, false) else HHG_CSMEM(true, false, false)
  } else {
    if (c->full) HHG_CSMEM(false, true, false) else HHG_CSMEM(false, false, false)
  }
#undef HHG_CSMEM
  if (r != HHG_OK) return bail(r);
  *out = c;
  return HHG_OK;
}

template <bool B, bool F, bool Q>
static int coarse_launch(CoarseSolver* c, cudaStream_t s) {
  if (c->sm) k_coarse_pcg_sm<B, F, Q><<<kCl, kCT, c->smem, s>>>(c->a);
  else k_coarse_pcg<B, F, Q><<<kCl, kCT, c->smem, s>>>(c->a);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

// Jacobi-PCG from x = 0 on rhs f (work vectors r, z, p, q of the level's length): exactly `iters` iterations,
// or (tol > 0) until sqrt(r.z) <= tol sqrt(r0.z0), at most `iters`
int coarse_run(CoarseSolver* c, const double* f, double* x, double* r, double* z, double* p, double* q, int iters,
               double tol, cudaStream_t s) {
  CoarseArgs& a = c->a;
  a.tol2 = tol * tol;
  a.f = f;
  a.x = x;
  a.r = r;
  a.z = z;
  a.p = p;
  a.q = q;
  a.iters = iters;
  if (c->etaq) return c->blend ? coarse_launch<true, true, true>(c, s) : coarse_launch<false, true, true>(c, s);
  if (c->blend) return c->full ? coarse_launch<true, true, false>(c, s) : coarse_launch<true, false, false>(c, s);
  return c->full ? coarse_launch<false, true, false>(c, s) : coarse_launch<false, false, false>(c, s);
}

int coarse_timing(const CoarseSolver* c, unsigned long long* ns6) {
  if (!c->a.dbg) return fail(HHG_EINVAL, "coarse solver: built without HHG_CCL_TIMING=1");
  HHG_CUDA(cudaDeviceSynchronize());
  HHG_CUDA(cudaMemcpy(ns6, c->a.dbg, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return HHG_OK;
}

int coarse_iterations(const CoarseSolver* c, int* out) {
  HHG_CUDA(cudaDeviceSynchronize());
  HHG_CUDA(cudaMemcpy(out, c->a.it_out, sizeof(int), cudaMemcpyDeviceToHost));
  if (c->a.dbg) {  // HHG_CCL_TIMING=1 diagnostics (shared-memory variant): accumulated ns per phase
    unsigned long long t[6];
    HHG_TRY(coarse_timing(c, t));
    fprintf(stderr, "{\"hhg_ccl_timing_ns\": {\"A\": %llu, \"sync_A\": %llu, \"B\": %llu, \"sum_pq\": %llu, \"C\": %llu, "
            "\"sum_rz\": %llu}}\n", t[0], t[1], t[2], t[3], t[4], t[5]);
  }
  return HHG_OK;
}

void coarse_destroy(CoarseSolver* c) { delete c; }

}  // namespace hhg
