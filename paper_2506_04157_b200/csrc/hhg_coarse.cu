// Coarse-grid solve of the V-cycle ("the coarse grid problem is solved by a Jacobi-preconditioned
// CG" with a fixed iteration count, R15) as ONE kernel resident on one thread-block cluster.
//
// The coarsest level is tiny (shell(3,2) L1: 1 920 micro tets, 8 400 stored P2 nodes), so the generic path
// -- element kernel, interface sum, fused dot, update, direction: five launches per iteration -- is bound by
// launch gaps and tails (~36 us per iteration, ~1.8 ms of a 26 ms V-cycle).  Here every PCG iteration runs
// inside one kernel on a cluster of kCl CTAs separated by hardware cluster barriers:
//   A  q_e = A_e p'  per micro tet (tet_body, the same arithmetic as the brick kernel), p' = z + beta p
//      formed on the fly; the 30 element outputs go to a per-tet buffer E (no atomics);
//   B  per stored node: p = z + beta p (stored), q = sum of the E slots of every copy of the node's
//      interface group in a fixed host-built order (so all copies are bitwise equal) + the group's BC
//      (= element kernel + k_fixup(sum, BC)); partial p.q over owned nodes;
//   C  alpha = r.z / p.q; x += alpha p, r -= alpha q, z = P_v M D^-1 r; partial r.z;
// three cluster barriers per iteration; the dots are reduced in fixed order by every CTA (deterministic,
// identical scalars everywhere).  Data written inside the kernel is read with ld.global.cg (L2), never
// through the non-coherent L1.  Semantics = mg_pcg (hhg_mg.cu) with the brick element kernel.
#include <cooperative_groups.h>

#include <vector>

#include "hhg_internal.h"
#include "hhg_device.cuh"
#include "hhg_tet.cuh"

namespace cg = cooperative_groups;

namespace hhg {

constexpr int kCT = 256;   // threads per CTA
constexpr int kClMax = 16; // non-portable cluster size (falls back to 8)

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
  const int32_t* sb;        // [ns] first slot of the node's gather list
  const int32_t* se;        // [ns] one past the last slot
  const int32_t* slot;      // slots a * ntet + tet
  const int32_t* gmap;      // [ns] interface/BC group or -1
  const uint8_t* kind;      // group BC kind
  const double* normal;     // group normals [3]
  const int32_t* bcn;       // per node BC for P_v M on directions
  const uint8_t* own;
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

template <bool BLEND, bool FULL, bool ETAQ>
__global__ void __launch_bounds__(kCT, 1) k_coarse_pcg(CoarseArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double sh[kCT / 32];
  const int nthr = gridDim.x * blockDim.x;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ns = a.ns, cs = a.ns;
  double* part = a.part;  // [3][kClMax] ping-pong partials (each buffer reused two barriers later)
  int pb = 0;
  auto next_part = [&]() {
    double* P = part + pb * kClMax;
    pb = (pb + 1) % 3;
    return P;
  };

  // x = 0, r = f, z = P_v M D^-1 r, p = z, rz = r.z
  double acc = 0.0;
  for (int64_t i = gt; i < ns; i += nthr) {
    double rv[3], zv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t j = i + c * cs;
      rv[c] = a.f[j];
      zv[c] = a.dinv[j] * rv[c];
      a.x[j] = 0.0;
      a.r[j] = rv[c];
    }
    bc_project(a.bcn[i], a.normal, zv[0], zv[1], zv[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a.z[i + c * cs] = zv[c];
      a.p[i + c * cs] = zv[c];
    }
    if (a.own[i]) acc += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
  }
  double rz = cluster_sum(acc, next_part(), sh, cl);
  const double rz_stop = a.tol2 * rz;  // every thread holds the same rz: the exit below is uniform
  double beta = 0.0;

  const int nt = a.ntet;
  int it = 0;
  for (; it < a.iters; ++it) {
    if (a.tol2 > 0.0 && (rz <= rz_stop || rz <= 1e-300)) break;
    // ---- A: element outputs of p' = z + beta p
    for (int e = gt; e < nt; e += nthr) {
      const int inf = __ldg(a.info + e), an = __ldg(a.anc + e);
      const int mac = inf & 0xffffff, t = inf >> 24;
      GU uu;
#pragma unroll
      for (int k = 0; k < 10; ++k) {
        const int64_t j = __ldg(a.node + k * nt + e);
#pragma unroll
        for (int c = 0; c < 3; ++c) uu.u[k][c] = fma(beta, ldcg(a.p + j + c * cs), ldcg(a.z + j + c * cs));
      }
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
      double accE[10][3], gy[4];
      tet_body<BLEND, ELEM_A, FULL, GU, ETAQ, GT>(G, wdet, xa, nh, cK, 0.0, uu, et, pp, accE, gy, tt, a.eq);
#pragma unroll
      for (int k = 0; k < 10; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) a.E[(int64_t)(c * 10 + k) * nt + e] = accE[k][c];
    }
    cl.sync();
    // ---- B: p = z + beta p; q = interface sum of the element outputs + BC; partial p.q
    acc = 0.0;
    for (int64_t i = gt; i < ns; i += nthr) {
      double qv[3] = {0.0, 0.0, 0.0}, pv[3];
      const int b0 = __ldg(a.sb + i), b1 = __ldg(a.se + i);
      for (int k = b0; k < b1; ++k) {
        const int64_t sl = __ldg(a.slot + k);
#pragma unroll
        for (int c = 0; c < 3; ++c) qv[c] += ldcg(a.E + (int64_t)c * 10 * nt + sl);
      }
      const int g = __ldg(a.gmap + i);
      if (g >= 0) group_bc<3>(__ldg(a.kind + g), a.normal + 3 * g, qv);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t j = i + c * cs;
        pv[c] = fma(beta, ldcg(a.p + j), ldcg(a.z + j));
        a.p[j] = pv[c];
        a.q[j] = qv[c];
      }
      if (a.own[i]) acc += pv[0] * qv[0] + pv[1] * qv[1] + pv[2] * qv[2];
    }
    const double pq = cluster_sum(acc, next_part(), sh, cl);
    const double alpha = (rz > 1e-300 && pq != 0.0) ? rz / pq : 0.0;
    // ---- C: x += alpha p, r -= alpha q, z = P_v M D^-1 r; partial r.z
    acc = 0.0;
    for (int64_t i = gt; i < ns; i += nthr) {
      double rv[3], zv[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int64_t j = i + c * cs;
        a.x[j] = fma(alpha, ldcg(a.p + j), ldcg(a.x + j));
        rv[c] = fma(-alpha, ldcg(a.q + j), ldcg(a.r + j));
        a.r[j] = rv[c];
        zv[c] = __ldg(a.dinv + j) * rv[c];
      }
      bc_project(a.bcn[i], a.normal, zv[0], zv[1], zv[2]);
#pragma unroll
      for (int c = 0; c < 3; ++c) a.z[i + c * cs] = zv[c];
      if (a.own[i]) acc += rv[0] * zv[0] + rv[1] * zv[1] + rv[2] * zv[2];
    }
    const double rzn = cluster_sum(acc, next_part(), sh, cl);
    beta = rz > 1e-300 ? rzn / rz : 0.0;
    rz = rzn;
  }
  if (gt == 0) *a.it_out = it;
}

struct CoarseSolver {
  CoarseArgs a{};
  int cl = 0;
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

template <bool B, bool F, bool Q>
static int coarse_attr(int* cl_out) {
  auto k = k_coarse_pcg<B, F, Q>;
  HHG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int cl = kClMax;
  for (; cl >= 2; cl >>= 1) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(kCT);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) == cudaSuccess && n >= 1) break;
    cudaGetLastError();
  }
  if (cl < 2) return fail(HHG_ECUDA, "coarse solver: no cluster configuration fits");
  *cl_out = cl;
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
  std::vector<std::vector<int32_t>> own_slots(ns);
  for (int e = 0; e < nt; ++e) {
    for (int q = 0; q < 10; ++q) {
      node[(size_t)q * nt + e] = tn[e][q];
      own_slots[tn[e][q]].push_back(q * nt + e);
    }
    for (int v = 0; v < 4; ++v) p1v[(size_t)v * nt + e] = tp[e][v];
  }
  // gather lists: a node in an interface/BC group sums the slots of every copy (group copy order), the same
  // list for all copies; any other node its own slots
  std::vector<int32_t> gmap(ns);
  HHG_CUDA(cudaMemcpy(gmap.data(), L.gmap2, ns * sizeof(int32_t), cudaMemcpyDeviceToHost));
  std::vector<int64_t> gptr(L.g2.n + 1), gcopy(L.g2.ncopy);
  if (L.g2.n > 0) {
    HHG_CUDA(cudaMemcpy(gptr.data(), L.g2.ptr, gptr.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
    HHG_CUDA(cudaMemcpy(gcopy.data(), L.g2.copy, gcopy.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
  }
  std::vector<int32_t> sb(ns), se(ns), slots;
  std::vector<int32_t> gfirst(L.g2.n, -1), glast(L.g2.n, -1);
  for (int64_t g = 0; g < L.g2.n; ++g) {
    gfirst[g] = (int32_t)slots.size();
    for (int64_t k = gptr[g]; k < gptr[g + 1]; ++k)
      for (int32_t sl : own_slots[gcopy[k]]) slots.push_back(sl);
    glast[g] = (int32_t)slots.size();
  }
  for (int64_t i = 0; i < ns; ++i) {
    if (gmap[i] >= 0) {
      sb[i] = gfirst[gmap[i]];
      se[i] = glast[gmap[i]];
    } else {
      sb[i] = (int32_t)slots.size();
      for (int32_t sl : own_slots[i]) slots.push_back(sl);
      se[i] = (int32_t)slots.size();
    }
  }
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
  if ((r = upload(c, node, &a.node)) || (r = upload(c, p1v, &a.p1)) || (r = upload(c, info, &a.info)) ||
      (r = upload(c, anc, &a.anc)) || (r = upload(c, sb, &a.sb)) || (r = upload(c, se, &a.se)) ||
      (r = upload(c, slots, &a.slot)))
    return bail(r);
  a.gmap = L.gmap2;
  a.kind = L.g2.kind;
  a.normal = L.g2.normal;
  a.bcn = L.bcn2;
  a.own = L.own2;
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
  c->blend = m->blend == HHG_BLEND_SHELL;
  c->full = form == HHG_VISC_FULL;
  c->etaq = T2 != nullptr;
  if (c->etaq && !c->full) return bail(fail(HHG_EINVAL, "coarse solver: quadrature-point viscosity needs the full form"));
#define HHG_CATTR(B, F, Q) r = coarse_attr<B, F, Q>(&c->cl);
  if (c->etaq) {
    if (c->blend) HHG_CATTR(true, true, true) else HHG_CATTR(false, true, true)
  } else if (c->blend) {
    if (c->full) HHG_CATTR(true, true, false) else HHG_CATTR(true, false, false)
  } else {
    if (c->full) HHG_CATTR(false, true, false) else HHG_CATTR(false, false, false)
  }
#undef HHG_CATTR
  if (r != HHG_OK) return bail(r);
  *out = c;
  return HHG_OK;
}

template <bool B, bool F, bool Q>
static int coarse_launch(CoarseSolver* c, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = c->cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(c->cl);
  cfg.blockDim = dim3(kCT);
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  HHG_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_pcg<B, F, Q>, c->a));
  count_launch();
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

int coarse_iterations(const CoarseSolver* c, int* out) {
  HHG_CUDA(cudaDeviceSynchronize());
  HHG_CUDA(cudaMemcpy(out, c->a.it_out, sizeof(int), cudaMemcpyDeviceToHost));
  return HHG_OK;
}

void coarse_destroy(CoarseSolver* c) { delete c; }

}  // namespace hhg
