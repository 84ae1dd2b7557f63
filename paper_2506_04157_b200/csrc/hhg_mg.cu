// GMG V-cycle for the A block (fig:ASolverStructure): Chebyshev smoothing with the
// inverse diagonal, P2 transfers with projections, coarse Jacobi-PCG (BASELINE
// config 3; replaces the paper's AMG-CG of P:443), power-iteration spectrum estimate.
// All scalars of the PCG stay on the device so the whole cycle can be captured in one CUDA graph.
#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <vector>

#include "hhg_internal.h"

namespace hhg {
int apply_op(const Mesh* m, int level, int mode, int form, const double* eta, double gamma, const double* u,
             const double* p, double* yu, double* yp, bool accumulate_u, cudaStream_t s);
int launch_pcg_dir(int64_t n, double* scal, const double* z, double* p, cudaStream_t s);

__global__ void k_recip(int64_t n, const double* __restrict__ d, double* __restrict__ o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = 1.0 / d[i];
}
__global__ void k_sub(int64_t n, const double* __restrict__ f, const double* __restrict__ t, double* __restrict__ r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = f[i] - t[i];
}
__global__ void k_scale_dinv(int64_t n, const double* __restrict__ t, const double* __restrict__ dinv,
                             double* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = dinv[i] * t[i];
}
__global__ void k_normalize(int64_t n, const double* __restrict__ sq, const double* __restrict__ z,
                            double* __restrict__ v) {
  const double inv = 1.0 / sqrt(*sq);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = z[i] * inv;
}
static inline unsigned vg(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)(b < 2368 ? (b < 1 ? 1 : b) : 2368);
}

static int64_t p2vec_len(const Mesh* m, int level) { return 3 * macro_count(m) * m->levels[level].npts2; }

// one Chebyshev sweep; x_is_zero lets the first residual skip A*0
static int cheb_sweep(const Mesh* m, int l, int form, const double* eta, const double* dinv, int degree, double lmin,
                      double lmax, const double* f, double* x, double* r, double* d, double* t, bool x_is_zero,
                      cudaStream_t s) {
  const Level& L = m->levels[l];
  const int64_t n = p2vec_len(m, l);
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  if (x_is_zero) {
    HHG_CUDA(cudaMemsetAsync(t, 0, n * sizeof(double), s));
  } else {
    HHG_TRY(apply_op(m, l, ELEM_A, form, eta, 0.0, x, nullptr, t, nullptr, false, s));
  }
  HHG_TRY(launch_cheb0(n, f, t, dinv, 1.0 / theta, r, d, s));
  HHG_TRY(launch_fixup(m, L, HHG_P2VEC, false, true, d, s));
  for (int k = 1; k <= degree; ++k) {
    if (k < degree) {
      HHG_TRY(apply_op(m, l, ELEM_A, form, eta, 0.0, d, nullptr, t, nullptr, false, s));
      const double rn = 1.0 / (2.0 * sigma - rho);
      HHG_TRY(launch_chebk(n, t, dinv, rn * rho, 2.0 * rn / delta, x, r, d, s));
      HHG_TRY(launch_fixup(m, L, HHG_P2VEC, false, true, d, s));
      rho = rn;
    } else {
      HHG_TRY(launch_axpby(n, 1.0, d, 1.0, x, s));
    }
  }
  return HHG_OK;
}

}  // namespace hhg

using namespace hhg;

struct hhg_mg {
  hhg_mesh* mesh = nullptr;
  hhg_mg_params prm{};
  struct Lv {
    double *x = nullptr, *f = nullptr, *r = nullptr, *d = nullptr, *t = nullptr, *dinv = nullptr, *p = nullptr;
    const double* eta = nullptr;
    const double* T2 = nullptr;   // P2 temperature: quadrature-point viscosity on this level (l <= l_eta)
    double lam = 0.0;
    uint8_t* fmask = nullptr;     // nodes updated by the fused smoother epilogue (launch_elem_epi), or nullptr
  };
  std::vector<Lv> lv;
  double* scal = nullptr;    // device scalars
  double* red = nullptr;     // this object's reduction scratch (dots never share it with other objects)
  bool fuse_fx = false;      // single rank: smoother / residual kernels do the interface sum of A's output
  CoarseSolver* ccs = nullptr;  // single rank: the coarse PCG as one cluster-resident kernel (hhg_coarse.cu)
  // redundant coarse solve (multi-rank, prm.coarse_redundant): the l_min problem of ALL macros on every
  // rank -- a single-rank mesh/hierarchy of the global macro mesh, the rank's local macro ids, global
  // coarse vectors (the agglomeration analogue of P:443)
  hhg_mesh* cmesh = nullptr;
  hhg_mg* cmg = nullptr;
  int64_t* cids = nullptr;   // device: global id of every local macro
  double *cf = nullptr, *cx = nullptr, *ceta = nullptr, *cT2 = nullptr;
  double* hbuf_rhs = nullptr;  // device staging for vcycle_host
  double* hbuf_x = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const double* g_rhs = nullptr;
  double* g_x = nullptr;
  cudaStream_t g_stream = nullptr;
  // A-block CG (hhg_ablock_cg): fine-level work vectors + its own V-cycle graph (r -> z)
  double *cg_r = nullptr, *cg_z = nullptr, *cg_p = nullptr, *cg_q = nullptr, *cg_s = nullptr;
  cudaGraphExec_t cg_gexec = nullptr;
  cudaStream_t cg_stream = nullptr;
  // vcycle_host_batch: double-buffered staging, copy streams, per-buffer graphs and events
  double *st_in[2] = {nullptr, nullptr}, *st_out[2] = {nullptr, nullptr};
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in_ready[2] = {}, ev_in_free[2] = {}, ev_out_ready[2] = {}, ev_out_free[2] = {}, ev_start = nullptr,
              ev_done = nullptr;
  cudaGraphExec_t pipe_gexec[2] = {nullptr, nullptr};
  cudaStream_t pipe_stream = nullptr;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  double apply_ms = 0, cycle_ms = 0, dense_ms = 0;  // dense_ms: k_elem_fp over the dense bricks alone
  int64_t apply_n = 0, cycle_n = 0;
  ~hhg_mg() {
    for (auto& L : lv) {
      for (double* p : {L.x, L.f, L.r, L.d, L.t, L.dinv, L.p})
        if (p) cudaFree(p);
      if (L.fmask) cudaFree(L.fmask);
    }
    if (scal) cudaFree(scal);
    if (red) cudaFree(red);
    if (cmg) delete cmg;
    if (cmesh) delete cmesh;
    for (void* p : {(void*)cids, (void*)cf, (void*)cx, (void*)ceta, (void*)cT2})
      if (p) cudaFree(p);
    if (mesh) --mesh->dependents;
    if (ccs) coarse_destroy(ccs);
    if (hbuf_rhs) cudaFree(hbuf_rhs);
    if (hbuf_x) cudaFree(hbuf_x);
    if (gexec) cudaGraphExecDestroy(gexec);
    for (double* p : {cg_r, cg_z, cg_p, cg_q, cg_s})
      if (p) cudaFree(p);
    if (cg_gexec) cudaGraphExecDestroy(cg_gexec);
    for (int b = 0; b < 2; ++b) {
      if (st_in[b]) cudaFree(st_in[b]);
      if (st_out[b]) cudaFree(st_out[b]);
      if (pipe_gexec[b]) cudaGraphExecDestroy(pipe_gexec[b]);
      for (cudaEvent_t e : {ev_in_ready[b], ev_in_free[b], ev_out_ready[b], ev_out_free[b]})
        if (e) cudaEventDestroy(e);
    }
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_done) cudaEventDestroy(ev_done);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    for (auto e : ev) cudaEventDestroy(e);
  }
};

static int mg_apply(hhg_mg* mg, int l, const double* u, double* y, cudaStream_t s, bool y_zeroed = false,
                    bool fixup = true, int epi = EPI_NONE, const ChebEpi* ep = nullptr) {
  const bool timed = mg->prof && l == mg->prm.l_max;
  if (timed) {
    if (mg->ev_used + 3 > mg->ev.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        HHG_CUDA(cudaEventCreate(&e));
        mg->ev.push_back(e);
      }
    }
  }
  // y = (M P_v) A u : zero, element kernel (timed alone when profiling), interface sum + BC
  const Level& L = mg->mesh->levels[l];
  if (!y_zeroed) HHG_CUDA(cudaMemsetAsync(y, 0, p2vec_len(mg->mesh, l) * sizeof(double), s));
  if (timed) {
    HHG_CUDA(cudaEventRecord(mg->ev[mg->ev_used], s));
    g_elem_mid_event = mg->ev[mg->ev_used + 1];
  }
  if (mg->lv[l].T2)
    HHG_TRY(launch_elem_qeta(mg->mesh, L, ELEM_A, mg->lv[l].T2, mg->prm.qeta_lnC, mg->prm.qeta_jump, mg->prm.qeta_rjump,
                             u, y, s));
  else if (epi != EPI_NONE)
    HHG_TRY(launch_elem_epi(mg->mesh, L, epi, *ep, mg->lv[l].eta, u, y, s));
  else
    HHG_TRY(launch_elem(mg->mesh, L, ELEM_A, mg->prm.visc_form, mg->lv[l].eta, 0.0, u, nullptr, y, nullptr, s));
  if (timed) {
    if (g_elem_mid_event) {  // no separate sparse launch (deterministic mode, HHG_NO_SPLIT): dense = the whole
      HHG_CUDA(cudaEventRecord(g_elem_mid_event, s));
      g_elem_mid_event = nullptr;
    }
    HHG_CUDA(cudaEventRecord(mg->ev[mg->ev_used + 2], s));
    mg->ev_used += 3;
  }
  if (!fixup) return HHG_OK;  // the consumer sums the interface copies itself (launch_*_fx)
  return launch_fixup(mg->mesh, L, HHG_P2VEC, true, true, y, s);
}

static int mg_cheb(hhg_mg* mg, int l, double* x, const double* f, bool x_is_zero, cudaStream_t s) {
  // Chebyshev sweep of degree k on D^-1 A over [b/10, b] (R12).  Vector updates fused:
  // the first step skips A x when x = 0, the last step folds "x += d" into the d-update and drops the
  // dead r/d writes, and every direction update applies the BC projection P_v M per node (no
  // separate BC pass).
  auto& L = mg->lv[l];
  const Mesh* m = mg->mesh;
  const double b = mg->prm.cheb_hi_factor * L.lam, a = mg->prm.cheb_lo_ratio * b;
  const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  const Level& LL = m->levels[l];
  const bool fx = mg->fuse_fx;  // consumers sum the interface copies of A's raw output themselves
  // smoother updates of brick-interior nodes fused into the element kernel's write-out (launch_elem_epi)
  const uint8_t* sk = fx ? L.fmask : nullptr;
  const int deg = mg->prm.degree;
  const double* t0 = nullptr;
  if (!x_is_zero) {
    const ChebEpi e0{f, x, L.r, L.d, L.dinv, 1.0 / theta, 0.0};
    HHG_TRY(mg_apply(mg, l, x, L.t, s, false, !fx, (sk && deg > 1) ? EPI_CHEB0 : EPI_NONE, &e0));
    t0 = L.t;
  }
  if (deg == 1)
    return fx && t0 ? launch_cheb_deg1_fx(m, LL, f, t0, L.dinv, 1.0 / theta, x, s)
                    : launch_cheb_deg1_bc(m, LL, f, t0, L.dinv, 1.0 / theta, x, s);
  if (fx && t0) HHG_TRY(launch_cheb0_fx(m, LL, f, t0, L.dinv, 1.0 / theta, L.r, L.d, s, sk));
  else HHG_TRY(launch_cheb0_bc(m, LL, f, t0, L.dinv, 1.0 / theta, L.r, L.d, s));
  for (int k = 1; k < deg; ++k) {
    const double rn = 1.0 / (2.0 * sigma - rho);
    const bool last = k == deg - 1;
    const ChebEpi ek{f, x, L.r, L.d, L.dinv, rn * rho, 2.0 * rn / delta};
    HHG_TRY(mg_apply(mg, l, L.d, L.t, s, false, !fx, sk ? (last ? EPI_CHEBK_LAST : EPI_CHEBK) : EPI_NONE, &ek));
    if (fx) {
      if (!last) HHG_TRY(launch_chebk_fx(m, LL, L.t, L.dinv, rn * rho, 2.0 * rn / delta, x, L.r, L.d, s, sk));
      else HHG_TRY(launch_chebk_last_fx(m, LL, L.t, L.dinv, rn * rho, 2.0 * rn / delta, L.r, L.d, x, s, sk));
    } else {
      if (!last) HHG_TRY(launch_chebk_bc(m, LL, L.t, L.dinv, rn * rho, 2.0 * rn / delta, x, L.r, L.d, s));
      else HHG_TRY(launch_chebk_last_bc(m, LL, L.t, L.dinv, rn * rho, 2.0 * rn / delta, L.r, L.d, x, s));
    }
    rho = rn;
  }
  return HHG_OK;
}

static int mg_pcg(hhg_mg* mg, int l, const double* f, double* x, cudaStream_t s) {
  // Jacobi-PCG, exactly coarse_iters iterations from x = 0 (R15).  Scalars stay on the
  // device (graph-capturable); r.z ping-pongs between scal[0] and scal[2]; p = z + beta p also
  // zeroes q for the next operator application.
  auto& L = mg->lv[l];
  const Mesh* m = mg->mesh;
  const Level& LL = m->levels[l];
  const int64_t n = p2vec_len(m, l);
  double* r = L.r;
  double* z = L.d;
  double* p = L.p;
  double* q = L.t;
  if (mg->ccs) return coarse_run(mg->ccs, f, x, r, z, p, q, mg->prm.coarse_iters, mg->prm.coarse_tol, s);
  HHG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  HHG_TRY(launch_cheb0_bc(m, LL, f, nullptr, L.dinv, 1.0, r, z, s));  // r = f, z = PM dinv r
  HHG_CUDA(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  HHG_TRY(launch_dot_fused(m, LL, HHG_P2VEC, r, z, mg->scal + 0, s, mg->red));
  HHG_CUDA(cudaMemsetAsync(q, 0, n * sizeof(double), s));
  for (int it = 0; it < mg->prm.coarse_iters; ++it) {
    HHG_TRY(mg_apply(mg, l, p, q, s, true));
    HHG_TRY(launch_dot_fused(m, LL, HHG_P2VEC, p, q, mg->scal + 1, s, mg->red));
    if (mg->fuse_fx) {  // single rank: the new r.z comes out of the update kernel
      HHG_TRY(launch_pcg_update_bc_dot(m, LL, it, mg->scal, x, r, p, q, L.dinv, z, mg->red, s));
    } else {
      HHG_TRY(launch_pcg_update_bc(m, LL, it, mg->scal, x, r, p, q, L.dinv, z, s));
      HHG_TRY(launch_dot_fused(m, LL, HHG_P2VEC, r, z, mg->scal + ((it & 1) ? 0 : 2), s, mg->red));
    }
    HHG_TRY(launch_pcg_dir_zero(n, it, mg->scal, z, p, q, s));
  }
  return HHG_OK;
}

// copy between a rank's macro-local layout and the global macro layout of the coarse mesh (nc
// components of per-macro lattices with npts points; component strides cs_loc / cs_glob)
__global__ void k_macro_copy(int64_t nloc, int64_t npts, int nc, const int64_t* __restrict__ ids, int64_t cs_loc,
                             int64_t cs_glob, const double* __restrict__ src, double* __restrict__ dst, int to_global) {
  const int64_t n = nloc * npts;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * nc; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / n, r = i - c * n, t = r / npts, k = r - t * npts;
    const int64_t lo = c * cs_loc + t * npts + k, gl = c * cs_glob + ids[t] * npts + k;
    if (to_global) dst[gl] = src[lo];
    else dst[lo] = src[gl];
  }
}
// local -> global (zero padding, then a sum over ranks: every macro lives on exactly one rank)
static int coarse_gather(hhg_mg* mg, int l, int nc, int64_t npts, const double* loc, double* glob, cudaStream_t s) {
  const int64_t nl = macro_count(mg->mesh), ng = mg->mesh->n_tets;
  HHG_CUDA(cudaMemsetAsync(glob, 0, nc * ng * npts * sizeof(double), s));
  if (nl > 0) {
    k_macro_copy<<<vg(nl * npts * nc), 256, 0, s>>>(nl, npts, nc, mg->cids, nl * npts, ng * npts, loc, glob, 1);
    count_launch();
  }
  return comm_allreduce_sum(mg->mesh->comm, glob, nc * ng * npts, s);
}
static int coarse_scatter(hhg_mg* mg, int nc, int64_t npts, const double* glob, double* loc, cudaStream_t s) {
  const int64_t nl = macro_count(mg->mesh), ng = mg->mesh->n_tets;
  if (nl == 0) return HHG_OK;
  k_macro_copy<<<vg(nl * npts * nc), 256, 0, s>>>(nl, npts, nc, mg->cids, nl * npts, ng * npts, glob, loc, 0);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

static int mg_cycle(hhg_mg* mg, int l, const double* f, double* x, cudaStream_t s) {
  if (l == mg->prm.l_min && mg->cmg) {  // redundant coarse solve: gather, solve the global problem, scatter
    const int64_t np2 = mg->mesh->levels[l].npts2;
    HHG_TRY(coarse_gather(mg, l, 3, np2, f, mg->cf, s));
    HHG_TRY(mg_cycle(mg->cmg, l, mg->cf, mg->cx, s));
    return coarse_scatter(mg, 3, np2, mg->cx, x, s);
  }
  if (l == mg->prm.l_min) return mg_pcg(mg, l, f, x, s);
  auto& L = mg->lv[l];
  const Mesh* m = mg->mesh;
  const int64_t n = p2vec_len(m, l);
  HHG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  for (int i = 0; i < mg->prm.pre; ++i) HHG_TRY(mg_cheb(mg, l, x, f, i == 0, s));
  // r = f - A x  (into L.r), restrict into f_{l-1}
  if (mg->fuse_fx) {
    const ChebEpi er{f, x, L.r, L.d, L.dinv, 0.0, 0.0};
    HHG_TRY(mg_apply(mg, l, x, L.t, s, false, false, L.fmask ? EPI_SUB : EPI_NONE, &er));
    HHG_TRY(launch_sub_fx(m, m->levels[l], f, L.t, L.r, s, L.fmask));
  } else {
    HHG_TRY(mg_apply(mg, l, x, L.t, s));
    k_sub<<<vg(n), 256, 0, s>>>(n, f, L.t, L.r);
    count_launch();
  }
  auto& C = mg->lv[l - 1];
  HHG_TRY(p2_restrict(mg->mesh, l, L.r, C.f, (hhg_stream_t)s));
  HHG_TRY(mg_cycle(mg, l - 1, C.f, C.x, s));
  HHG_TRY(p2_prolong(mg->mesh, l - 1, C.x, x, (hhg_stream_t)s));
  for (int i = 0; i < mg->prm.post; ++i) HHG_TRY(mg_cheb(mg, l, x, f, false, s));
  return HHG_OK;
}

// power iteration of hhg_power_iteration with the hierarchy's own operator (quadrature-point
// viscosity levels): w = P_v M D^-1 A v, lambda = |w|, v = w / lambda
static int mg_power(hhg_mg* mg, int l, double* v0, double* lam) {
  auto& L = mg->lv[l];
  const Mesh* m = mg->mesh;
  const Level& LL = m->levels[l];
  const int64_t n = p2vec_len(m, l);
  cudaStream_t s = nullptr;
  HHG_TRY(launch_fixup(m, LL, HHG_P2VEC, false, true, v0, s));
  for (int it = 0; it < mg->prm.power_iters; ++it) {
    HHG_TRY(mg_apply(mg, l, v0, L.t, s));
    k_scale_dinv<<<vg(n), 256, 0, s>>>(n, L.t, L.dinv, L.t);
    count_launch();
    HHG_TRY(launch_fixup(m, LL, HHG_P2VEC, false, true, L.t, s));
    HHG_TRY(launch_dot(m, LL, HHG_P2VEC, L.t, L.t, mg->scal + 8, s, mg->red));
    k_normalize<<<vg(n), 256, 0, s>>>(n, mg->scal + 8, L.t, v0);
    count_launch();
  }
  double h = 0;
  HHG_CUDA(cudaMemcpy(&h, mg->scal + 8, sizeof(double), cudaMemcpyDeviceToHost));
  if (!(h > 0) || !std::isfinite(h)) return fail(HHG_EZEROOP, "power iteration on a zero operator");
  *lam = std::sqrt(h);
  return HHG_OK;
}

extern "C" {

int hhg_mg_create(hhg_mesh* mesh, const hhg_mg_params* params, const double* const* eta_per_level,
                  double* const* power_v0, hhg_mg** out) {
  return hhg_mg_create_qeta(mesh, params, eta_per_level, nullptr, power_v0, out);
}

int hhg_mg_create_qeta(hhg_mesh* mesh, const hhg_mg_params* params, const double* const* eta_per_level,
                       const double* const* T2_per_level, double* const* power_v0, hhg_mg** out) {
  if (!mesh || !params || !out) return fail(HHG_EINVAL, "hhg_mg_create: NULL argument");
  const hhg_mg_params& P = *params;
  if (P.l_min < 0 || P.l_max > mesh->level_max || P.l_min > P.l_max)
    return fail(HHG_ELEVEL, "hhg_mg_create: need 0 <= l_min <= l_max <= level_max");
  if (P.degree < 1 || P.pre < 0 || P.post < 0 || P.coarse_iters < 0 || P.power_iters < 1 || !(P.coarse_tol >= 0.0))
    return fail(HHG_EINVAL, "hhg_mg_create: bad smoother parameters");
  auto* mg = new hhg_mg();
  mg->mesh = mesh;
  mg->prm = P;
  mg->lv.resize(P.l_max + 1);
  auto bail = [&](int code) {
    delete mg;
    return code;
  };
  ++mesh->dependents;
  {
    const char* e = getenv("HHG_NO_FX");  // A/B switch for measurements
    mg->fuse_fx = mesh->nranks == 1 && !(e && e[0] == '1');
  }
  if (cudaMalloc(&mg->scal, 16 * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "scal"));
  if (red_alloc(&mg->red) != HHG_OK) return bail(HHG_ENOMEM);
  for (int l = P.l_min; l <= P.l_max; ++l) {
    int r = ensure_level(mesh, l);
    if (r != HHG_OK) return bail(r);
    const int64_t n = p2vec_len(mesh, l);
    auto& L = mg->lv[l];
    L.eta = eta_per_level ? eta_per_level[l] : nullptr;
    if (T2_per_level && l <= P.l_eta) {
      if (!T2_per_level[l]) return bail(fail(HHG_EINVAL, "hhg_mg_create_qeta: T2_per_level[l] missing"));
      if (P.visc_form != HHG_VISC_FULL) return bail(fail(HHG_EINVAL, "hhg_mg_create_qeta: full form only"));
      L.T2 = T2_per_level[l];
    }
    for (double** p : {&L.x, &L.f, &L.r, &L.d, &L.t, &L.dinv})
      if (cudaMalloc(p, n * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "mg vectors"));
    if (l == P.l_min && cudaMalloc(&L.p, n * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "mg p"));
    // diag(A) without P_v -> D^-1
    if (L.T2)
      r = hhg_diag_qeta(mesh, l, L.T2, P.qeta_lnC, P.qeta_jump, P.qeta_rjump, L.t, nullptr);
    else
      r = apply_op(mesh, l, ELEM_DIAG, P.visc_form, L.eta, 0.0, nullptr, nullptr, L.t, nullptr, false, 0);
    if (r != HHG_OK) return bail(r);
    k_recip<<<vg(n), 256>>>(n, L.t, L.dinv);
    count_launch();
    if (l > P.l_min) {
      if (!power_v0 || !power_v0[l]) return bail(fail(HHG_EINVAL, "hhg_mg_create: power_v0[l] missing"));
      r = L.T2 ? mg_power(mg, l, power_v0[l], &L.lam)
               : hhg_power_iteration(mesh, l, L.eta, L.dinv, P.power_iters, power_v0[l], &L.lam, nullptr);
      if (r != HHG_OK) return bail(r);
    }
  }
  {
    // fused smoother epilogue: single rank (interface sums in the consumers), atomic element kernels, full form,
    // P1 viscosity levels above l_min
    // Opt-in (HHG_EPI=1): measured SLOWER at L5 (V(3,3) 39.6 ms fused vs 25.8 ms unfused, profiles/r02_epi_ab.jsonl):
    // the write-out's per-point read-modify-write of f, r, d, x, D^-1 serialises DRAM round trips inside a CTA that
    // holds 43 KB of shared memory, and the *_fx consumers still stream every node (mask test) -- DESIGN.md §6.
    const char* e = getenv("HHG_EPI");
    if (mg->fuse_fx && !mesh->deterministic && P.visc_form == HHG_VISC_FULL && e && e[0] == '1')
      for (int l = P.l_min + 1; l <= P.l_max; ++l)
        if (!mg->lv[l].T2) {
          const int r = elem_fused_mask(mesh, mesh->levels[l], &mg->lv[l].fmask);
          if (r != HHG_OK) return bail(r);
        }
  }
  {
    const char* e = getenv("HHG_NO_CCL");  // A/B switch: the coarse PCG through the generic launches
    if (mg->fuse_fx && !mesh->comm && !(e && e[0] == '1')) {
      auto& C = mg->lv[P.l_min];
      const int r = coarse_create(mesh, P.l_min, P.visc_form, C.eta, C.T2, P.qeta_lnC, P.qeta_jump, P.qeta_rjump,
                                  C.dinv, &mg->ccs);
      // a coarse level too large for one cluster keeps the generic path (unless a tolerance needs the kernel)
      if (r != HHG_OK && !(r == HHG_ENOMEM && P.coarse_tol == 0.0)) return bail(r);
    }
  }
  if (P.coarse_tol > 0.0 && !mg->ccs && !(P.coarse_redundant && mesh->nranks > 1))
    return bail(fail(HHG_EINVAL, "hhg_mg_create: coarse_tol > 0 needs the cluster-resident coarse solver "
                                 "(single-rank mesh or coarse_redundant)"));
  if (P.coarse_redundant && mesh->nranks > 1) {
    // the coarse level of all macros on every rank: global mesh (no communicator), global eta (and T2)
    const int lc = P.l_min;
    hhg_mesh* cm = nullptr;
    int r = hhg_mesh_create(mesh->xyz.data(), mesh->n_vert, mesh->tets.data(), mesh->n_tets, mesh->vtag.data(), lc,
                            nullptr, nullptr, &cm);
    if (r != HHG_OK) return bail(r);
    mg->cmesh = cm;
    cm->blend = mesh->blend;
    for (int i = 0; i < 3; ++i) cm->bc_kind[i] = mesh->bc_kind[i];
    cm->deterministic = mesh->deterministic;
    cm->dgeo_dirty = true;
    if ((r = mesh_set_geometry(cm)) != HHG_OK || (r = ensure_level(cm, lc)) != HHG_OK) return bail(r);
    std::vector<int64_t> ids(mesh->local.begin(), mesh->local.end());
    if (cudaMalloc(&mg->cids, std::max<size_t>(ids.size(), 1) * sizeof(int64_t)) != cudaSuccess)
      return bail(fail(HHG_ENOMEM, "coarse ids"));
    if (!ids.empty() && cudaMemcpy(mg->cids, ids.data(), ids.size() * sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(HHG_ECUDA, "coarse ids"));
    const Level& LC = cm->levels[lc];
    const int64_t ng = mesh->n_tets;
    for (double** p : {&mg->cf, &mg->cx})
      if (cudaMalloc(p, 3 * ng * LC.npts2 * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "coarse vectors"));
    const double* ce = nullptr;
    if (mg->lv[lc].eta) {
      if (cudaMalloc(&mg->ceta, ng * LC.npts1 * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "coarse eta"));
      if ((r = coarse_gather(mg, lc, 1, LC.npts1, mg->lv[lc].eta, mg->ceta, 0)) != HHG_OK) return bail(r);
      ce = mg->ceta;
    }
    const double* ct = nullptr;
    if (mg->lv[lc].T2) {
      if (cudaMalloc(&mg->cT2, ng * LC.npts2 * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "coarse T2"));
      if ((r = coarse_gather(mg, lc, 1, LC.npts2, mg->lv[lc].T2, mg->cT2, 0)) != HHG_OK) return bail(r);
      ct = mg->cT2;
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(HHG_ECUDA, "coarse gather"));
    hhg_mg_params cp = P;
    cp.l_max = lc;
    cp.coarse_redundant = 0;
    std::vector<const double*> etas(lc + 1, nullptr), t2s(lc + 1, nullptr);
    etas[lc] = ce;
    t2s[lc] = ct;
    r = ct ? hhg_mg_create_qeta(cm, &cp, etas.data(), t2s.data(), nullptr, &mg->cmg)
           : hhg_mg_create(cm, &cp, etas.data(), nullptr, &mg->cmg);
    if (r != HHG_OK) return bail(r);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(HHG_ECUDA, "hhg_mg_create: sync failed"));
  *out = mg;
  return HHG_OK;
}

int hhg_mg_coarse_iterations(const hhg_mg* mg, int* iters_out) {
  if (!mg || !iters_out) return fail(HHG_EINVAL, "NULL argument");
  if (mg->cmg) return hhg_mg_coarse_iterations(mg->cmg, iters_out);
  if (!mg->ccs) return fail(HHG_EINVAL, "hhg_mg_coarse_iterations: the coarse level runs the generic PCG");
  return coarse_iterations(mg->ccs, iters_out);
}

int hhg_mg_lambda(const hhg_mg* mg, int level, double* lambda_host) {
  if (!mg || !lambda_host) return fail(HHG_EINVAL, "NULL argument");
  if (level < mg->prm.l_min || level > mg->prm.l_max) return fail(HHG_ELEVEL, "level outside hierarchy");
  *lambda_host = mg->lv[level].lam;
  return HHG_OK;
}

int vcycle(hhg_mg* mg, const double* rhs, double* x, hhg_stream_t stream) {
  if (!mg || !rhs || !x) return fail(HHG_EINVAL, "vcycle: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  for (int l = mg->prm.l_min + 1; l <= mg->prm.l_max; ++l)
    if (!(mg->lv[l].lam > 0)) return fail(HHG_ENOTREADY, "vcycle: no spectrum estimate");
  const bool use_graph = mg->prm.use_graph && s != nullptr && !mg->prof && comm_capturable(mg->mesh->comm);
  if (!use_graph) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (mg->prof) {
      if (mg->ev_used + 2 > mg->ev.size())
        for (int i = 0; i < 64; ++i) {
          cudaEvent_t e;
          HHG_CUDA(cudaEventCreate(&e));
          mg->ev.push_back(e);
        }
      e0 = mg->ev[mg->ev_used];
      e1 = mg->ev[mg->ev_used + 1];
      mg->ev_used += 2;
      HHG_CUDA(cudaEventRecord(e0, s));
    }
    size_t first_apply_ev = mg->ev_used;
    HHG_TRY(mg_cycle(mg, mg->prm.l_max, rhs, x, s));
    if (mg->prof) {
      HHG_CUDA(cudaEventRecord(e1, s));
      HHG_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      HHG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      mg->cycle_ms += ms;
      mg->cycle_n += 1;
      for (size_t i = first_apply_ev; i + 2 < mg->ev_used; i += 3) {  // [start, after the dense launch, end]
        HHG_CUDA(cudaEventElapsedTime(&ms, mg->ev[i], mg->ev[i + 2]));
        mg->apply_ms += ms;
        HHG_CUDA(cudaEventElapsedTime(&ms, mg->ev[i], mg->ev[i + 1]));
        mg->dense_ms += ms;
        mg->apply_n += 1;
      }
      mg->ev_used = 0;
    }
    return HHG_OK;
  }
  if (!mg->gexec || mg->g_rhs != rhs || mg->g_x != x || mg->g_stream != s) {
    if (mg->gexec) cudaGraphExecDestroy(mg->gexec);
    mg->gexec = nullptr;
    cudaGraph_t g;
    HHG_TRY(elem_side_prepare(mg->mesh, s));  // the element launcher forks its sparse launch: side stream before capture
    HHG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int r = mg_cycle(mg, mg->prm.l_max, rhs, x, s);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (r != HHG_OK) return r;
    if (ce != cudaSuccess) return fail(HHG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    HHG_CUDA(cudaGraphInstantiate(&mg->gexec, g, 0));
    cudaGraphDestroy(g);
    mg->g_rhs = rhs;
    mg->g_x = x;
    mg->g_stream = s;
  }
  HHG_CUDA(cudaGraphLaunch(mg->gexec, s));
  count_launch();
  return HHG_OK;
}

// ---- A-block solver: CG preconditioned by one V-cycle per iteration, to a relative
// residual tolerance tol_A.  x = 0 on entry; rhs consistent and BC-projected.
__global__ void k_cg_step(int64_t n, const double* __restrict__ sc, double* __restrict__ x, double* __restrict__ r,
                          const double* __restrict__ p, const double* __restrict__ q) {
  const double alpha = sc[1] != 0.0 ? sc[0] / sc[1] : 0.0;  // sc[0] = r.z, sc[1] = p.q
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * q[i];
  }
}
__global__ void k_cg_dir(int64_t n, double* __restrict__ sc, const double* __restrict__ z, double* __restrict__ p) {
  const double beta = sc[0] != 0.0 ? sc[2] / sc[0] : 0.0;  // sc[2] = new r.z
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}
__global__ void k_cg_roll(double* sc) {
  if (threadIdx.x == 0) sc[0] = sc[2];
}

static int cg_precond(hhg_mg* mg, cudaStream_t s) {  // z = V(r) with a cached graph
  if (!mg->prm.use_graph || s == nullptr || !comm_capturable(mg->mesh->comm))
    return mg_cycle(mg, mg->prm.l_max, mg->cg_r, mg->cg_z, s);
  if (!mg->cg_gexec || mg->cg_stream != s) {
    if (mg->cg_gexec) cudaGraphExecDestroy(mg->cg_gexec);
    mg->cg_gexec = nullptr;
    cudaGraph_t g;
    HHG_TRY(elem_side_prepare(mg->mesh, s));  // the element launcher forks its sparse launch: side stream before capture
    HHG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int r = mg_cycle(mg, mg->prm.l_max, mg->cg_r, mg->cg_z, s);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (r != HHG_OK) return r;
    if (ce != cudaSuccess) return fail(HHG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    HHG_CUDA(cudaGraphInstantiate(&mg->cg_gexec, g, 0));
    cudaGraphDestroy(g);
    mg->cg_stream = s;
  }
  HHG_CUDA(cudaGraphLaunch(mg->cg_gexec, s));
  count_launch();
  return HHG_OK;
}

int hhg_ablock_cg(hhg_mg* mg, const double* rhs, double* x, double tol, int max_iters, int* iters_out,
                  double* rel_res_out, hhg_stream_t stream) {
  if (!mg || !rhs || !x) return fail(HHG_EINVAL, "hhg_ablock_cg: NULL argument");
  if (!(tol > 0) || max_iters < 1) return fail(HHG_EINVAL, "hhg_ablock_cg: need tol > 0, max_iters >= 1");
  for (int l = mg->prm.l_min + 1; l <= mg->prm.l_max; ++l)
    if (!(mg->lv[l].lam > 0)) return fail(HHG_ENOTREADY, "hhg_ablock_cg: no spectrum estimate");
  cudaStream_t s = (cudaStream_t)stream;
  const int l = mg->prm.l_max;
  const Mesh* m = mg->mesh;
  const Level& LL = m->levels[l];
  const int64_t n = p2vec_len(m, l);
  if (!mg->cg_r) {
    for (double** p : {&mg->cg_r, &mg->cg_z, &mg->cg_p, &mg->cg_q})
      if (cudaMalloc(p, n * sizeof(double)) != cudaSuccess) return fail(HHG_ENOMEM, "hhg_ablock_cg workspace");
    if (cudaMalloc(&mg->cg_s, 8 * sizeof(double)) != cudaSuccess) return fail(HHG_ENOMEM, "hhg_ablock_cg scalars");
  }
  double* sc = mg->cg_s;  // [0] r.z  [1] p.q  [2] r.z new  [3] r.r  [4] r0.r0
  HHG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  HHG_CUDA(cudaMemcpyAsync(mg->cg_r, rhs, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  HHG_TRY(launch_dot(m, LL, HHG_P2VEC, mg->cg_r, mg->cg_r, sc + 4, s, mg->red));
  double r00 = 0.0;
  HHG_CUDA(cudaMemcpyAsync(&r00, sc + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
  HHG_CUDA(cudaStreamSynchronize(s));
  const double r0 = std::sqrt(r00);
  int it = 0;
  double rel = r0 > 0 ? 1.0 : 0.0;
  if (r0 > 0) {
    HHG_TRY(cg_precond(mg, s));
    HHG_CUDA(cudaMemcpyAsync(mg->cg_p, mg->cg_z, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    HHG_TRY(launch_dot(m, LL, HHG_P2VEC, mg->cg_r, mg->cg_z, sc + 0, s, mg->red));
    const unsigned nb = vg(n);
    while (it < max_iters) {
      ++it;
      HHG_TRY(mg_apply(mg, l, mg->cg_p, mg->cg_q, s));
      HHG_TRY(launch_dot(m, LL, HHG_P2VEC, mg->cg_p, mg->cg_q, sc + 1, s, mg->red));
      k_cg_step<<<nb, 256, 0, s>>>(n, sc, x, mg->cg_r, mg->cg_p, mg->cg_q);
      count_launch();
      HHG_TRY(launch_dot(m, LL, HHG_P2VEC, mg->cg_r, mg->cg_r, sc + 3, s, mg->red));
      double rr = 0.0;
      HHG_CUDA(cudaMemcpyAsync(&rr, sc + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
      HHG_CUDA(cudaStreamSynchronize(s));
      rel = std::sqrt(std::max(rr, 0.0)) / r0;
      if (rel <= tol) break;
      HHG_TRY(cg_precond(mg, s));
      HHG_TRY(launch_dot(m, LL, HHG_P2VEC, mg->cg_r, mg->cg_z, sc + 2, s, mg->red));
      k_cg_dir<<<nb, 256, 0, s>>>(n, sc, mg->cg_z, mg->cg_p);
      k_cg_roll<<<1, 32, 0, s>>>(sc);
      count_launch(2);
    }
  }
  HHG_CUDA(cudaGetLastError());
  if (iters_out) *iters_out = it;
  if (rel_res_out) *rel_res_out = rel;
  return HHG_OK;
}

int vcycle_host(hhg_mg* mg, const double* rhs_host, double* x_host, hhg_stream_t stream) {
  if (!mg || !rhs_host || !x_host) return fail(HHG_EINVAL, "vcycle_host: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = p2vec_len(mg->mesh, mg->prm.l_max);
  if (!mg->hbuf_rhs) {
    if (cudaMalloc(&mg->hbuf_rhs, n * sizeof(double)) != cudaSuccess) return fail(HHG_ENOMEM, "staging");
    if (cudaMalloc(&mg->hbuf_x, n * sizeof(double)) != cudaSuccess) return fail(HHG_ENOMEM, "staging");
  }
  HHG_CUDA(cudaMemcpyAsync(mg->hbuf_rhs, rhs_host, n * sizeof(double), cudaMemcpyHostToDevice, s));
  HHG_TRY(vcycle(mg, mg->hbuf_rhs, mg->hbuf_x, stream));
  HHG_CUDA(cudaMemcpyAsync(x_host, mg->hbuf_x, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  return HHG_OK;
}

// nsteps V-cycles on host buffers with the copies hidden behind the compute: H2D of step k+1 (copy
// stream) and D2H of step k-1 (second copy stream) overlap V-cycle k; two device staging pairs
// alternate, each with its own captured graph; events order reuse of a buffer pair.
int vcycle_host_batch(hhg_mg* mg, const double* const* rhs_host, double* const* x_host, int nsteps,
                      hhg_stream_t stream) {
  if (!mg || !rhs_host || !x_host || nsteps < 0) return fail(HHG_EINVAL, "vcycle_host_batch: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = p2vec_len(mg->mesh, mg->prm.l_max);
  const size_t nb = n * sizeof(double);
  if (!mg->st_in[0]) {
    for (int b = 0; b < 2; ++b) {
      if (cudaMalloc(&mg->st_in[b], nb) != cudaSuccess || cudaMalloc(&mg->st_out[b], nb) != cudaSuccess)
        return fail(HHG_ENOMEM, "vcycle_host_batch: staging");
      for (cudaEvent_t* e : {&mg->ev_in_ready[b], &mg->ev_in_free[b], &mg->ev_out_ready[b], &mg->ev_out_free[b]})
        HHG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    HHG_CUDA(cudaEventCreateWithFlags(&mg->ev_start, cudaEventDisableTiming));
    HHG_CUDA(cudaEventCreateWithFlags(&mg->ev_done, cudaEventDisableTiming));
    HHG_CUDA(cudaStreamCreateWithFlags(&mg->s_h2d, cudaStreamNonBlocking));
    HHG_CUDA(cudaStreamCreateWithFlags(&mg->s_d2h, cudaStreamNonBlocking));
  }
  for (int l = mg->prm.l_min + 1; l <= mg->prm.l_max; ++l)
    if (!(mg->lv[l].lam > 0)) return fail(HHG_ENOTREADY, "vcycle_host_batch: no spectrum estimate");
  const bool use_graph = mg->prm.use_graph && s != nullptr && !mg->prof && comm_capturable(mg->mesh->comm);
  if (use_graph && mg->pipe_stream != s) {
    for (int b = 0; b < 2; ++b) {
      if (mg->pipe_gexec[b]) cudaGraphExecDestroy(mg->pipe_gexec[b]);
      mg->pipe_gexec[b] = nullptr;
      cudaGraph_t g;
      HHG_TRY(elem_side_prepare(mg->mesh, s));  // the element launcher forks its sparse launch: side stream before capture
      HHG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      int r = mg_cycle(mg, mg->prm.l_max, mg->st_in[b], mg->st_out[b], s);
      cudaError_t ce = cudaStreamEndCapture(s, &g);
      if (r != HHG_OK) return r;
      if (ce != cudaSuccess) return fail(HHG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      HHG_CUDA(cudaGraphInstantiate(&mg->pipe_gexec[b], g, 0));
      cudaGraphDestroy(g);
    }
    mg->pipe_stream = s;
  }
  if (nsteps == 0) return HHG_OK;
  HHG_CUDA(cudaEventRecord(mg->ev_start, s));
  HHG_CUDA(cudaStreamWaitEvent(mg->s_h2d, mg->ev_start, 0));
  HHG_CUDA(cudaStreamWaitEvent(mg->s_d2h, mg->ev_start, 0));
  auto h2d = [&](int k) -> int {
    const int b = k & 1;
    if (k >= 2) HHG_CUDA(cudaStreamWaitEvent(mg->s_h2d, mg->ev_in_free[b], 0));
    HHG_CUDA(cudaMemcpyAsync(mg->st_in[b], rhs_host[k], nb, cudaMemcpyHostToDevice, mg->s_h2d));
    HHG_CUDA(cudaEventRecord(mg->ev_in_ready[b], mg->s_h2d));
    return HHG_OK;
  };
  HHG_TRY(h2d(0));
  for (int k = 0; k < nsteps; ++k) {
    const int b = k & 1;
    HHG_CUDA(cudaStreamWaitEvent(s, mg->ev_in_ready[b], 0));
    if (k >= 2) HHG_CUDA(cudaStreamWaitEvent(s, mg->ev_out_free[b], 0));
    if (use_graph) HHG_CUDA(cudaGraphLaunch(mg->pipe_gexec[b], s));
    else HHG_TRY(mg_cycle(mg, mg->prm.l_max, mg->st_in[b], mg->st_out[b], s));
    HHG_CUDA(cudaEventRecord(mg->ev_in_free[b], s));
    HHG_CUDA(cudaEventRecord(mg->ev_out_ready[b], s));
    if (k + 1 < nsteps) HHG_TRY(h2d(k + 1));
    HHG_CUDA(cudaStreamWaitEvent(mg->s_d2h, mg->ev_out_ready[b], 0));
    HHG_CUDA(cudaMemcpyAsync(x_host[k], mg->st_out[b], nb, cudaMemcpyDeviceToHost, mg->s_d2h));
    HHG_CUDA(cudaEventRecord(mg->ev_out_free[b], mg->s_d2h));
  }
  HHG_CUDA(cudaEventRecord(mg->ev_done, mg->s_d2h));
  HHG_CUDA(cudaStreamWaitEvent(s, mg->ev_done, 0));
  return HHG_OK;
}

int hhg_mg_profile(hhg_mg* mg, int enable) {
  if (!mg) return fail(HHG_EINVAL, "NULL mg");
  mg->prof = enable != 0;
  mg->apply_ms = mg->cycle_ms = mg->dense_ms = 0;
  mg->apply_n = mg->cycle_n = 0;
  mg->ev_used = 0;
  return HHG_OK;
}

int hhg_mg_profile_get(hhg_mg* mg, double* apply_ms_sum, int64_t* apply_count, double* cycle_ms_sum,
                       int64_t* cycle_count) {
  if (!mg) return fail(HHG_EINVAL, "NULL mg");
  if (apply_ms_sum) *apply_ms_sum = mg->apply_ms;
  if (apply_count) *apply_count = mg->apply_n;
  if (cycle_ms_sum) *cycle_ms_sum = mg->cycle_ms;
  if (cycle_count) *cycle_count = mg->cycle_n;
  return HHG_OK;
}

int hhg_mg_profile_get_dense(hhg_mg* mg, double* dense_ms_sum) {
  if (!mg || !dense_ms_sum) return fail(HHG_EINVAL, "NULL argument");
  *dense_ms_sum = mg->dense_ms;
  return HHG_OK;
}

int hhg_mg_destroy(hhg_mg* mg) {
  delete mg;
  return HHG_OK;
}

int chebyshev_smooth(const hhg_mesh* mesh, int level, const double* eta_p1, const double* dinv, int degree,
                     double lmin, double lmax, const double* rhs, double* x, double* work, hhg_stream_t stream) {
  if (!mesh || !dinv || !rhs || !x || !work) return fail(HHG_EINVAL, "chebyshev_smooth: NULL argument");
  if (level < 0 || level > mesh->level_max) return fail(HHG_ELEVEL, "level outside [0, level_max]");
  if (degree < 1) return fail(HHG_EINVAL, "degree must be >= 1");
  if (!(lmax > 0) || !(lmin >= 0) || !(lmin < lmax)) return fail(HHG_ENOTREADY, "chebyshev_smooth: bad spectrum");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  const int64_t n = p2vec_len(m, level);
  return cheb_sweep(m, level, HHG_VISC_FULL, eta_p1, dinv, degree, lmin, lmax, rhs, x, work, work + n, work + 2 * n,
                    false, (cudaStream_t)stream);
}

int hhg_power_iteration(const hhg_mesh* mesh, int level, const double* eta_p1, const double* dinv, int iters,
                        double* v0, double* lambda_host, hhg_stream_t stream) {
  if (!mesh || !dinv || !v0 || !lambda_host) return fail(HHG_EINVAL, "hhg_power_iteration: NULL argument");
  if (level < 0 || level > mesh->level_max) return fail(HHG_ELEVEL, "level outside [0, level_max]");
  if (iters < 1) return fail(HHG_EINVAL, "iters must be >= 1");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  cudaStream_t s = (cudaStream_t)stream;
  const Level& L = m->levels[level];
  const int64_t n = p2vec_len(m, level);
  double *t = nullptr, *sc = nullptr, *red = nullptr;
  if (cudaMalloc(&t, n * sizeof(double)) != cudaSuccess) return fail(HHG_ENOMEM, "power iteration workspace");
  if (cudaMalloc(&sc, sizeof(double)) != cudaSuccess || red_alloc(&red) != HHG_OK) {
    cudaFree(t);
    if (sc) cudaFree(sc);
    return fail(HHG_ENOMEM, "power iteration workspace");
  }
  int r = HHG_OK;
  auto run = [&]() -> int {
    HHG_TRY(launch_fixup(m, L, HHG_P2VEC, false, true, v0, s));
    for (int it = 0; it < iters; ++it) {
      HHG_TRY(apply_op(m, level, ELEM_A, HHG_VISC_FULL, eta_p1, 0.0, v0, nullptr, t, nullptr, false, s));
      k_scale_dinv<<<vg(n), 256, 0, s>>>(n, t, dinv, t);
      count_launch();
      HHG_TRY(launch_fixup(m, L, HHG_P2VEC, false, true, t, s));
      HHG_TRY(launch_dot(m, L, HHG_P2VEC, t, t, sc, s, red));
      k_normalize<<<vg(n), 256, 0, s>>>(n, sc, t, v0);
      count_launch();
    }
    double h = 0;
    HHG_CUDA(cudaMemcpyAsync(&h, sc, sizeof(double), cudaMemcpyDeviceToHost, s));
    HHG_CUDA(cudaStreamSynchronize(s));
    if (!(h > 0) || !std::isfinite(h)) return fail(HHG_EZEROOP, "power iteration on a zero operator");
    *lambda_host = std::sqrt(h);
    return HHG_OK;
  };
  r = run();
  cudaStreamSynchronize(s);
  cudaFree(t);
  cudaFree(sc);
  cudaFree(red);
  return r;
}

}  // extern "C"

// ================================================================ K_{1/sqrt(eta)} multigrid (w-BFBT, NEXT-3)
// The Poisson replacement of (B M_{sqrt(eta)}^-1 B^T)^-1 in eq:schurWBFBT: "an inverse viscosity scaled
// Poisson problem with Neumann boundary conditions ... CG solver preconditioned by a GMG approach"
// (P:470).  P1 levels l_min..l_max, Chebyshev(D^-1 K) smoothing as for A (R12), P1 linear
// transfers, coarse Jacobi-PCG (fixed iteration count, device scalars).  No constraints; the constant
// kernel is handled by projecting the outer CG's vectors to mean zero.
namespace {
// Counter-based start vector of the K power iteration, keyed by canonical node identity (the harness
// contract of SURVEY Appendix A2, implemented here independently of the input generators): the value at a
// node does not depend on the storage layout, the partition or the level, so any implementation of the
// method that keys its random numbers the same way draws the same start vector.
uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double keyed_uniform(const int64_t* key, uint64_t seed, int component) {
  int64_t w[5] = {key[5], key[6], key[7], key[8], key[9]};  // weights (0 padded) and resolution
  while (w[4] > 1 && !((w[0] | w[1] | w[2] | w[3] | w[4]) & 1))
    for (auto& x : w) x /= 2;
  const int dim = (int)key[0];
  uint64_t h = seed;
  h = splitmix64(h ^ (uint64_t)key[0]);
  for (int c = 0; c < 4; ++c) h = splitmix64(h ^ (uint64_t)(c <= dim ? key[1 + c] : 0));
  for (int c = 0; c < 4; ++c) h = splitmix64(h ^ (uint64_t)(c <= dim ? w[c] : 0));
  h = splitmix64(h ^ (uint64_t)w[4]);
  h = splitmix64(h ^ (uint64_t)component);
  return 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
}
// PCG step with ping-pong r.z scalars (scal[0] / scal[2] by iteration parity, scal[1] = p.q), no BC
__global__ void k_pcg_update_pp(int64_t n, int it, const double* __restrict__ scal, double* __restrict__ x,
                                double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ q,
                                const double* __restrict__ dinv, double* __restrict__ z) {
  const double rz = scal[(it & 1) ? 2 : 0], pq = scal[1];
  const double alpha = (rz > 1e-300 && pq != 0.0) ? rz / pq : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    z[i] = dinv[i] * ri;
  }
}
__global__ void k_shift(int64_t n, const double* __restrict__ sum, double inv_count, double* __restrict__ v) {
  const double m = *sum * inv_count;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] -= m;
}
}  // namespace

struct hhg_kmg {
  hhg_mesh* mesh = nullptr;
  hhg_mg_params prm{};
  double a = 1.0;
  struct Lv {
    double *x = nullptr, *f = nullptr, *r = nullptr, *d = nullptr, *t = nullptr, *dinv = nullptr, *p = nullptr;
    double* ones = nullptr;
    const double* eta = nullptr;
    double lam = 0.0, inv_count = 0.0;  // 1 / number of unique nodes
  };
  std::vector<Lv> lv;
  double* scal = nullptr;
  double* red = nullptr;  // reduction scratch of this object
  double *cr = nullptr, *cz = nullptr, *cp = nullptr, *cq = nullptr;  // outer CG (finest level)
  ~hhg_kmg() {
    if (mesh) --mesh->dependents;
    for (auto& L : lv)
      for (double* p : {L.x, L.f, L.r, L.d, L.t, L.dinv, L.p, L.ones})
        if (p) cudaFree(p);
    for (double* p : {scal, red, cr, cz, cp, cq})
      if (p) cudaFree(p);
  }
};

namespace {
int64_t p1_len(const Mesh* m, int l) { return macro_count(m) * m->levels[l].npts1; }
int km_apply(hhg_kmg* K, int l, const double* u, double* y, cudaStream_t s) {
  return surf_op(K->mesh, l, ELEM_KP1, K->lv[l].eta, K->a, u, y, s);
}
int km_mean0(hhg_kmg* K, int l, double* v, cudaStream_t s) {  // v -= mean over unique nodes (no sync)
  const Mesh* m = K->mesh;
  HHG_TRY(launch_dot_fused(m, m->levels[l], HHG_P1, v, K->lv[l].ones, K->scal + 6, s, K->red));
  const int64_t n = p1_len(m, l);
  k_shift<<<vg(n), 256, 0, s>>>(n, K->scal + 6, K->lv[l].inv_count, v);
  count_launch();
  return HHG_OK;
}
int km_cheb(hhg_kmg* K, int l, double* x, const double* f, bool x_is_zero, cudaStream_t s) {
  auto& L = K->lv[l];
  const int64_t n = p1_len(K->mesh, l);
  const double b = K->prm.cheb_hi_factor * L.lam, a = K->prm.cheb_lo_ratio * b;
  const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  const double* t0 = nullptr;
  if (!x_is_zero) {
    HHG_TRY(km_apply(K, l, x, L.t, s));
    t0 = L.t;
  }
  if (K->prm.degree == 1) return launch_cheb_deg1(n, f, t0, L.dinv, 1.0 / theta, x, s);
  HHG_TRY(launch_cheb0(n, f, t0, L.dinv, 1.0 / theta, L.r, L.d, s));
  for (int k = 1; k < K->prm.degree; ++k) {
    HHG_TRY(km_apply(K, l, L.d, L.t, s));
    const double rn = 1.0 / (2.0 * sigma - rho);
    if (k < K->prm.degree - 1) HHG_TRY(launch_chebk(n, L.t, L.dinv, rn * rho, 2.0 * rn / delta, x, L.r, L.d, s));
    else HHG_TRY(launch_chebk_last(n, L.t, L.dinv, rn * rho, 2.0 * rn / delta, L.r, L.d, x, s));
    rho = rn;
  }
  return HHG_OK;
}
int km_pcg(hhg_kmg* K, int l, const double* f, double* x, cudaStream_t s) {
  auto& L = K->lv[l];
  const Mesh* m = K->mesh;
  const Level& LL = m->levels[l];
  const int64_t n = p1_len(m, l);
  HHG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  HHG_TRY(launch_cheb0(n, f, nullptr, L.dinv, 1.0, L.r, L.d, s));  // r = f, z = D^-1 r
  HHG_TRY(km_mean0(K, l, L.r, s));                                  // consistent singular system
  HHG_TRY(launch_pcg_scale(n, L.dinv, L.r, L.d, s));
  HHG_CUDA(cudaMemcpyAsync(L.p, L.d, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  HHG_TRY(launch_dot_fused(m, LL, HHG_P1, L.r, L.d, K->scal + 0, s, K->red));
  for (int it = 0; it < K->prm.coarse_iters; ++it) {
    HHG_TRY(km_apply(K, l, L.p, L.t, s));
    HHG_TRY(launch_dot_fused(m, LL, HHG_P1, L.p, L.t, K->scal + 1, s, K->red));
    k_pcg_update_pp<<<vg(n), 256, 0, s>>>(n, it, K->scal, x, L.r, L.p, L.t, L.dinv, L.d);
    count_launch();
    HHG_TRY(launch_dot_fused(m, LL, HHG_P1, L.r, L.d, K->scal + ((it & 1) ? 0 : 2), s, K->red));
    HHG_TRY(launch_pcg_dir_zero(n, it, K->scal, L.d, L.p, L.t, s));
  }
  return HHG_OK;
}
int km_cycle(hhg_kmg* K, int l, const double* f, double* x, cudaStream_t s) {
  if (l == K->prm.l_min) return km_pcg(K, l, f, x, s);
  auto& L = K->lv[l];
  const int64_t n = p1_len(K->mesh, l);
  HHG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  for (int i = 0; i < K->prm.pre; ++i) HHG_TRY(km_cheb(K, l, x, f, i == 0, s));
  HHG_TRY(km_apply(K, l, x, L.t, s));
  k_sub<<<vg(n), 256, 0, s>>>(n, f, L.t, L.r);
  count_launch();
  auto& C = K->lv[l - 1];
  HHG_TRY(p1_restrict(K->mesh, l, L.r, C.f, (hhg_stream_t)s));
  HHG_TRY(km_cycle(K, l - 1, C.f, C.x, s));
  HHG_TRY(p1_prolong(K->mesh, l - 1, C.x, x, (hhg_stream_t)s));
  for (int i = 0; i < K->prm.post; ++i) HHG_TRY(km_cheb(K, l, x, f, false, s));
  return HHG_OK;
}
int km_power(hhg_kmg* K, int l) {  // lambda_max(D^-1 K) from a keyed consistent start vector
  auto& L = K->lv[l];
  const Mesh* m = K->mesh;
  const Level& LL = m->levels[l];
  const int64_t n = p1_len(m, l);
  cudaStream_t s = nullptr;
  {  // start vector U[-1,1) keyed by canonical node (seed kKPowerSeed), scattered to all copies
    int64_t nc = 0;
    HHG_TRY(canonical_count(m, LL.n1, &nc));
    std::vector<int64_t> keys((size_t)nc * 10);
    HHG_TRY(canonical_keys(m, LL.n1, keys.data()));
    std::vector<double> v0((size_t)nc);
    for (int64_t i = 0; i < nc; ++i) v0[i] = keyed_uniform(&keys[(size_t)10 * i], kKPowerSeed, 0);
    HHG_TRY(ensure_canon(const_cast<Mesh*>(m), l, HHG_P1));
    double* cdev = nullptr;
    if (cudaMalloc(&cdev, std::max<int64_t>(nc, 1) * sizeof(double)) != cudaSuccess) return fail(HHG_ENOMEM, "kmg start");
    int r = HHG_OK;
    if (cudaMemcpy(cdev, v0.data(), nc * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      r = fail(HHG_ECUDA, "kmg start upload");
    if (r == HHG_OK) r = launch_gather_canon(LL, HHG_P1, n, cdev, L.x, false, s);
    if (r == HHG_OK && cudaDeviceSynchronize() != cudaSuccess) r = fail(HHG_ECUDA, "kmg start");
    cudaFree(cdev);
    HHG_TRY(r);
  }
  for (int it = 0; it < K->prm.power_iters; ++it) {
    HHG_TRY(km_apply(K, l, L.x, L.t, s));
    k_scale_dinv<<<vg(n), 256, 0, s>>>(n, L.t, L.dinv, L.t);
    HHG_TRY(launch_dot(m, LL, HHG_P1, L.t, L.t, K->scal + 8, s, K->red));
    k_normalize<<<vg(n), 256, 0, s>>>(n, K->scal + 8, L.t, L.x);
    count_launch(2);
  }
  double h = 0;
  HHG_CUDA(cudaMemcpy(&h, K->scal + 8, sizeof(double), cudaMemcpyDeviceToHost));
  if (!(h > 0) || !std::isfinite(h)) return fail(HHG_EZEROOP, "K power iteration on a zero operator");
  L.lam = std::sqrt(h);
  return HHG_OK;
}
// CG with device scalars; op / prec write their outputs; proj (may be empty) projects a vector in place
// (mean zero, or nothing).  check_every = 1: one host sync per iteration for the stopping test.  check_every
// = k > 1 (cheap inner solves): the stopping test runs on the device every iteration (k_cg_check latches
// done / iteration / |r|^2 in fl[0..2]) and freezes x and r once it holds (alpha = 0), and the host reads the
// latch every k iterations -- same iterate, iteration count and residual as checking every iteration, with
// k-1 of k host round trips removed (the frozen tail iterations do no harm: x and r stay put).
constexpr int kCheckEvery = 8;  // host reads of the stopping latch in cheap inner solves (mass, vector mass, T)
__global__ void k_cg_step_fz(int64_t n, const double* __restrict__ sc, const double* __restrict__ fl,
                             double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ q) {
  const double alpha = (fl[0] == 0.0 && sc[1] != 0.0) ? sc[0] / sc[1] : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * q[i];
  }
}
__global__ void k_cg_check(const double* __restrict__ sc, double* __restrict__ fl, int it, double r0, double tol,
                           double tol_abs) {
  if (threadIdx.x != 0 || fl[0] != 0.0) return;
  const double rn = sqrt(fmax(sc[3], 0.0));
  if (rn / r0 <= tol || rn <= tol_abs) {
    fl[0] = 1.0;
    fl[1] = it;
    fl[2] = sc[3];
  }
}
int dev_pcg(const Mesh* m, const Level& LL, int space, int64_t n, const std::function<int(const double*, double*)>& op,
            const std::function<int(const double*, double*)>& prec, const std::function<int(double*)>& proj,
            const double* rhs, double* x, double tol, double tol_abs, int max_iters, double* r, double* z, double* p,
            double* q, double* sc, double* red, cudaStream_t s, int* iters_out, double* rel_out, int check_every = 1,
            double* fl = nullptr) {
  if (check_every > 1 && !fl) return fail(HHG_EINVAL, "dev_pcg: batched stopping test needs a latch");
  HHG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  HHG_CUDA(cudaMemcpyAsync(r, rhs, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (proj) HHG_TRY(proj(r));
  HHG_TRY(launch_dot(m, LL, space, r, r, sc + 3, s, red));
  double r0 = 0.0;
  HHG_CUDA(cudaMemcpyAsync(&r0, sc + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
  HHG_CUDA(cudaStreamSynchronize(s));
  r0 = std::sqrt(std::max(r0, 0.0));
  int it = 0;
  double rel = r0 > 0 ? 1.0 : 0.0;
  if (r0 > 0 && r0 > tol_abs) {
    HHG_TRY(prec(r, z));
    if (proj) HHG_TRY(proj(z));
    HHG_CUDA(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    HHG_TRY(launch_dot(m, LL, space, r, z, sc + 0, s, red));
    const unsigned nb = vg(n);
    if (check_every > 1) HHG_CUDA(cudaMemsetAsync(fl, 0, 3 * sizeof(double), s));
    while (it < max_iters) {
      ++it;
      HHG_TRY(op(p, q));
      HHG_TRY(launch_dot(m, LL, space, p, q, sc + 1, s, red));
      if (check_every > 1) k_cg_step_fz<<<nb, 256, 0, s>>>(n, sc, fl, x, r, p, q);
      else k_cg_step<<<nb, 256, 0, s>>>(n, sc, x, r, p, q);
      count_launch();
      HHG_TRY(launch_dot(m, LL, space, r, r, sc + 3, s, red));
      if (check_every > 1) {
        k_cg_check<<<1, 32, 0, s>>>(sc, fl, it, r0, tol, tol_abs);
        count_launch();
        if (it % check_every == 0 || it == max_iters) {
          double h[3];
          HHG_CUDA(cudaMemcpyAsync(h, fl, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
          HHG_CUDA(cudaStreamSynchronize(s));
          if (h[0] != 0.0) {
            it = (int)h[1];
            rel = std::sqrt(std::max(h[2], 0.0)) / r0;
            break;
          }
          double rr = 0.0;
          HHG_CUDA(cudaMemcpy(&rr, sc + 3, sizeof(double), cudaMemcpyDeviceToHost));
          rel = std::sqrt(std::max(rr, 0.0)) / r0;
        }
      } else {
        double rr = 0.0;
        HHG_CUDA(cudaMemcpyAsync(&rr, sc + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
        HHG_CUDA(cudaStreamSynchronize(s));
        const double rn = std::sqrt(std::max(rr, 0.0));
        rel = rn / r0;
        if (rel <= tol || rn <= tol_abs) break;
      }
      HHG_TRY(prec(r, z));
      if (proj) HHG_TRY(proj(z));
      HHG_TRY(launch_dot(m, LL, space, r, z, sc + 2, s, red));
      k_cg_dir<<<nb, 256, 0, s>>>(n, sc, z, p);
      k_cg_roll<<<1, 32, 0, s>>>(sc);
      count_launch(2);
    }
  }
  if (proj) HHG_TRY(proj(x));
  if (iters_out) *iters_out = it;
  if (rel_out) *rel_out = rel;
  return HHG_OK;
}
}  // namespace

extern "C" {
int hhg_kmg_create(hhg_mesh* mesh, const hhg_mg_params* params, const double* const* eta_per_level, double a,
                   hhg_kmg** out) {
  if (!mesh || !params || !out) return fail(HHG_EINVAL, "hhg_kmg_create: NULL argument");
  const hhg_mg_params& P = *params;
  if (P.l_min < 0 || P.l_max > mesh->level_max || P.l_min > P.l_max)
    return fail(HHG_ELEVEL, "hhg_kmg_create: need 0 <= l_min <= l_max <= level_max");
  if (P.degree < 1 || P.pre < 0 || P.post < 0 || P.coarse_iters < 0 || P.power_iters < 1 || !(a > 0))
    return fail(HHG_EINVAL, "hhg_kmg_create: bad parameters");
  if (a != 1.0 && mesh->blend != HHG_BLEND_SHELL)
    return fail(HHG_EINVAL, "hhg_kmg_create: surface scaling a != 1 needs a shell-blended mesh");
  auto* K = new hhg_kmg();
  K->mesh = mesh;
  K->prm = P;
  K->a = a;
  K->lv.resize(P.l_max + 1);
  auto bail = [&](int code) {
    delete K;
    return code;
  };
  ++mesh->dependents;
  if (cudaMalloc(&K->scal, 16 * sizeof(double)) != cudaSuccess || cudaMemset(K->scal, 0, 16 * sizeof(double)) != cudaSuccess)
    return bail(fail(HHG_ENOMEM, "kmg scal"));
  if (red_alloc(&K->red) != HHG_OK) return bail(HHG_ENOMEM);
  const int64_t nf = p1_len(mesh, P.l_max);
  for (double** p : {&K->cr, &K->cz, &K->cp, &K->cq})
    if (cudaMalloc(p, std::max<int64_t>(nf, 1) * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "kmg cg"));
  for (int l = P.l_min; l <= P.l_max; ++l) {
    int r = ensure_level(mesh, l);
    if (r != HHG_OK) return bail(r);
    const int64_t n = p1_len(mesh, l);
    auto& L = K->lv[l];
    L.eta = eta_per_level ? eta_per_level[l] : nullptr;
    for (double** p : {&L.x, &L.f, &L.r, &L.d, &L.t, &L.dinv, &L.p, &L.ones})
      if (cudaMalloc(p, std::max<int64_t>(n, 1) * sizeof(double)) != cudaSuccess) return bail(fail(HHG_ENOMEM, "kmg vectors"));
    r = launch_fill(n, 1.0, L.ones, nullptr);
    if (r == HHG_OK) r = launch_dot(mesh, mesh->levels[l], HHG_P1, L.ones, L.ones, K->scal + 9, nullptr, K->red);
    double cnt = 0.0;
    if (r == HHG_OK && cudaMemcpy(&cnt, K->scal + 9, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      r = fail(HHG_ECUDA, "kmg count");
    if (r != HHG_OK) return bail(r);
    L.inv_count = 1.0 / cnt;
    r = surf_op(mesh, l, ELEM_KP1D, L.eta, a, nullptr, L.t, nullptr);
    if (r != HHG_OK) return bail(r);
    k_recip<<<vg(n), 256>>>(n, L.t, L.dinv);
    count_launch();
    if (l > P.l_min && (r = km_power(K, l)) != HHG_OK) return bail(r);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(HHG_ECUDA, "hhg_kmg_create: sync failed"));
  *out = K;
  return HHG_OK;
}

int hhg_kmg_solve(hhg_kmg* K, const double* rhs, double* x, double tol, double tol_abs, int max_iters, int* iters,
                  double* rel_res, hhg_stream_t stream) {
  if (!K || !rhs || !x) return fail(HHG_EINVAL, "hhg_kmg_solve: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int lf = K->prm.l_max;
  const Mesh* m = K->mesh;
  auto op = [&](const double* u, double* y) { return km_apply(K, lf, u, y, s); };
  auto prec = [&](const double* r, double* z) { return km_cycle(K, lf, r, z, s); };
  auto proj = [&](double* v) { return km_mean0(K, lf, v, s); };
  return dev_pcg(m, m->levels[lf], HHG_P1, p1_len(m, lf), op, prec, proj, rhs, x, tol, tol_abs, max_iters, K->cr,
                 K->cz, K->cp, K->cq, K->scal + 10, K->red, s, iters, rel_res);
}

int hhg_kmg_destroy(hhg_kmg* K) {
  delete K;
  return HHG_OK;
}
}  // extern "C"

// ---------------------------------------------------------------- solve statistics (HHG_STATS=1)
// Inner-solver call counts, iterations and host wall time (every inner CG synchronises on its stopping test,
// so wall time = device time + launch/sync latency); printed as one JSON line per hhg_stokes_solve (stderr).
namespace {
struct SolveStat {
  const char* name;
  long calls, iters;
  double sec;
};
SolveStat g_stat[] = {{"ablock_cg", 0, 0, 0}, {"bacbt_cg", 0, 0, 0}, {"mass_cg", 0, 0, 0}, {"vmass_cg", 0, 0, 0},
                      {"kmg_cg", 0, 0, 0}};
enum { ST_ABLOCK, ST_BACBT, ST_MASS, ST_VMASS, ST_KMG, ST_N };
bool stats_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HHG_STATS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
struct StatScope {
  int k;
  const int* it;
  std::chrono::steady_clock::time_point t0;
  StatScope(int k_, const int* it_) : k(k_), it(it_), t0(std::chrono::steady_clock::now()) {}
  ~StatScope() {
    if (!stats_on()) return;
    g_stat[k].calls += 1;
    g_stat[k].iters += *it;
    g_stat[k].sec += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};
void stats_print(int fgmres_iters, double sec) {
  if (!stats_on()) return;
  fprintf(stderr, "{\"hhg_stats\": \"stokes_solve\", \"fgmres_iters\": %d, \"solve_s\": %.3f", fgmres_iters, sec);
  for (int k = 0; k < ST_N; ++k) {
    fprintf(stderr, ", \"%s\": {\"calls\": %ld, \"iters\": %ld, \"s\": %.3f}", g_stat[k].name, g_stat[k].calls,
            g_stat[k].iters, g_stat[k].sec);
    g_stat[k].calls = g_stat[k].iters = 0;
    g_stat[k].sec = 0;
  }
  fprintf(stderr, "}\n");
}
}  // namespace

// ================================================================ Stokes solve (NEXT-1)
// FGMRES right-preconditioned by the symmetric Uzawa block preconditioner
// (eq:SymmetricUzawaStep1) with B replaced by B + C in the pressure update:
//   u_hat = sigma A^-1 r_u ;  p = -omega S^-1 (r_p - (B+C) u_hat) ;  u = u_hat + sigma A^-1 (r_u - A u_hat - B^T p)
// A^-1 = CG preconditioned by the V-cycle to tol_A (hhg_ablock_cg), S^-1 = M_{1/eta}^-1 by
// Jacobi-CG to tol_M (eq:schurMass).  The pressure part of every Krylov vector, operator
// output and preconditioner output is projected to arithmetic mean zero (P_p).
// Block vectors are [u (P2VEC) | p (P1)] in one allocation.
struct hhg_stokes {
  hhg_mg* mg = nullptr;
  hhg_mg* mgC = nullptr;     // cheap V-cycle A_C of the V-cycle BFBT (m_V = 1, deg_V = 1), may be NULL
  hhg_mesh* mesh = nullptr;
  int level = 0;
  const double* eta = nullptr;
  double gamma = 0.0;
  hhg_stokes_params prm{};
  int64_t n2 = 0, n1 = 0;
  std::vector<double*> V, Z;
  double *w = nullptr, *t = nullptr, *a = nullptr, *b = nullptr, *ones = nullptr, *mdinv = nullptr, *sc = nullptr;
  double* red = nullptr;  // reduction scratch of this object
  double *mr = nullptr, *mz = nullptr, *mp = nullptr, *mq = nullptr;
  double *br = nullptr, *bz = nullptr, *bp = nullptr, *bq = nullptr, *bt = nullptr;  // BFBT CG (P1)
  double *bu = nullptr, *bv = nullptr;                                                 // BFBT velocity temps
  // w-BFBT (schur = 2): K_{1/sqrt(eta_l)}, K_{1/sqrt(eta_r)} hierarchies (kr == kl when a_l == a_r),
  // inverse diagonals of M_{sqrt(eta_l)}, M_{sqrt(eta_r)} and the vector-mass CG vectors
  hhg_kmg *kl = nullptr, *kr = nullptr;
  double *vdl = nullptr, *vdr = nullptr, *vr = nullptr, *vz = nullptr, *vp = nullptr, *vq = nullptr;
  double n_unique_p = 0.0;
  ~hhg_stokes() {
    for (double* p : V) cudaFree(p);
    for (double* p : Z) cudaFree(p);
    if (mesh) --mesh->dependents;
    for (double* p : {w, t, a, b, ones, mdinv, sc, red, mr, mz, mp, mq, br, bz, bp, bq, bt, bu, bv, vdl, vdr, vr, vz, vp, vq})
      if (p) cudaFree(p);
    if (kr && kr != kl) delete kr;
    if (kl) delete kl;
  }
};

namespace {
int st_dot(hhg_stokes* S, const double* x, const double* y, int what, double* out, cudaStream_t s) {
  // what: 1 = velocity part, 2 = pressure part, 3 = both
  const Mesh* m = S->mesh;
  const Level& L = m->levels[S->level];
  double h[2] = {0.0, 0.0};
  if (what & 1) HHG_TRY(launch_dot(m, L, HHG_P2VEC, x, y, S->sc + 0, s, S->red));
  if (what & 2) HHG_TRY(launch_dot(m, L, HHG_P1, x + S->n2, y + S->n2, S->sc + 1, s, S->red));
  HHG_CUDA(cudaMemcpyAsync(h, S->sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  HHG_CUDA(cudaStreamSynchronize(s));
  *out = ((what & 1) ? h[0] : 0.0) + ((what & 2) ? h[1] : 0.0);
  HHG_CUDA(cudaMemsetAsync(S->sc, 0, 2 * sizeof(double), s));
  return HHG_OK;
}
int st_mean0(hhg_stokes* S, double* p, cudaStream_t s) {  // P_p: arithmetic mean zero over unique nodes
  // device-only: fused owner-masked sum, then p -= sum / n_unique read on the device (no host sync)
  const Level& L = S->mesh->levels[S->level];
  HHG_TRY(launch_dot_fused(S->mesh, L, HHG_P1, p, S->ones, S->sc + 2, s, S->red));
  k_shift<<<vg(S->n1), 256, 0, s>>>(S->n1, S->sc + 2, 1.0 / S->n_unique_p, p);
  count_launch();
  return HHG_OK;
}
// y = P K x : [ (M P_v)(A u + B^T p) ; P_p (B + C) u ]
int st_op(hhg_stokes* S, const double* x, double* y, cudaStream_t s) {
  HHG_TRY(stokes_apply(S->mesh, S->level, S->eta, S->gamma, x, x + S->n2, y, y + S->n2, (hhg_stream_t)s));
  return st_mean0(S, y + S->n2, s);
}
// z_p = M_{1/eta}^-1 r_p by Jacobi-CG from 0 to relative tolerance tol_M (mass SPD); device scalars,
// one host sync per iteration (dev_pcg), scalar slots sc[8..11]
int st_mass_solve(hhg_stokes* S, const double* rp, double* zp, cudaStream_t s) {
  const Mesh* m = S->mesh;
  const Level& L = m->levels[S->level];
  auto op = [&](const double* x, double* y) -> int { return hhg_mass_apply(S->mesh, S->level, S->eta, x, y, (hhg_stream_t)s); };
  auto jac = [&](const double* r, double* z) -> int { return launch_pcg_scale(S->n1, S->mdinv, r, z, s); };
  int it = 0;
  double rel;
  StatScope st(ST_MASS, &it);
  return dev_pcg(m, L, HHG_P1, S->n1, op, jac, std::function<int(double*)>(), rp, zp, S->prm.tol_mass, 0.0,
                 S->prm.mass_max_iters, S->mr, S->mz, S->mp, S->mq, S->sc + 8, S->red, s, &it, &rel, kCheckEvery,
                 S->sc + 24);
}
// w = P_p B A_C^-1 B^T y  (A_C^-1 = one cheap V-cycle, eq:schurV)
int st_bacbt(hhg_stokes* S, const double* y, double* w, cudaStream_t s) {
  HHG_TRY(divT_apply(S->mesh, S->level, y, S->bu, 0, (hhg_stream_t)s));
  HHG_TRY(vcycle(S->mgC, S->bu, S->bv, (hhg_stream_t)s));
  HHG_TRY(div_apply(S->mesh, S->level, 0.0, S->bv, w, (hhg_stream_t)s));
  return st_mean0(S, w, s);
}
// y = (B A_C^-1 B^T)^-1 t by CG preconditioned by M_{1/eta} (mass CG to tol_mass), to tol_vbfbt;
// mean-zero projections of r, z and y (P_p); scalar slots sc[12..15]
int st_bacbt_solve(hhg_stokes* S, const double* t, double* y, cudaStream_t s) {
  const Mesh* m = S->mesh;
  const Level& L = m->levels[S->level];
  auto op = [&](const double* x, double* w) -> int { return st_bacbt(S, x, w, s); };
  auto prec = [&](const double* r, double* z) -> int { return st_mass_solve(S, r, z, s); };
  auto proj = [&](double* v) -> int { return st_mean0(S, v, s); };
  int it = 0;
  double rel;
  StatScope st(ST_BACBT, &it);
  return dev_pcg(m, L, HHG_P1, S->n1, op, prec, proj, t, y, S->prm.tol_vbfbt, 0.0, S->prm.vbfbt_max_iters, S->br,
                 S->bz, S->bp, S->bq, S->sc + 12, S->red, s, &it, &rel);
}
// z_p = S_V^-1 t (eq:schurV): (B A_C^-1 B^T)^-1 (B A_C^-1 A A_C^-1 B^T) (B A_C^-1 B^T)^-1 t
int st_vbfbt(hhg_stokes* S, const double* t, double* z, cudaStream_t s) {
  HHG_TRY(st_bacbt_solve(S, t, S->bt, s));
  HHG_TRY(divT_apply(S->mesh, S->level, S->bt, S->bu, 0, (hhg_stream_t)s));
  HHG_TRY(vcycle(S->mgC, S->bu, S->bv, (hhg_stream_t)s));
  HHG_TRY(epsilon_apply(S->mesh, S->level, HHG_VISC_FULL, S->eta, S->bv, S->bu, (hhg_stream_t)s));
  HHG_TRY(vcycle(S->mgC, S->bu, S->bv, (hhg_stream_t)s));
  HHG_TRY(div_apply(S->mesh, S->level, 0.0, S->bv, S->bt, (hhg_stream_t)s));
  HHG_TRY(st_mean0(S, S->bt, s));
  return st_bacbt_solve(S, S->bt, z, s);
}

// x = M_{sqrt(eta_a)}^-1 v on the constrained velocity space: Jacobi-CG (D^-1 then P_v M) to tol_vmass
int st_vmass_solve(hhg_stokes* S, double a, const double* vdinv, const double* v, double* x, cudaStream_t s) {
  const Mesh* m = S->mesh;
  const Level& L = m->levels[S->level];
  auto op = [&](const double* u, double* y) { return hhg_vmass_apply(S->mesh, S->level, S->eta, a, u, y, (hhg_stream_t)s); };
  auto prec = [&](const double* r, double* z) {
    HHG_TRY(launch_pcg_scale(S->n2, vdinv, r, z, s));
    return launch_fixup(m, L, HHG_P2VEC, false, true, z, s);
  };
  int it = 0;
  double rel;
  StatScope st(ST_VMASS, &it);
  return dev_pcg(m, L, HHG_P2VEC, S->n2, op, prec, std::function<int(double*)>(), v, x, S->prm.tol_vmass, 0.0,
                 S->prm.vmass_max_iters, S->vr, S->vz, S->vp, S->vq, S->sc + 16, S->red, s, &it, &rel, kCheckEvery,
                 S->sc + 28);
}
// z = S_w^-1 t (eq:schurWBFBT with a_l / a_r):
//   K_{1/sqrt(eta_l)}^-1 B M_{sqrt(eta_l)}^-1 A M_{sqrt(eta_r)}^-1 B^T K_{1/sqrt(eta_r)}^-1 t
int st_wbfbt(hhg_stokes* S, const double* t, double* z, cudaStream_t s) {
  int it = 0;
  double rel;
  const auto& P = S->prm;
  {
    StatScope st(ST_KMG, &it);
    HHG_TRY(hhg_kmg_solve(S->kr, t, S->bt, P.tol_wbfbt, P.tol_wbfbt_abs, P.wbfbt_max_iters, &it, &rel, (hhg_stream_t)s));
  }
  HHG_TRY(divT_apply(S->mesh, S->level, S->bt, S->bu, 0, (hhg_stream_t)s));
  HHG_TRY(st_vmass_solve(S, P.a_r, S->vdr, S->bu, S->bv, s));
  HHG_TRY(epsilon_apply(S->mesh, S->level, HHG_VISC_FULL, S->eta, S->bv, S->bu, (hhg_stream_t)s));
  HHG_TRY(st_vmass_solve(S, P.a_l, S->vdl, S->bu, S->bv, s));
  HHG_TRY(div_apply(S->mesh, S->level, 0.0, S->bv, S->bt, (hhg_stream_t)s));
  HHG_TRY(st_mean0(S, S->bt, s));
  StatScope st(ST_KMG, &it);
  return hhg_kmg_solve(S->kl, S->bt, z, P.tol_wbfbt, P.tol_wbfbt_abs, P.wbfbt_max_iters, &it, &rel, (hhg_stream_t)s);
}

int st_schur_inv(hhg_stokes* S, const double* t, double* z, cudaStream_t s) {  // z = S^-1 t
  if (S->prm.schur == 1) return st_vbfbt(S, t, z, s);
  if (S->prm.schur == 2) return st_wbfbt(S, t, z, s);
  return st_mass_solve(S, t, z, s);
}
// z = Prec(r): one symmetric Uzawa step from (0, 0)
int st_schur(hhg_stokes* S, const double* t, double* z, cudaStream_t s) {  // z = -omega S^-1 t, mean zero
  HHG_TRY(st_schur_inv(S, t, z, s));
  HHG_TRY(launch_axpby(S->n1, 0.0, z, -S->prm.omega, z, s));
  return st_mean0(S, z, s);
}
// z = Prec(r): one Uzawa step from (0, 0) -- symmetric (eq:SymmetricUzawaStep1, default), inexact
// (eq:InexactUzawaStep1) or adjoint inexact (eq:AdjointInexactUzawaStep1), B -> B + C in the
// pressure update
int st_prec(hhg_stokes* S, const double* r, double* z, cudaStream_t s) {
  const int64_t n2 = S->n2, n1 = S->n1;
  const double sig = S->prm.sigma;
  int it;
  double rel;
  if (S->prm.uzawa == 2) {
    // adjoint: p = -omega S^-1 (r_p - (B+C) 0) ; u = sigma A^-1 (r_u - B^T p)
    HHG_CUDA(cudaMemcpyAsync(S->t + n2, r + n2, n1 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    HHG_TRY(st_mean0(S, S->t + n2, s));
    HHG_TRY(st_schur(S, S->t + n2, z + n2, s));
    HHG_TRY(divT_apply(S->mesh, S->level, z + n2, S->t, 0, (hhg_stream_t)s));
    HHG_TRY(launch_axpby(n2, 1.0, r, -1.0, S->t, s));
    {
      StatScope st(ST_ABLOCK, &it);
      HHG_TRY(hhg_ablock_cg(S->mg, S->t, z, S->prm.tol_A, S->prm.ablock_max_iters, &it, &rel, (hhg_stream_t)s));
    }
    return launch_axpby(n2, 0.0, z, sig, z, s);
  }
  // u_hat = sigma A^-1 r_u  (z_u holds u_hat)
  {
    StatScope st(ST_ABLOCK, &it);
    HHG_TRY(hhg_ablock_cg(S->mg, r, z, S->prm.tol_A, S->prm.ablock_max_iters, &it, &rel, (hhg_stream_t)s));
  }
  HHG_TRY(launch_axpby(n2, 0.0, z, sig, z, s));
  // t_p = r_p - (B + C) u_hat ; p = -omega S^-1 t_p ; P_p
  HHG_TRY(div_apply(S->mesh, S->level, S->gamma, z, S->t + n2, (hhg_stream_t)s));
  HHG_TRY(launch_axpby(n1, 1.0, r + n2, -1.0, S->t + n2, s));
  HHG_TRY(st_mean0(S, S->t + n2, s));
  HHG_TRY(st_schur(S, S->t + n2, z + n2, s));
  if (S->prm.uzawa == 1) return HHG_OK;  // inexact: (u_hat, p)
  // t_u = r_u - A u_hat - B^T p ; u = u_hat + sigma A^-1 t_u
  HHG_TRY(stokes_apply(S->mesh, S->level, S->eta, S->gamma, z, z + n2, S->t, S->a + n2, (hhg_stream_t)s));
  HHG_TRY(launch_axpby(n2, 1.0, r, -1.0, S->t, s));
  {
    StatScope st(ST_ABLOCK, &it);
    HHG_TRY(hhg_ablock_cg(S->mg, S->t, S->a, S->prm.tol_A, S->prm.ablock_max_iters, &it, &rel, (hhg_stream_t)s));
  }
  return launch_axpby(n2, sig, S->a, 1.0, z, s);
}
}  // namespace

extern "C" {

int hhg_stokes_create(hhg_mg* mg, hhg_mg* mg_cheap, const double* eta_p1, double gamma, const hhg_stokes_params* prm,
                      hhg_stokes** out) {
  if (!mg || !prm || !out) return fail(HHG_EINVAL, "hhg_stokes_create: NULL argument");
  if (prm->restart < 1 || prm->max_iters < 1 || !(prm->tol > 0) || !(prm->tol_A > 0) || !(prm->tol_mass > 0))
    return fail(HHG_EINVAL, "hhg_stokes_create: bad parameters");
  if (prm->schur < 0 || prm->schur > 2)
    return fail(HHG_EINVAL, "hhg_stokes_create: schur must be 0 (mass), 1 (V-BFBT) or 2 (w-BFBT)");
  if (prm->schur == 2 && (!(prm->a_l > 0) || !(prm->a_r > 0) || !(prm->tol_wbfbt > 0 || prm->tol_wbfbt_abs > 0) ||
                          prm->wbfbt_max_iters < 1 || !(prm->tol_vmass > 0) || prm->vmass_max_iters < 1))
    return fail(HHG_EINVAL, "hhg_stokes_create: w-BFBT needs a_l, a_r > 0, a K tolerance, tol_vmass and iteration caps");
  if (prm->uzawa < 0 || prm->uzawa > 2) return fail(HHG_EINVAL, "hhg_stokes_create: uzawa must be 0, 1 or 2");
  // the saddle-point operator applies A with the P1 viscosity eta_p1 on the finest level; a hierarchy that evaluates
  // eta at the quadrature points there (l_eta >= l_max) would precondition a different A (l_eta < l_max)
  if (mg->lv[mg->prm.l_max].T2 || (mg_cheap && mg_cheap->lv[mg_cheap->prm.l_max].T2))
    return fail(HHG_EINVAL, "hhg_stokes_create: the hierarchies must use the P1 viscosity on the finest level "
                            "(l_eta < l_max)");
  if (prm->schur == 1 && (!mg_cheap || mg_cheap->mesh != mg->mesh || mg_cheap->prm.l_max != mg->prm.l_max ||
                          !(prm->tol_vbfbt > 0) || prm->vbfbt_max_iters < 1))
    return fail(HHG_EINVAL, "hhg_stokes_create: V-BFBT needs a cheap hierarchy on the same mesh/levels and tol_vbfbt");
  auto* S = new hhg_stokes();
  S->mg = mg;
  S->mgC = mg_cheap;
  S->mesh = mg->mesh;
  S->level = mg->prm.l_max;
  S->eta = eta_p1;
  S->gamma = gamma;
  S->prm = *prm;
  const Level& L = S->mesh->levels[S->level];
  S->n2 = p2vec_len(S->mesh, S->level);
  S->n1 = macro_count(S->mesh) * L.npts1;
  const int64_t nb = S->n2 + S->n1;
  auto alloc = [&](double** p, int64_t n) { return cudaMalloc(p, std::max<int64_t>(n, 1) * sizeof(double)) == cudaSuccess; };
  bool ok = true;
  S->V.resize(prm->restart + 1, nullptr);
  S->Z.resize(prm->restart, nullptr);
  for (auto& p : S->V) ok = ok && alloc(&p, nb);
  for (auto& p : S->Z) ok = ok && alloc(&p, nb);
  for (double** p : {&S->w, &S->t, &S->a, &S->b}) ok = ok && alloc(p, nb);
  for (double** p : {&S->ones, &S->mdinv, &S->mr, &S->mz, &S->mp, &S->mq, &S->br, &S->bz, &S->bp, &S->bq, &S->bt})
    ok = ok && alloc(p, S->n1);
  for (double** p : {&S->bu, &S->bv}) ok = ok && alloc(p, S->n2);
  if (prm->schur == 2)
    for (double** p : {&S->vdl, &S->vdr, &S->vr, &S->vz, &S->vp, &S->vq}) ok = ok && alloc(p, S->n2);
  ok = ok && alloc(&S->sc, 32) && red_alloc(&S->red) == HHG_OK;
  ++S->mesh->dependents;
  if (!ok) {
    delete S;
    return fail(HHG_ENOMEM, "hhg_stokes_create: workspace");
  }
  cudaStream_t s = nullptr;
  int r = HHG_OK;
  auto run = [&]() -> int {
    HHG_CUDA(cudaMemset(S->sc, 0, 32 * sizeof(double)));
    HHG_TRY(launch_fill(S->n1, 1.0, S->ones, s));
    HHG_TRY(hhg_mass_diag(S->mesh, S->level, S->eta, S->mdinv, nullptr));
    HHG_TRY(launch_recip(S->n1, S->mdinv, s));
    HHG_TRY(launch_dot(S->mesh, L, HHG_P1, S->ones, S->ones, S->sc + 4, s, S->red));
    HHG_CUDA(cudaMemcpy(&S->n_unique_p, S->sc + 4, sizeof(double), cudaMemcpyDeviceToHost));
    if (prm->schur == 2) {
      std::vector<const double*> etas(mg->prm.l_max + 1, nullptr);
      for (int l = mg->prm.l_min; l <= mg->prm.l_max; ++l) etas[l] = mg->lv[l].eta;
      HHG_TRY(hhg_kmg_create(S->mesh, &mg->prm, etas.data(), prm->a_l, &S->kl));
      if (prm->a_r == prm->a_l) S->kr = S->kl;
      else HHG_TRY(hhg_kmg_create(S->mesh, &mg->prm, etas.data(), prm->a_r, &S->kr));
      HHG_TRY(hhg_vmass_diag(S->mesh, S->level, S->eta, prm->a_l, S->vdl, nullptr));
      HHG_TRY(launch_recip(S->n2, S->vdl, s));
      HHG_TRY(hhg_vmass_diag(S->mesh, S->level, S->eta, prm->a_r, S->vdr, nullptr));
      HHG_TRY(launch_recip(S->n2, S->vdr, s));
      HHG_CUDA(cudaDeviceSynchronize());
    }
    return HHG_OK;
  };
  r = run();
  if (r != HHG_OK) {
    delete S;
    return r;
  }
  *out = S;
  return HHG_OK;
}

int hhg_stokes_schur_apply(hhg_stokes* S, const double* t, double* z, hhg_stream_t stream) {
  if (!S || !t || !z) return fail(HHG_EINVAL, "hhg_stokes_schur_apply: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  HHG_CUDA(cudaMemcpyAsync(S->t + S->n2, t, S->n1 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  HHG_TRY(st_mean0(S, S->t + S->n2, s));
  HHG_TRY(st_schur_inv(S, S->t + S->n2, z, s));
  HHG_TRY(st_mean0(S, z, s));
  HHG_CUDA(cudaStreamSynchronize(s));
  return HHG_OK;
}

int hhg_stokes_destroy(hhg_stokes* S) {
  delete S;
  return HHG_OK;
}

int hhg_stokes_solve(hhg_stokes* S, const double* rhs, double* x, int* iters_out, double* rel_res_out,
                     hhg_stream_t stream) {
  if (!S || !rhs || !x) return fail(HHG_EINVAL, "hhg_stokes_solve: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n2 = S->n2, n1 = S->n1, nb = n2 + n1;
  const int m = S->prm.restart;
  const auto t_start = std::chrono::steady_clock::now();
  // b = P rhs
  HHG_CUDA(cudaMemcpyAsync(S->b, rhs, nb * sizeof(double), cudaMemcpyDeviceToDevice, s));
  HHG_TRY(launch_fixup(S->mesh, S->mesh->levels[S->level], HHG_P2VEC, false, true, S->b, s));
  HHG_TRY(st_mean0(S, S->b + n2, s));
  double bn = 0.0;
  HHG_TRY(st_dot(S, S->b, S->b, 3, &bn, s));
  bn = std::sqrt(bn);
  HHG_CUDA(cudaMemsetAsync(x, 0, nb * sizeof(double), s));
  int total = 0;
  double rel = bn > 0 ? 1.0 : 0.0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  while (bn > 0 && total < S->prm.max_iters && rel > S->prm.tol) {
    // r = b - P K x
    HHG_TRY(st_op(S, x, S->w, s));
    HHG_TRY(launch_axpby(nb, 1.0, S->b, -1.0, S->w, s));
    double beta = 0.0;
    HHG_TRY(st_dot(S, S->w, S->w, 3, &beta, s));
    beta = std::sqrt(beta);
    rel = beta / bn;
    if (rel <= S->prm.tol) break;
    HHG_TRY(launch_axpby(nb, 1.0 / beta, S->w, 0.0, S->V[0], s));
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m && total < S->prm.max_iters; ++j) {
      ++total;
      HHG_TRY(st_prec(S, S->V[j], S->Z[j], s));
      HHG_TRY(st_op(S, S->Z[j], S->w, s));
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
        double h = 0.0;
        HHG_TRY(st_dot(S, S->w, S->V[i], 3, &h, s));
        H[(size_t)i * m + j] = h;
        HHG_TRY(launch_axpby(nb, -h, S->V[i], 1.0, S->w, s));
      }
      double hn = 0.0;
      HHG_TRY(st_dot(S, S->w, S->w, 3, &hn, s));
      hn = std::sqrt(hn);
      H[(size_t)(j + 1) * m + j] = hn;
      if (hn > 0) HHG_TRY(launch_axpby(nb, 1.0 / hn, S->w, 0.0, S->V[j + 1], s));
      for (int i = 0; i < j; ++i) {  // previous Givens rotations
        const double h0 = H[(size_t)i * m + j], h1 = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * h0 + sn[i] * h1;
        H[(size_t)(i + 1) * m + j] = -sn[i] * h0 + cs[i] * h1;
      }
      const double h0 = H[(size_t)j * m + j], h1 = H[(size_t)(j + 1) * m + j];
      const double d = std::hypot(h0, h1);
      cs[j] = d > 0 ? h0 / d : 1.0;
      sn[j] = d > 0 ? h1 / d : 0.0;
      H[(size_t)j * m + j] = d;
      H[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rel = std::fabs(g[j + 1]) / bn;
      if (stats_on())
        fprintf(stderr, "{\"hhg_stats\": \"fgmres\", \"it\": %d, \"rel\": %.6e, \"t_s\": %.3f}\n", total, rel,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
      if (rel <= S->prm.tol || hn == 0.0) {
        ++j;
        break;
      }
    }
    // x += Z y,  H(0:j,0:j) y = g(0:j)
    for (int i = j - 1; i >= 0; --i) {
      double acc = g[i];
      for (int k = i + 1; k < j; ++k) acc -= H[(size_t)i * m + k] * y[k];
      y[i] = acc / H[(size_t)i * m + i];
    }
    for (int i = 0; i < j; ++i) HHG_TRY(launch_axpby(nb, y[i], S->Z[i], 1.0, x, s));
  }
  // true residual of the projected system
  if (bn > 0) {
    HHG_TRY(st_op(S, x, S->w, s));
    HHG_TRY(launch_axpby(nb, 1.0, S->b, -1.0, S->w, s));
    double rr = 0.0;
    HHG_TRY(st_dot(S, S->w, S->w, 3, &rr, s));
    rel = std::sqrt(rr) / bn;
  }
  HHG_CUDA(cudaStreamSynchronize(s));
  if (iters_out) *iters_out = total;
  if (rel_res_out) *rel_res_out = rel;
  stats_print(total, std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
  return HHG_OK;
}

}  // extern "C"

// ================================================================ temperature solve (NEXT-4, part)
// "an FGMRES outer loop preconditioned by a CG solver solving the symmetric, positive
// semidefinite mass and diffusion part of the left-hand-side"; Dirichlet values on the surface and
// the CMB.  Unknown delta = T - T_D lives on the interior nodes (bcn2 == -1); every Krylov vector and
// operator output is masked to them (the boundary rows of the constrained system are the identity
// with a zero right-hand side, so they stay zero).
namespace {
__global__ void k_mask(int64_t n, const int32_t* __restrict__ bcn, int keep_boundary, const double* __restrict__ in,
                       double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool bnd = bcn[i] != -1;
    out[i] = (bnd == (keep_boundary != 0)) ? in[i] : 0.0;
  }
}
int temp_apply_raw(const Mesh* m, int level, const hhg_temp_params& prm, const double* u, const double* T, double* y,
                   int which, cudaStream_t s) {
  const Level& L = m->levels[level];
  HHG_CUDA(cudaMemsetAsync(y, 0, macro_count(m) * L.npts2 * sizeof(double), s));
  HHG_TRY(launch_temp(m, L, which, prm, u, T, y, s));
  return launch_fixup(m, L, HHG_P2, true, false, y, s);
}
// restarted right-preconditioned FGMRES (MGS + Givens), host Hessenberg, device vectors
int fgmres(int64_t n, int m, int max_iters, double tol, double tol_abs,
           const std::function<int(const double*, double*)>& op, const std::function<int(const double*, double*)>& prec,
           const std::function<int(const double*, const double*, double*)>& dot, std::vector<double*>& V,
           std::vector<double*>& Z, double* w, const double* b, double* x, cudaStream_t s, int* iters_out,
           double* rel_out) {
  double bn = 0.0;
  HHG_TRY(dot(b, b, &bn));
  bn = std::sqrt(bn);
  HHG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  int total = 0;
  double rel = bn > 0 ? 1.0 : 0.0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  while (bn > 0 && total < max_iters && rel > tol && rel * bn > tol_abs) {
    HHG_TRY(op(x, w));
    HHG_TRY(launch_axpby(n, 1.0, b, -1.0, w, s));
    double beta = 0.0;
    HHG_TRY(dot(w, w, &beta));
    beta = std::sqrt(beta);
    rel = beta / bn;
    if (rel <= tol || beta <= tol_abs) break;
    HHG_TRY(launch_axpby(n, 1.0 / beta, w, 0.0, V[0], s));
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m && total < max_iters; ++j) {
      ++total;
      HHG_TRY(prec(V[j], Z[j]));
      HHG_TRY(op(Z[j], w));
      for (int i = 0; i <= j; ++i) {
        double h = 0.0;
        HHG_TRY(dot(w, V[i], &h));
        H[(size_t)i * m + j] = h;
        HHG_TRY(launch_axpby(n, -h, V[i], 1.0, w, s));
      }
      double hn = 0.0;
      HHG_TRY(dot(w, w, &hn));
      hn = std::sqrt(hn);
      H[(size_t)(j + 1) * m + j] = hn;
      if (hn > 0) HHG_TRY(launch_axpby(n, 1.0 / hn, w, 0.0, V[j + 1], s));
      for (int i = 0; i < j; ++i) {
        const double h0 = H[(size_t)i * m + j], h1 = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * h0 + sn[i] * h1;
        H[(size_t)(i + 1) * m + j] = -sn[i] * h0 + cs[i] * h1;
      }
      const double h0 = H[(size_t)j * m + j], h1 = H[(size_t)(j + 1) * m + j];
      const double d = std::hypot(h0, h1);
      cs[j] = d > 0 ? h0 / d : 1.0;
      sn[j] = d > 0 ? h1 / d : 0.0;
      H[(size_t)j * m + j] = d;
      H[(size_t)(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rel = std::fabs(g[j + 1]) / bn;
      if (rel <= tol || rel * bn <= tol_abs || hn == 0.0) {
        ++j;
        break;
      }
    }
    for (int i = j - 1; i >= 0; --i) {
      double acc = g[i];
      for (int k = i + 1; k < j; ++k) acc -= H[(size_t)i * m + k] * y[k];
      y[i] = acc / H[(size_t)i * m + i];
    }
    for (int i = 0; i < j; ++i) HHG_TRY(launch_axpby(n, y[i], Z[i], 1.0, x, s));
  }
  if (bn > 0) {  // true residual
    HHG_TRY(op(x, w));
    HHG_TRY(launch_axpby(n, 1.0, b, -1.0, w, s));
    double rr = 0.0;
    HHG_TRY(dot(w, w, &rr));
    rel = std::sqrt(rr) / bn;
  }
  if (iters_out) *iters_out = total;
  if (rel_out) *rel_out = rel;
  return HHG_OK;
}
}  // namespace

struct hhg_temp_solver {
  hhg_mesh* mesh = nullptr;
  int level = 0, restart = 0;
  hhg_temp_params prm{};
  int64_t n = 0;
  std::vector<double*> V, Z;
  double *w = nullptr, *td = nullptr, *bp = nullptr, *dl = nullptr, *dinv = nullptr, *t1 = nullptr;
  double *cr = nullptr, *cz = nullptr, *cp = nullptr, *cq = nullptr, *sc = nullptr;
  double* red = nullptr;  // reduction scratch of this object
  ~hhg_temp_solver() {
    if (mesh) --mesh->dependents;
    for (double* p : V) cudaFree(p);
    for (double* p : Z) cudaFree(p);
    for (double* p : {w, td, bp, dl, dinv, t1, cr, cz, cp, cq, sc, red})
      if (p) cudaFree(p);
  }
};

extern "C" {
int hhg_temp_apply(const hhg_mesh* mesh, int level, const hhg_temp_params* prm, const double* u, const double* T,
                   double* y, int which, hhg_stream_t stream) {
  if (!mesh || !prm || !y || (which != 2 && !T) || (which == 0 && !u)) return fail(HHG_EINVAL, "hhg_temp_apply: NULL argument");
  if (which < 0 || which > 2) return fail(HHG_EINVAL, "hhg_temp_apply: which must be 0, 1 or 2");
  if (level < 0 || level > mesh->level_max) return fail(HHG_ELEVEL, "hhg_temp_apply: bad level");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return temp_apply_raw(m, level, *prm, u, T, y, which, (cudaStream_t)stream);
}

int hhg_temp_solver_create(hhg_mesh* mesh, int level, const hhg_temp_params* prm, int restart, hhg_temp_solver** out) {
  if (!mesh || !prm || !out) return fail(HHG_EINVAL, "hhg_temp_solver_create: NULL argument");
  if (level < 0 || level > mesh->level_max) return fail(HHG_ELEVEL, "hhg_temp_solver_create: bad level");
  if (restart < 1) return fail(HHG_EINVAL, "hhg_temp_solver_create: restart >= 1");
  HHG_TRY(ensure_level(mesh, level));
  auto* S = new hhg_temp_solver();
  S->mesh = mesh;
  S->level = level;
  S->prm = *prm;
  S->restart = restart;
  S->n = macro_count(mesh) * mesh->levels[level].npts2;
  auto alloc = [&](double** p) { return cudaMalloc(p, std::max<int64_t>(S->n, 1) * sizeof(double)) == cudaSuccess; };
  bool ok = true;
  S->V.resize(restart + 1, nullptr);
  S->Z.resize(restart, nullptr);
  for (auto& p : S->V) ok = ok && alloc(&p);
  for (auto& p : S->Z) ok = ok && alloc(&p);
  for (double** p : {&S->w, &S->td, &S->bp, &S->dl, &S->dinv, &S->t1, &S->cr, &S->cz, &S->cp, &S->cq}) ok = ok && alloc(p);
  ok = ok && cudaMalloc(&S->sc, 16 * sizeof(double)) == cudaSuccess && red_alloc(&S->red) == HHG_OK;
  ++mesh->dependents;
  if (!ok) {
    delete S;
    return fail(HHG_ENOMEM, "hhg_temp_solver_create: workspace");
  }
  int r = temp_apply_raw(mesh, level, S->prm, nullptr, nullptr, S->dinv, 2, nullptr);
  if (r == HHG_OK) r = launch_recip(S->n, S->dinv, nullptr);
  if (r == HHG_OK && cudaDeviceSynchronize() != cudaSuccess) r = fail(HHG_ECUDA, "hhg_temp_solver_create: sync");
  if (r != HHG_OK) {
    delete S;
    return r;
  }
  *out = S;
  return HHG_OK;
}

int hhg_temp_solve(hhg_temp_solver* S, const double* u, const double* b, double* T, double tol, double tol_abs,
                   int max_iters, double tol_cg, int cg_max_iters, int* iters, double* rel_res, hhg_stream_t stream) {
  if (!S || !u || !b || !T) return fail(HHG_EINVAL, "hhg_temp_solve: NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const Mesh* m = S->mesh;
  const Level& L = m->levels[S->level];
  const int64_t n = S->n;
  const unsigned nb = vg(n);
  auto mask = [&](const double* in, double* out, int keep_bnd) -> int {
    k_mask<<<nb, 256, 0, s>>>(n, L.bcn2, keep_bnd, in, out);
    count_launch();
    return HHG_OK;
  };
  auto dot = [&](const double* x, const double* y, double* out) -> int {
    HHG_TRY(launch_dot(m, L, HHG_P2, x, y, S->sc + 8, s, S->red));
    HHG_CUDA(cudaMemcpyAsync(out, S->sc + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
    HHG_CUDA(cudaStreamSynchronize(s));
    return HHG_OK;
  };
  auto opL = [&](const double* x, double* y) -> int {
    HHG_TRY(temp_apply_raw(m, S->level, S->prm, u, x, y, 0, s));
    return mask(y, y, 0);
  };
  auto opP = [&](const double* x, double* y) -> int {
    HHG_TRY(temp_apply_raw(m, S->level, S->prm, nullptr, x, y, 1, s));
    return mask(y, y, 0);
  };
  auto jac = [&](const double* r, double* z) -> int {
    HHG_TRY(launch_pcg_scale(n, S->dinv, r, z, s));
    return mask(z, z, 0);
  };
  auto prec = [&](const double* r, double* z) -> int {
    int it;
    double rel;
    return dev_pcg(m, L, HHG_P2, n, opP, jac, std::function<int(double*)>(), r, z, tol_cg, 0.0, cg_max_iters, S->cr,
                   S->cz, S->cp, S->cq, S->sc, S->red, s, &it, &rel, kCheckEvery, S->sc + 8);
  };
  // T_D on the boundary, b' = mask_int(b - L T_D)
  HHG_TRY(mask(T, S->td, 1));
  HHG_TRY(temp_apply_raw(m, S->level, S->prm, u, S->td, S->t1, 0, s));
  HHG_TRY(launch_axpby(n, 1.0, b, -1.0, S->t1, s));
  HHG_TRY(mask(S->t1, S->bp, 0));
  HHG_TRY(fgmres(n, S->restart, max_iters, tol, tol_abs, opL, prec, dot, S->V, S->Z, S->w, S->bp, S->dl, s, iters,
                 rel_res));
  // T = T_D + delta
  HHG_CUDA(cudaMemcpyAsync(T, S->td, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  HHG_TRY(launch_axpby(n, 1.0, S->dl, 1.0, T, s));
  HHG_CUDA(cudaStreamSynchronize(s));
  return HHG_OK;
}

int hhg_mmoc(const hhg_mesh* mesh, int level, const double* T, const double* u_new, const double* u_old, double tau,
             double* T_hat, hhg_stream_t stream) {
  if (!mesh || !T || !u_new || !u_old || !T_hat) return fail(HHG_EINVAL, "hhg_mmoc: NULL argument");
  if (level < 0 || level > mesh->level_max) return fail(HHG_ELEVEL, "hhg_mmoc: bad level");
  if (mesh->nranks > 1)  // particles may leave the rank's macros: would need a macro halo (not built)
    return fail(HHG_EINVAL, "hhg_mmoc: single-rank meshes only");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  const Level& L = m->levels[level];
  cudaStream_t s = (cudaStream_t)stream;
  double rmin = 1e300, rmax = 0.0;
  for (int64_t v = 0; v < m->n_vert; ++v) {
    const double r = std::sqrt(m->xyz[3 * v] * m->xyz[3 * v] + m->xyz[3 * v + 1] * m->xyz[3 * v + 1] +
                               m->xyz[3 * v + 2] * m->xyz[3 * v + 2]);
    rmin = std::min(rmin, r);
    rmax = std::max(rmax, r);
  }
  int* flag = reinterpret_cast<int*>(L.red + kRedBlocks + 6);
  HHG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  HHG_CUDA(cudaMemsetAsync(T_hat, 0, macro_count(m) * L.npts2 * sizeof(double), s));
  HHG_TRY(launch_mmoc(m, L, rmin, rmax, tau, T, u_new, u_old, T_hat, flag, s));
  HHG_TRY(launch_fixup(m, L, HHG_P2, true, false, T_hat, s));  // owner values to every copy
  int h = 0;
  HHG_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  HHG_CUDA(cudaStreamSynchronize(s));
  if (h) return fail(HHG_EINVAL, "hhg_mmoc: a back-tracked point could not be located in the mesh");
  return HHG_OK;
}

int hhg_temp_solver_destroy(hhg_temp_solver* S) {
  delete S;
  return HHG_OK;
}
}  // extern "C"
