// extern "C" entry points of libhhgstokes.so (include/hhg_stokes.h).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>

#include "hhg_internal.h"

namespace hhg {
const char* last_error();
int64_t launches(int reset);
int mesh_set_geometry(Mesh* m);
int canonical_count(const Mesh* m, int N, int64_t* n);
int canonical_keys(const Mesh* m, int N, int64_t* keys);
int comm_allreduce_sum(hhg_comm* c, double* buf, int64_t n, cudaStream_t s);
}  // namespace hhg

using namespace hhg;

#define CHECK_PTR(p) \
  if (!(p)) return fail(HHG_EINVAL, std::string(__func__) + ": NULL argument " #p)

static int check_level(const hhg_mesh* m, int level) {
  if (!m) return fail(HHG_EINVAL, "NULL mesh");
  if (level < 0 || level > m->level_max) return fail(HHG_ELEVEL, "level outside [0, level_max]");
  return HHG_OK;
}

static int vec_len(const Mesh* m, const Level& L, int space, int64_t* n) {
  const int64_t nm = macro_count(m);
  switch (space) {
    case HHG_P1: *n = nm * L.npts1; return HHG_OK;
    case HHG_P2: *n = nm * L.npts2; return HHG_OK;
    case HHG_P2VEC: *n = 3 * nm * L.npts2; return HHG_OK;
  }
  return fail(HHG_EINVAL, "bad space");
}

extern "C" {

const char* hhg_last_error(void) { return last_error(); }

const char* hhg_version(void) {
  return "libhhgstokes 0.1 (sm_100a, fp64, " __DATE__ ")";
}

int64_t hhg_launch_count(int reset) { return launches(reset); }

static int mesh_create_impl(const double* macro_xyz, int64_t n_vert, const int32_t* macro_tets, int64_t n_tets,
                            const int32_t* vertex_tag, int level_max, const int32_t* tet_rank, int nranks, int rank,
                            hhg_comm* comm, hhg_mesh** out) {
  CHECK_PTR(macro_xyz);
  CHECK_PTR(macro_tets);
  CHECK_PTR(out);
  *out = nullptr;
  if (n_vert < 4 || n_tets < 1) return fail(HHG_EINVAL, "need >= 4 vertices and >= 1 tet");
  if (level_max < 0 || level_max > 8) return fail(HHG_EINVAL, "level_max must be in [0, 8]");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HHG_EINVAL, "bad rank / nranks");
  if (nranks > 1 && !tet_rank) return fail(HHG_EINVAL, "a partitioned mesh needs tet_rank");
  auto* m = new hhg_mesh();
  m->n_vert = n_vert;
  m->n_tets = n_tets;
  m->xyz.assign(macro_xyz, macro_xyz + 3 * n_vert);
  m->tets.assign(macro_tets, macro_tets + 4 * n_tets);
  m->vtag.assign(n_vert, 0);
  if (vertex_tag) m->vtag.assign(vertex_tag, vertex_tag + n_vert);
  for (int64_t t = 0; t < n_tets; ++t) {
    int32_t* v = &m->tets[4 * t];
    std::sort(v, v + 4);
    for (int a = 0; a < 4; ++a)
      if (v[a] < 0 || v[a] >= n_vert || (a > 0 && v[a] == v[a - 1])) {
        delete m;
        return fail(HHG_EINVAL, "bad macro tet vertex ids");
      }
  }
  m->level_max = level_max;
  m->comm = comm;
  m->rank = rank;
  m->nranks = nranks;
  m->tet_rank.assign(n_tets, 0);
  if (tet_rank) m->tet_rank.assign(tet_rank, tet_rank + n_tets);
  for (int64_t t = 0; t < n_tets; ++t) {
    if (m->tet_rank[t] < 0 || m->tet_rank[t] >= nranks) {
      delete m;
      return fail(HHG_EINVAL, "tet_rank entry outside [0, nranks)");
    }
    if (m->tet_rank[t] == m->rank) m->local.push_back(t);
  }
  if (cudaGetDevice(&m->device) != cudaSuccess) {
    m->device = -1;  // host-only use (keys, lengths, plans) is still valid without a GPU
    cudaGetLastError();
  }
  m->levels.resize(level_max + 1);
  for (int l = 0; l <= level_max; ++l) m->levels[l].level = l;
  int r = mesh_set_geometry(m);
  if (r != HHG_OK) {
    delete m;
    return r;
  }
  *out = m;
  return HHG_OK;
}

int hhg_mesh_create(const double* macro_xyz, int64_t n_vert, const int32_t* macro_tets, int64_t n_tets,
                    const int32_t* vertex_tag, int level_max, const int32_t* tet_rank, hhg_comm* comm,
                    hhg_mesh** out) {
  const int nranks = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
  if (!comm && tet_rank) {
    for (int64_t t = 0; t < n_tets; ++t)
      if (tet_rank[t] != 0) return fail(HHG_EINVAL, "tet_rank without a communicator: use hhg_mesh_create_part");
  }
  return mesh_create_impl(macro_xyz, n_vert, macro_tets, n_tets, vertex_tag, level_max, tet_rank, nranks, rank, comm,
                          out);
}

int hhg_mesh_create_part(const double* macro_xyz, int64_t n_vert, const int32_t* macro_tets, int64_t n_tets,
                         const int32_t* vertex_tag, int level_max, const int32_t* tet_rank, int nranks, int rank,
                         hhg_mesh** out) {
  CHECK_PTR(tet_rank);
  return mesh_create_impl(macro_xyz, n_vert, macro_tets, n_tets, vertex_tag, level_max, tet_rank, nranks, rank,
                          nullptr, out);
}

int hhg_partition_rcb(const double* macro_xyz, int64_t n_vert, const int32_t* macro_tets, int64_t n_tets,
                      int nparts, int radial, int32_t* tet_rank) {
  CHECK_PTR(macro_xyz);
  CHECK_PTR(macro_tets);
  CHECK_PTR(tet_rank);
  if (nparts < 1 || nparts > n_tets) return fail(HHG_EINVAL, "nparts must be in [1, n_tets]");
  // macro centroids (radial != 0: projected to the unit sphere, so radial columns stay together)
  std::vector<std::array<double, 3>> c(n_tets);
  for (int64_t t = 0; t < n_tets; ++t) {
    double x[3] = {0, 0, 0};
    for (int a = 0; a < 4; ++a)
      for (int r = 0; r < 3; ++r) x[r] += 0.25 * macro_xyz[3 * macro_tets[4 * t + a] + r];
    if (radial) {
      const double nr = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
      for (int r = 0; r < 3; ++r) x[r] = nr > 0 ? x[r] / nr : 0.0;
    }
    c[t] = {x[0], x[1], x[2]};
  }
  std::vector<int64_t> idx(n_tets);
  for (int64_t t = 0; t < n_tets; ++t) idx[t] = t;
  // recursive bisection along the widest coordinate; part sizes proportional to part counts
  std::function<void(int64_t, int64_t, int, int)> rec = [&](int64_t b, int64_t e, int p0, int np) {
    if (np == 1) {
      for (int64_t i = b; i < e; ++i) tet_rank[idx[i]] = p0;
      return;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t i = b; i < e; ++i)
      for (int r = 0; r < 3; ++r) {
        lo[r] = std::min(lo[r], c[idx[i]][r]);
        hi[r] = std::max(hi[r], c[idx[i]][r]);
      }
    int ax = 0;
    for (int r = 1; r < 3; ++r)
      if (hi[r] - lo[r] > hi[ax] - lo[ax]) ax = r;
    const int nl = np / 2;
    const int64_t mid = b + (e - b) * nl / np;
    std::stable_sort(idx.begin() + b, idx.begin() + e, [&](int64_t x, int64_t y) {
      if (c[x][ax] != c[y][ax]) return c[x][ax] < c[y][ax];
      return x < y;
    });
    rec(b, mid, p0, nl);
    rec(mid, e, p0 + nl, np - nl);
  };
  rec(0, n_tets, 0, nparts);
  return HHG_OK;
}

int hhg_mesh_destroy(hhg_mesh* mesh) {
  delete mesh;
  return HHG_OK;
}

int hhg_mesh_local_macros(const hhg_mesh* mesh, int64_t* n) {
  CHECK_PTR(mesh);
  CHECK_PTR(n);
  *n = macro_count(mesh);
  return HHG_OK;
}

static void invalidate(hhg_mesh* m) {
  for (auto& L : m->levels) free_level(L);
}

static int check_no_dependents(const hhg_mesh* m, const char* what) {
  if (m->dependents > 0)
    return fail(HHG_EINVAL, std::string(what) + ": " + std::to_string(m->dependents) +
                                " solver object(s) (hhg_mg / hhg_kmg / hhg_stokes / hhg_temp_solver) still use this mesh; "
                                "destroy them first (their diagonals, spectra and captured graphs depend on it)");
  return HHG_OK;
}

int blend_map(hhg_mesh* mesh, int kind) {
  CHECK_PTR(mesh);
  if (kind != HHG_BLEND_IDENTITY && kind != HHG_BLEND_SHELL) return fail(HHG_EINVAL, "bad blending kind");
  HHG_TRY(check_no_dependents(mesh, "blend_map"));
  int old = mesh->blend;
  mesh->blend = kind;
  int r = mesh_set_geometry(mesh);
  if (r != HHG_OK) {
    mesh->blend = old;
    mesh_set_geometry(mesh);
    return r;
  }
  return HHG_OK;
}

int hhg_mesh_prepare(hhg_mesh* mesh) {
  CHECK_PTR(mesh);
  for (int l = 0; l <= mesh->level_max; ++l) HHG_TRY(ensure_level(mesh, l));
  return HHG_OK;
}

int hhg_set_deterministic(hhg_mesh* mesh, int on) {
  CHECK_PTR(mesh);
  HHG_TRY(check_no_dependents(mesh, "hhg_set_deterministic"));
  mesh->deterministic = on != 0;
  return HHG_OK;
}

int hhg_set_bc(hhg_mesh* mesh, int tag, int kind) {
  CHECK_PTR(mesh);
  if (kind < HHG_BC_NONE || kind > HHG_BC_FREESLIP) return fail(HHG_EINVAL, "bad BC kind");
  HHG_TRY(check_no_dependents(mesh, "hhg_set_bc"));
  if (tag == HHG_BND_ALL) {
    mesh->bc_kind[0] = mesh->bc_kind[1] = mesh->bc_kind[2] = kind;
  } else if (tag == HHG_BND_INNER || tag == HHG_BND_OUTER) {
    mesh->bc_kind[tag] = kind;
  } else {
    return fail(HHG_EINVAL, "bad boundary tag");
  }
  invalidate(mesh);
  return HHG_OK;
}

int hhg_vec_len(const hhg_mesh* mesh, int level, int space, int64_t* n) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(n);
  const int64_t nm = macro_count(mesh);
  const int64_t n1 = 1LL << level;
  switch (space) {
    case HHG_P1: *n = nm * npts3(n1); return HHG_OK;
    case HHG_P2: *n = nm * npts3(2 * n1); return HHG_OK;
    case HHG_P2VEC: *n = 3 * nm * npts3(2 * n1); return HHG_OK;
  }
  return fail(HHG_EINVAL, "bad space");
}

int hhg_canonical_len(const hhg_mesh* mesh, int level, int space, int64_t* n_unique) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(n_unique);
  if (space != HHG_P1 && space != HHG_P2 && space != HHG_P2VEC) return fail(HHG_EINVAL, "bad space");
  int N = (space == HHG_P1 ? 1 : 2) << level;
  HHG_TRY(canonical_count(mesh, N, n_unique));
  if (space == HHG_P2VEC) *n_unique *= 3;
  return HHG_OK;
}

int hhg_canonical_keys(const hhg_mesh* mesh, int level, int space, int64_t* keys_host) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(keys_host);
  if (space != HHG_P1 && space != HHG_P2) return fail(HHG_EINVAL, "keys: space must be HHG_P1 or HHG_P2");
  int N = (space == HHG_P1 ? 1 : 2) << level;
  return canonical_keys(mesh, N, keys_host);
}

static int canon_io(const hhg_mesh* mesh, int level, int space, const double* src, double* dst, bool to,
                    cudaStream_t s) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(src);
  CHECK_PTR(dst);
  if (space != HHG_P1 && space != HHG_P2 && space != HHG_P2VEC) return fail(HHG_EINVAL, "bad space");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_canon(m, level, space == HHG_P1 ? HHG_P1 : HHG_P2));
  const Level& L = m->levels[level];
  const int64_t nst = macro_count(m) * (space == HHG_P1 ? L.npts1 : L.npts2);
  return launch_gather_canon(L, space, nst, src, dst, to, s);
}

int hhg_to_canonical(const hhg_mesh* mesh, int level, int space, const double* v_dev, double* c_dev,
                     hhg_stream_t stream) {
  return canon_io(mesh, level, space, v_dev, c_dev, true, (cudaStream_t)stream);
}

int hhg_from_canonical(const hhg_mesh* mesh, int level, int space, const double* c_dev, double* v_dev,
                       hhg_stream_t stream) {
  return canon_io(mesh, level, space, c_dev, v_dev, false, (cudaStream_t)stream);
}

int hhg_node_coords(const hhg_mesh* mesh, int level, int space, double* xyz_dev, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(xyz_dev);
  if (space != HHG_P1 && space != HHG_P2) return fail(HHG_EINVAL, "coords: space must be HHG_P1 or HHG_P2");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return launch_coords(m, m->levels[level], space, xyz_dev, (cudaStream_t)stream);
}

int hhg_apply_bc(const hhg_mesh* mesh, int level, double* u, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(u);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return launch_fixup(m, m->levels[level], HHG_P2VEC, false, true, u, (cudaStream_t)stream);
}

int hhg_interface_sum(const hhg_mesh* mesh, int level, int space, double* v, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(v);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return launch_fixup(m, m->levels[level], space, true, space == HHG_P2VEC, v, (cudaStream_t)stream);
}

}  // extern "C"

// ------------------------------------------------------------------ operators
namespace hhg {
// y_u/y_p = op(u, p) on level L, zeroing the outputs, interface sum + BC.
int apply_op(const Mesh* m, int level, int mode, int form, const double* eta, double gamma, const double* u,
             const double* p, double* yu, double* yp, bool accumulate_u, cudaStream_t s) {
  const Level& L = m->levels[level];
  const int64_t nm = macro_count(m);
  const bool has_u = elem_u_out(mode);
  const bool has_p = elem_p_out(mode);
  if (has_u && !accumulate_u) HHG_CUDA(cudaMemsetAsync(yu, 0, 3 * nm * L.npts2 * sizeof(double), s));
  if (has_p) HHG_CUDA(cudaMemsetAsync(yp, 0, nm * L.npts1 * sizeof(double), s));
  if (has_u && accumulate_u) {
    // accumulate into a consistent yu: keep only the owner copy so the interface sum counts it once
    return fail(HHG_EINVAL, "accumulate mode is implemented in divT_apply only");
  }
  HHG_TRY(launch_elem(m, L, mode, form, eta, gamma, u, p, yu, yp, s));
  if (has_u) HHG_TRY(launch_fixup(m, L, HHG_P2VEC, true, mode != ELEM_DIAG, yu, s));
  if (has_p) HHG_TRY(launch_fixup(m, L, HHG_P1, true, false, yp, s));
  return HHG_OK;
}

// radius of the outer boundary sphere (D_eta of the w-BFBT scaling): max |x| over outer-tagged vertices
static double r_outer(const Mesh* m) {
  double r = 0.0;
  for (int64_t v = 0; v < m->n_vert; ++v)
    if (m->vtag[v] == HHG_BND_OUTER)
      r = std::max(r, std::sqrt(m->xyz[3 * v] * m->xyz[3 * v] + m->xyz[3 * v + 1] * m->xyz[3 * v + 1] +
                                m->xyz[3 * v + 2] * m->xyz[3 * v + 2]));
  return r > 0.0 ? r : 1e300;
}

// w-BFBT operators: element kernel + interface sum (+ P_v M for the vector mass apply)
int surf_op(const Mesh* m, int level, int mode, const double* eta, double a, const double* in, double* out,
            cudaStream_t s) {
  const Level& L = m->levels[level];
  const int64_t nm = macro_count(m);
  const bool vec = (mode & (ELEM_VMASS | ELEM_VMASSD)) != 0;
  HHG_CUDA(cudaMemsetAsync(out, 0, (vec ? 3 * nm * L.npts2 : nm * L.npts1) * sizeof(double), s));
  HHG_TRY(launch_elem_surf(m, L, mode, eta, a, r_outer(m), in, out, s));
  return launch_fixup(m, L, vec ? HHG_P2VEC : HHG_P1, true, mode == ELEM_VMASS, out, s);
}
}  // namespace hhg

extern "C" {

int epsilon_apply(const hhg_mesh* mesh, int level, int form, const double* eta_p1, const double* u, double* y,
                  hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(u);
  CHECK_PTR(y);
  if (form != HHG_VISC_FULL && form != HHG_VISC_EPS) return fail(HHG_EINVAL, "bad viscous form");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return apply_op(m, level, ELEM_A, form, eta_p1, 0.0, u, nullptr, y, nullptr, false, (cudaStream_t)stream);
}

int epsilon_apply_qeta(const hhg_mesh* mesh, int level, const double* T_p2, double lnC, double jump, double r_jump,
                       const double* u, double* y, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(T_p2);
  CHECK_PTR(u);
  CHECK_PTR(y);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  const Level& L = m->levels[level];
  cudaStream_t s = (cudaStream_t)stream;
  HHG_CUDA(cudaMemsetAsync(y, 0, 3 * macro_count(m) * L.npts2 * sizeof(double), s));
  HHG_TRY(launch_elem_qeta(m, L, ELEM_A, T_p2, lnC, jump, r_jump, u, y, s));
  return launch_fixup(m, L, HHG_P2VEC, true, true, y, s);
}

int hhg_diag_qeta(const hhg_mesh* mesh, int level, const double* T_p2, double lnC, double jump, double r_jump,
                  double* diag, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(T_p2);
  CHECK_PTR(diag);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  const Level& L = m->levels[level];
  cudaStream_t s = (cudaStream_t)stream;
  HHG_CUDA(cudaMemsetAsync(diag, 0, 3 * macro_count(m) * L.npts2 * sizeof(double), s));
  HHG_TRY(launch_elem_qeta(m, L, ELEM_DIAG, T_p2, lnC, jump, r_jump, nullptr, diag, s));
  return launch_fixup(m, L, HHG_P2VEC, true, false, diag, s);
}

int hhg_mass_apply(const hhg_mesh* mesh, int level, const double* eta_p1, const double* p, double* y,
                   hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(p);
  CHECK_PTR(y);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return apply_op(m, level, ELEM_MASS, HHG_VISC_FULL, eta_p1, 0.0, nullptr, p, nullptr, y, false, (cudaStream_t)stream);
}

int hhg_buoyancy_load(const hhg_mesh* mesh, int level, const double* T_p1, double* f, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(T_p1);
  CHECK_PTR(f);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return apply_op(m, level, ELEM_LOAD, HHG_VISC_FULL, nullptr, 0.0, nullptr, T_p1, f, nullptr, false, (cudaStream_t)stream);
}

int hhg_mass_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double* diag, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(diag);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return apply_op(m, level, ELEM_MASSD, HHG_VISC_FULL, eta_p1, 0.0, nullptr, nullptr, nullptr, diag, false,
                  (cudaStream_t)stream);
}

int hhg_kp1_apply(const hhg_mesh* mesh, int level, const double* eta_p1, double a, const double* p, double* y,
                  hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(p);
  CHECK_PTR(y);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return surf_op(m, level, ELEM_KP1, eta_p1, a, p, y, (cudaStream_t)stream);
}

int hhg_kp1_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double a, double* diag, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(diag);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return surf_op(m, level, ELEM_KP1D, eta_p1, a, nullptr, diag, (cudaStream_t)stream);
}

int hhg_vmass_apply(const hhg_mesh* mesh, int level, const double* eta_p1, double a, const double* u, double* y,
                    hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(u);
  CHECK_PTR(y);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return surf_op(m, level, ELEM_VMASS, eta_p1, a, u, y, (cudaStream_t)stream);
}

int hhg_vmass_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double a, double* diag,
                   hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(diag);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return surf_op(m, level, ELEM_VMASSD, eta_p1, a, nullptr, diag, (cudaStream_t)stream);
}

int p1_prolong(const hhg_mesh* mesh, int coarse_level, const double* x_coarse, double* x_fine, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, coarse_level));
  if (coarse_level + 1 > mesh->level_max) return fail(HHG_ELEVEL, "p1_prolong: coarse_level must be < level_max");
  CHECK_PTR(x_coarse);
  CHECK_PTR(x_fine);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, coarse_level));
  HHG_TRY(ensure_level(m, coarse_level + 1));
  return launch_p1_prolong(m, m->levels[coarse_level], m->levels[coarse_level + 1], x_coarse, x_fine,
                           (cudaStream_t)stream);
}

int p1_restrict(const hhg_mesh* mesh, int fine_level, const double* r_fine, double* r_coarse, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, fine_level));
  if (fine_level < 1) return fail(HHG_ELEVEL, "p1_restrict: fine_level must be >= 1");
  CHECK_PTR(r_fine);
  CHECK_PTR(r_coarse);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, fine_level));
  HHG_TRY(ensure_level(m, fine_level - 1));
  const Level& Lc = m->levels[fine_level - 1];
  cudaStream_t s = (cudaStream_t)stream;
  HHG_TRY(launch_p1_restrict(m, Lc, m->levels[fine_level], r_fine, r_coarse, s));
  return launch_fixup(m, Lc, HHG_P1, true, false, r_coarse, s);
}

int div_apply(const hhg_mesh* mesh, int level, double gamma, const double* u, double* q, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(u);
  CHECK_PTR(q);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return apply_op(m, level, ELEM_DIV, HHG_VISC_FULL, nullptr, gamma, u, nullptr, nullptr, q, false,
                  (cudaStream_t)stream);
}

int divT_apply(const hhg_mesh* mesh, int level, const double* p, double* y_u, int accumulate, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(p);
  CHECK_PTR(y_u);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  cudaStream_t s = (cudaStream_t)stream;
  if (!accumulate) return apply_op(m, level, ELEM_BT, HHG_VISC_FULL, nullptr, 0.0, nullptr, p, y_u, nullptr, false, s);
  // y_u += (M P_v) B^T p: into the level's scratch vector (allocated on first use), then added
  Level& L = m->levels[level];
  const int64_t n = 3 * macro_count(m) * L.npts2;
  if (!L.scratch_u && cudaMalloc(&L.scratch_u, n * sizeof(double)) != cudaSuccess)
    return fail(HHG_ENOMEM, "divT_apply scratch");
  HHG_TRY(apply_op(m, level, ELEM_BT, HHG_VISC_FULL, nullptr, 0.0, nullptr, p, L.scratch_u, nullptr, false, s));
  return launch_axpby(n, 1.0, L.scratch_u, 1.0, y_u, s);
}

int stokes_apply(const hhg_mesh* mesh, int level, const double* eta_p1, double gamma, const double* u,
                 const double* p, double* y_u, double* y_p, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(u);
  CHECK_PTR(p);
  CHECK_PTR(y_u);
  CHECK_PTR(y_p);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return apply_op(m, level, ELEM_A | ELEM_BT | ELEM_DIV, HHG_VISC_FULL, eta_p1, gamma, u, p, y_u, y_p, false,
                  (cudaStream_t)stream);
}

int hhg_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double* diag, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(diag);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return apply_op(m, level, ELEM_DIAG, HHG_VISC_FULL, eta_p1, 0.0, nullptr, nullptr, diag, nullptr, false,
                  (cudaStream_t)stream);
}

int hhg_dot(const hhg_mesh* mesh, int level, int space, const double* x, const double* y, double* out_dev,
            hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(x);
  CHECK_PTR(y);
  CHECK_PTR(out_dev);
  if (space != HHG_P1 && space != HHG_P2 && space != HHG_P2VEC) return fail(HHG_EINVAL, "bad space");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return launch_dot(m, m->levels[level], space, x, y, out_dev, (cudaStream_t)stream, m->levels[level].red);
}

int p2_restrict(const hhg_mesh* mesh, int fine_level, const double* r_fine, double* r_coarse, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, fine_level));
  if (fine_level < 1) return fail(HHG_ELEVEL, "p2_restrict: fine_level must be >= 1");
  CHECK_PTR(r_fine);
  CHECK_PTR(r_coarse);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, fine_level));
  HHG_TRY(ensure_level(m, fine_level - 1));
  const Level& Lf = m->levels[fine_level];
  const Level& Lc = m->levels[fine_level - 1];
  cudaStream_t s = (cudaStream_t)stream;
  HHG_TRY(launch_restrict(m, Lc, Lf, r_fine, r_coarse, s));
  return launch_fixup(m, Lc, HHG_P2VEC, true, true, r_coarse, s);
}

int p2_prolong(const hhg_mesh* mesh, int coarse_level, const double* x_coarse, double* x_fine, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, coarse_level));
  if (coarse_level + 1 > mesh->level_max) return fail(HHG_ELEVEL, "p2_prolong: coarse_level must be < level_max");
  CHECK_PTR(x_coarse);
  CHECK_PTR(x_fine);
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, coarse_level));
  HHG_TRY(ensure_level(m, coarse_level + 1));
  cudaStream_t s = (cudaStream_t)stream;
  const Level& Lc = m->levels[coarse_level];
  const Level& Lf = m->levels[coarse_level + 1];
  HHG_TRY(launch_prolong(m, Lc, Lf, x_coarse, x_fine, s));
  return launch_fixup(m, Lf, HHG_P2VEC, false, true, x_fine, s);
}


// ------------------------------------------------------------------ partitioned meshes (multi-GPU)
int hhg_mesh_rank(const hhg_mesh* mesh, int* rank, int* nranks) {
  CHECK_PTR(mesh);
  if (rank) *rank = mesh->rank;
  if (nranks) *nranks = mesh->nranks;
  return HHG_OK;
}

static int halo_host(const hhg_mesh* mesh, int level, int space, Halo& H, std::vector<uint8_t>* own_out) {
  HHG_TRY(check_level(mesh, level));
  if (space != HHG_P1 && space != HHG_P2 && space != HHG_P2VEC) return fail(HHG_EINVAL, "bad space");
  std::vector<int64_t> ptr, copy, sg;
  std::vector<uint8_t> kind, own;
  std::vector<double> normal;
  HHG_TRY(build_host_groups(mesh, level, space == HHG_P1 ? HHG_P1 : HHG_P2VEC, ptr, copy, kind, normal, own, H, sg));
  if (own_out) own_out->swap(own);
  return HHG_OK;
}

int hhg_halo_info(const hhg_mesh* mesh, int level, int space, int* n_nbr, int32_t* nbr_ranks, int64_t* counts) {
  CHECK_PTR(n_nbr);
  Halo H;
  HHG_TRY(halo_host(mesh, level, space, H, nullptr));
  *n_nbr = (int)H.nbr.size();
  for (size_t i = 0; i < H.nbr.size(); ++i) {
    if (nbr_ranks) nbr_ranks[i] = H.nbr[i];
    if (counts) counts[i] = H.off[i + 1] - H.off[i];
  }
  return HHG_OK;
}

int hhg_halo_keys(const hhg_mesh* mesh, int level, int space, int64_t* keys_host) {
  CHECK_PTR(keys_host);
  Halo H;
  HHG_TRY(halo_host(mesh, level, space, H, nullptr));
  std::copy(H.keys.begin(), H.keys.end(), keys_host);
  return HHG_OK;
}

int hhg_owned_count(const hhg_mesh* mesh, int level, int space, int64_t* n_owned) {
  CHECK_PTR(n_owned);
  Halo H;
  std::vector<uint8_t> own;
  HHG_TRY(halo_host(mesh, level, space, H, &own));
  int64_t n = 0;
  for (uint8_t o : own) n += o;
  *n_owned = n;
  return HHG_OK;
}

int hhg_halo_pack(const hhg_mesh* mesh, int level, int space, const double* v, double* sendbuf,
                  hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(v);
  CHECK_PTR(sendbuf);
  if (space != HHG_P1 && space != HHG_P2VEC) return fail(HHG_EINVAL, "halo exchange: space must be P1 or P2VEC");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  return launch_halo_pack(m, m->levels[level], space, v, sendbuf, (cudaStream_t)stream);
}

int hhg_interface_sum_remote(const hhg_mesh* mesh, int level, int space, const double* recvbuf, double* v,
                             hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(v);
  if (space != HHG_P1 && space != HHG_P2VEC) return fail(HHG_EINVAL, "halo exchange: space must be P1 or P2VEC");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  const Level& L = m->levels[level];
  if (!recvbuf && (space == HHG_P1 ? L.g1 : L.g2).halo.nslots > 0) return fail(HHG_EINVAL, "NULL recvbuf");
  return launch_fixup_remote(m, L, space, space == HHG_P2VEC, recvbuf, v, (cudaStream_t)stream);
}

int epsilon_apply_partial(const hhg_mesh* mesh, int level, int form, const double* eta_p1, const double* u,
                          double* y, hhg_stream_t stream) {
  HHG_TRY(check_level(mesh, level));
  CHECK_PTR(u);
  CHECK_PTR(y);
  if (form != HHG_VISC_FULL && form != HHG_VISC_EPS) return fail(HHG_EINVAL, "bad viscous form");
  auto* m = const_cast<hhg_mesh*>(mesh);
  HHG_TRY(ensure_level(m, level));
  const Level& L = m->levels[level];
  cudaStream_t s = (cudaStream_t)stream;
  HHG_CUDA(cudaMemsetAsync(y, 0, 3 * macro_count(m) * L.npts2 * sizeof(double), s));
  return launch_elem(m, L, ELEM_A, form, eta_p1, 0.0, u, nullptr, y, nullptr, s);
}

}  // extern "C"

// ------------------------------------------------------------------ icosahedral shell generator
// shell(ntan, nrad) (R4): each icosahedron face split into (ntan-1)^2 flat
// triangles (vertices normalised to the unit sphere, numbered by their sorted (vertex, weight)
// keys), nrad spheres r_l = r_min + l (r_max - r_min)/(nrad-1), every layer prism split into 3 tets
// by the sorted-id staircase rule (p_i,q_i,r_i,r_o), (p_i,q_i,q_o,r_o), (p_i,p_o,q_o,r_o).
namespace {
int icoshell_build(int ntan, int nrad, double r_min, double r_max, std::vector<double>& verts,
                   std::vector<int32_t>& tets, std::vector<int32_t>& vtag) {
  if (ntan < 2 || nrad < 2 || !(0.0 < r_min && r_min < r_max)) return fail(HHG_EINVAL, "icoshell: need ntan>=2, nrad>=2, 0<r_min<r_max");
  const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<std::array<double, 3>> ico;
  for (double s1 : {-1.0, 1.0})
    for (double s2 : {-1.0, 1.0}) {
      ico.push_back({0.0, s1, s2 * phi});
      ico.push_back({s1, s2 * phi, 0.0});
      ico.push_back({s2 * phi, 0.0, s1});
    }
  const int n = (int)ico.size();
  auto dist = [&](int a, int b) {
    double s = 0;
    for (int c = 0; c < 3; ++c) s += (ico[a][c] - ico[b][c]) * (ico[a][c] - ico[b][c]);
    return std::sqrt(s);
  };
  auto adj = [&](int a, int b) { return std::fabs(dist(a, b) - 2.0) < 1e-9; };
  std::vector<std::array<int, 3>> faces;
  for (int a = 0; a < n; ++a)
    for (int b = a + 1; b < n; ++b) {
      if (!adj(a, b)) continue;
      for (int c = b + 1; c < n; ++c)
        if (adj(a, c) && adj(b, c)) faces.push_back({a, b, c});
    }
  if (faces.size() != 20) return fail(HHG_EINVAL, "icoshell: icosahedron face search failed");
  const int m = ntan - 1;
  using Key = std::vector<std::pair<int, int>>;
  std::map<Key, int> key_to_id;
  std::vector<std::array<double, 3>> pts;
  std::vector<std::map<std::pair<int, int>, int>> grids;
  for (auto& f : faces) {
    std::map<std::pair<int, int>, int> grid;
    for (int i = 0; i <= m; ++i)
      for (int j = 0; j <= m - i; ++j) {
        const int wa = m - i - j, wb = i, wc = j;
        Key key;
        for (auto vw : {std::make_pair(f[0], wa), std::make_pair(f[1], wb), std::make_pair(f[2], wc)})
          if (vw.second > 0) key.push_back(vw);
        std::sort(key.begin(), key.end());
        auto it = key_to_id.find(key);
        if (it == key_to_id.end()) {
          it = key_to_id.emplace(key, (int)pts.size()).first;
          std::array<double, 3> p;
          for (int c = 0; c < 3; ++c) p[c] = (wa * ico[f[0]][c] + wb * ico[f[1]][c] + wc * ico[f[2]][c]) / m;
          const double nr = std::sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
          for (int c = 0; c < 3; ++c) p[c] /= nr;
          pts.push_back(p);
        }
        grid[{i, j}] = it->second;
      }
    grids.push_back(grid);
  }
  std::vector<int> remap(pts.size());
  {
    int k = 0;
    for (auto& kv : key_to_id) remap[kv.second] = k++;  // std::map iterates in sorted key order
  }
  const int ns = (int)pts.size();
  std::vector<std::array<int, 3>> tris;
  for (auto& grid : grids)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m - i; ++j) {
        tris.push_back({remap[grid[{i, j}]], remap[grid[{i + 1, j}]], remap[grid[{i, j + 1}]]});
        if (i + j < m - 1) tris.push_back({remap[grid[{i + 1, j}]], remap[grid[{i, j + 1}]], remap[grid[{i + 1, j + 1}]]});
      }
  verts.assign((size_t)ns * nrad * 3, 0.0);
  vtag.assign((size_t)ns * nrad, 0);
  for (int l = 0; l < nrad; ++l) {
    const double r = r_min + l * (r_max - r_min) / (nrad - 1);
    for (int old = 0; old < ns; ++old)
      for (int c = 0; c < 3; ++c) verts[3 * ((size_t)l * ns + remap[old]) + c] = r * pts[old][c];
  }
  for (int v = 0; v < ns; ++v) {
    vtag[v] = 1;                                  // inner sphere (CMB)
    vtag[(size_t)(nrad - 1) * ns + v] = 2;        // outer sphere (surface)
  }
  tets.clear();
  for (int l = 0; l < nrad - 1; ++l)
    for (auto& tri : tris) {
      std::array<int, 3> s = tri;
      std::sort(s.begin(), s.end());
      const int pi = l * ns + s[0], qi = l * ns + s[1], ri = l * ns + s[2];
      const int po = pi + ns, qo = qi + ns, ro = ri + ns;
      for (std::array<int, 4> t : {std::array<int, 4>{pi, qi, ri, ro}, std::array<int, 4>{pi, qi, qo, ro},
                                   std::array<int, 4>{pi, po, qo, ro}}) {
        std::sort(t.begin(), t.end());
        tets.insert(tets.end(), t.begin(), t.end());
      }
    }
  return HHG_OK;
}
}  // namespace

extern "C" {
int hhg_icoshell_macro(int ntan, int nrad, double r_min, double r_max, double* verts, int32_t* tets,
                       int32_t* vtag, int64_t* n_vert, int64_t* n_tets) {
  std::vector<double> v;
  std::vector<int32_t> t, g;
  HHG_TRY(icoshell_build(ntan, nrad, r_min, r_max, v, t, g));
  if (n_vert) *n_vert = (int64_t)g.size();
  if (n_tets) *n_tets = (int64_t)t.size() / 4;
  if (verts) std::copy(v.begin(), v.end(), verts);
  if (tets) std::copy(t.begin(), t.end(), tets);
  if (vtag) std::copy(g.begin(), g.end(), vtag);
  return HHG_OK;
}

int hhg_mesh_create_icoshell(int ntan, int nrad, double r_min, double r_max, int level_max, const int32_t* tet_rank,
                             hhg_comm* comm, hhg_mesh** out) {
  std::vector<double> v;
  std::vector<int32_t> t, g;
  HHG_TRY(icoshell_build(ntan, nrad, r_min, r_max, v, t, g));
  return hhg_mesh_create(v.data(), (int64_t)g.size(), t.data(), (int64_t)t.size() / 4, g.data(), level_max, tet_rank,
                         comm, out);
}
}  // extern "C"
