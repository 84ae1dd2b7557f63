// Host-side setup of the hierarchical hybrid grid: macro primitives, per-level
// element geometry tables, replicated-node groups, owner masks and canonical maps.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <numeric>
#include <set>

#include "hhg_internal.h"

namespace hhg {

static thread_local std::string g_err = "no error";
static thread_local int64_t g_launches = 0;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
const char* last_error() { return g_err.c_str(); }
void count_launch(int n) { g_launches += n; }
int64_t launches(int reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

// The six micro-tet types of one lattice cube (anchor a): vertex offsets (digits = di,dj,dk).
// 0: up {000,100,010,001} (s<=n-1); 1-4: octahedron around diagonal 010-101 (s<=n-2);
// 5: down {011,101,110,111} (s<=n-3).  Identical to the iterated Bey refinement.
const int kTypeVerts[6][4][3] = {
    {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
    {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}},
    {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}},
    {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}},
};

static void inv3(const double* a, double* r, double* det_out) {
  double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
               a[2] * (a[3] * a[7] - a[4] * a[6]);
  double id = 1.0 / det;
  r[0] = (a[4] * a[8] - a[5] * a[7]) * id;
  r[1] = (a[2] * a[7] - a[1] * a[8]) * id;
  r[2] = (a[1] * a[5] - a[2] * a[4]) * id;
  r[3] = (a[5] * a[6] - a[3] * a[8]) * id;
  r[4] = (a[0] * a[8] - a[2] * a[6]) * id;
  r[5] = (a[2] * a[3] - a[0] * a[5]) * id;
  r[6] = (a[3] * a[7] - a[4] * a[6]) * id;
  r[7] = (a[1] * a[6] - a[0] * a[7]) * id;
  r[8] = (a[0] * a[4] - a[1] * a[3]) * id;
  if (det_out) *det_out = det;
}

int64_t macro_count(const Mesh* m) { return (int64_t)m->local.size(); }

void free_level(Level& L) {
  auto f = [](void* p) {
    if (p) cudaFree(p);
  };
  f(L.geo);
  f(L.bricks);
  f(L.bricks_col);
  f(L.rs1);
  f(L.rs2);
  f(L.rows1);
  f(L.rows2);
  for (Groups* g : {&L.g1, &L.g2}) {
    f(g->ptr);
    f(g->copy);
    f(g->kind);
    f(g->normal);
    f(g->halo.slot_group);
    f(g->halo.gs_ptr);
    f(g->halo.gs_idx);
    f(g->halo.sbuf);
    f(g->halo.rbuf);
    *g = Groups();
  }
  f(L.own1);
  f(L.own2);
  f(L.bcn2);
  f(L.gmap2);
  f(L.canon1);
  f(L.canon2);
  f(L.red);
  f(L.scratch_u);
  int lv = L.level;
  L = Level();
  L.level = lv;
}

Mesh::~Mesh() {
  for (auto& L : levels) free_level(L);
  if (dgeo) cudaFree(dgeo);
  for (auto& kv : side) {
    if (kv.second.fork) cudaEventDestroy(kv.second.fork);
    if (kv.second.join) cudaEventDestroy(kv.second.join);
    if (kv.second.s) cudaStreamDestroy(kv.second.s);
  }
}

// ------------------------------------------------------------------ primitives
using Key3 = std::array<int32_t, 3>;  // sorted vertex ids, -1 padded

struct Prims {
  std::map<Key3, std::vector<int64_t>> macros;  // primitive (dim 0..2) -> containing global macros
  std::map<Key3, int> bc;                       // primitive -> BC kind
};

static Key3 mk(int a, int b = -1, int c = -1) { return Key3{a, b, c}; }

static void build_prims(const Mesh* m, Prims& P) {
  for (int64_t t = 0; t < m->n_tets; ++t) {
    const int32_t* v = &m->tets[4 * t];
    for (int a = 0; a < 4; ++a) {
      P.macros[mk(v[a])].push_back(t);
      for (int b = a + 1; b < 4; ++b) {
        P.macros[mk(v[a], v[b])].push_back(t);
        for (int c = b + 1; c < 4; ++c) P.macros[mk(v[a], v[b], v[c])].push_back(t);
      }
    }
  }
  // boundary faces -> BC of all their sub-primitives (Dirichlet dominates)
  for (auto& kv : P.macros) {
    const Key3& f = kv.first;
    if (f[2] < 0 || kv.second.size() != 1) continue;
    int t0 = m->vtag[f[0]], t1 = m->vtag[f[1]], t2 = m->vtag[f[2]];
    int tag = (t0 == t1 && t1 == t2) ? t0 : 0;
    if (tag < 0 || tag > 2) tag = 0;
    int kind = m->bc_kind[tag];
    if (kind == HHG_BC_NONE) continue;
    Key3 subs[7] = {mk(f[0]), mk(f[1]), mk(f[2]), mk(f[0], f[1]), mk(f[0], f[2]), mk(f[1], f[2]), f};
    for (auto& s : subs) {
      auto it = P.bc.find(s);
      if (it == P.bc.end() || kind == HHG_BC_DIRICHLET0) P.bc[s] = kind;
    }
  }
}

// local (i,j,k) at resolution N of the point with weights w[0..d] over primitive ids pid[0..d]
static inline void local_ijk(const int32_t* tv, const int32_t* pid, const int* w, int d, int* ijk) {
  int W[4] = {0, 0, 0, 0};
  for (int r = 0; r <= d; ++r)
    for (int a = 0; a < 4; ++a)
      if (tv[a] == pid[r]) W[a] = w[r];
  ijk[0] = W[1];
  ijk[1] = W[2];
  ijk[2] = W[3];
}

// enumerate interior weight tuples of a (d)-primitive at resolution N, lexicographic
template <class F>
static void for_interior(int d, int N, F&& f) {
  int w[3];
  if (d == 0) {
    w[0] = N;
    f(w);
  } else if (d == 1) {
    for (int a = 1; a <= N - 1; ++a) {
      w[0] = a;
      w[1] = N - a;
      f(w);
    }
  } else {
    for (int a = 1; a <= N - 2; ++a)
      for (int b = 1; b <= N - 1 - a; ++b) {
        w[0] = a;
        w[1] = b;
        w[2] = N - a - b;
        f(w);
      }
  }
}

template <class T>
static int upload(T** dst, const std::vector<T>& src) {
  if (src.empty()) {
    *dst = nullptr;
    return HHG_OK;
  }
  if (cudaMalloc(dst, src.size() * sizeof(T)) != cudaSuccess) return fail(HHG_ENOMEM, "cudaMalloc failed");
  HHG_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return HHG_OK;
}

// Replicated-node groups of one level/space (host): every node that lives on a macro primitive
// held by several local macros, carries a BC, or is shared with another rank gets a group (its
// local copies).  Owner of a node = its copy in the LOWEST GLOBAL macro id containing it (so the
// owner masks of all ranks together count every node once).  Cross-rank slots: for each other
// rank holding the primitive, one slot per interior node, in (primitive key, weight) order.
static void host_groups(const Mesh* m, const Prims& P, int N, bool with_bc, int64_t npts,
                        std::vector<int64_t>& ptr, std::vector<int64_t>& copy, std::vector<uint8_t>& kind,
                        std::vector<double>& normal, std::vector<uint8_t>& own, Halo& halo,
                        std::vector<int64_t>& slot_group) {
  std::vector<int64_t> gl_to_loc(m->n_tets, -1);
  for (size_t i = 0; i < m->local.size(); ++i) gl_to_loc[m->local[i]] = (int64_t)i;
  ptr.assign(1, 0);
  copy.clear();
  kind.clear();
  normal.clear();
  own.assign((size_t)npts * m->local.size(), 1);
  std::map<Key3, int64_t> gstart;
  // two passes: groups carrying a BC first (so BC-only fixups touch just them), then the rest
  for (int pass = 0; pass < 2; ++pass)
    for (auto& kv : P.macros) {
      const Key3& p = kv.first;
      const int d = p[1] < 0 ? 0 : (p[2] < 0 ? 1 : 2);
      std::vector<int64_t> loc;
      bool remote = false;
      for (int64_t t : kv.second) {
        if (gl_to_loc[t] >= 0) loc.push_back(t);
        else remote = true;
      }
      if (loc.empty()) continue;
      int k = HHG_BC_NONE;
      if (with_bc) {
        auto it = P.bc.find(p);
        if (it != P.bc.end()) k = it->second;
      }
      const int64_t owner = kv.second.front();  // macros listed in ascending global id
      if (pass == 0)
        for_interior(d, N, [&](const int* w) {  // owner masks (all replicated nodes, grouped or not)
          for (size_t c = 0; c < loc.size(); ++c) {
            int ijk[3];
            local_ijk(&m->tets[4 * loc[c]], p.data(), w, d, ijk);
            own[gl_to_loc[loc[c]] * npts + lidx(ijk[0], ijk[1], ijk[2], N)] = loc[c] == owner ? 1 : 0;
          }
        });
      if (loc.size() < 2 && k == HHG_BC_NONE && !remote) continue;
      if ((pass == 0) != (k != HHG_BC_NONE)) continue;
      gstart[p] = (int64_t)ptr.size() - 1;
      for_interior(d, N, [&](const int* w) {
        for (size_t c = 0; c < loc.size(); ++c) {
          int ijk[3];
          local_ijk(&m->tets[4 * loc[c]], p.data(), w, d, ijk);
          copy.push_back(gl_to_loc[loc[c]] * npts + lidx(ijk[0], ijk[1], ijk[2], N));
        }
        ptr.push_back((int64_t)copy.size());
        if (with_bc) {
          kind.push_back((uint8_t)k);
          double x[3] = {0, 0, 0};
          for (int r = 0; r <= d; ++r)
            for (int c = 0; c < 3; ++c) x[c] += (double)w[r] / N * m->xyz[3 * p[r] + c];
          double nr = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
          for (int c = 0; c < 3; ++c) normal.push_back(nr > 0 ? x[c] / nr : 0.0);
        }
      });
    }
  // cross-rank slots, neighbor-major, then primitive-key / weight order
  halo = Halo();
  slot_group.clear();
  std::map<int, std::vector<std::pair<int64_t, std::array<int64_t, 10>>>> per;
  for (auto& kv : P.macros) {
    const Key3& p = kv.first;
    auto gs = gstart.find(p);
    if (gs == gstart.end()) continue;
    std::set<int> ranks;
    for (int64_t t : kv.second)
      if (m->tet_rank[t] != m->rank) ranks.insert(m->tet_rank[t]);
    if (ranks.empty()) continue;
    const int d = p[1] < 0 ? 0 : (p[2] < 0 ? 1 : 2);
    int64_t i = 0;
    for_interior(d, N, [&](const int* w) {
      std::array<int64_t, 10> key;
      key[0] = d;
      for (int c = 0; c < 4; ++c) key[1 + c] = c <= d ? p[c] : -1;
      for (int c = 0; c < 4; ++c) key[5 + c] = c <= d ? w[c] : 0;
      key[9] = N;
      for (int q : ranks) per[q].push_back({gs->second + i, key});
      ++i;
    });
  }
  halo.off.push_back(0);
  for (auto& kv : per) {
    halo.nbr.push_back(kv.first);
    for (auto& e : kv.second) {
      slot_group.push_back(e.first);
      halo.keys.insert(halo.keys.end(), e.second.begin(), e.second.end());
    }
    halo.off.push_back((int64_t)slot_group.size());
  }
  halo.nslots = (int64_t)slot_group.size();

  // Memory locality of the interface-sum kernels: within the BC block [0, nbc) and the rest, order
  // the groups by the flat index of their first copy (consecutive threads then walk each macro's
  // boundary storage monotonically).  Slot -> group references are remapped.
  const int64_t ng = (int64_t)ptr.size() - 1;
  int64_t nbc = 0;
  if (with_bc)
    for (uint8_t k : kind) nbc += k != HHG_BC_NONE;
  std::vector<int64_t> order(ng);
  std::iota(order.begin(), order.end(), 0);
  auto by_first = [&](int64_t a, int64_t b) { return copy[ptr[a]] < copy[ptr[b]]; };
  std::stable_sort(order.begin(), order.begin() + nbc, by_first);
  std::stable_sort(order.begin() + nbc, order.end(), by_first);
  std::vector<int64_t> nptr(1, 0), ncopy, newid(ng);
  std::vector<uint8_t> nkind;
  std::vector<double> nnormal;
  ncopy.reserve(copy.size());
  for (int64_t gi = 0; gi < ng; ++gi) {
    const int64_t g = order[gi];
    newid[g] = gi;
    for (int64_t k = ptr[g]; k < ptr[g + 1]; ++k) ncopy.push_back(copy[k]);
    nptr.push_back((int64_t)ncopy.size());
    if (with_bc) {
      nkind.push_back(kind[g]);
      for (int c = 0; c < 3; ++c) nnormal.push_back(normal[3 * g + c]);
    }
  }
  ptr.swap(nptr);
  copy.swap(ncopy);
  kind.swap(nkind);
  normal.swap(nnormal);
  for (auto& g : slot_group) g = newid[g];
}

int build_host_groups(const Mesh* m, int level, int space, std::vector<int64_t>& ptr, std::vector<int64_t>& copy,
                      std::vector<uint8_t>& kind, std::vector<double>& normal, std::vector<uint8_t>& own,
                      Halo& halo, std::vector<int64_t>& slot_group) {
  Prims P;
  build_prims(m, P);
  const int n1 = 1 << level;
  const bool p1 = space == HHG_P1;
  const int N = p1 ? n1 : 2 * n1;
  host_groups(m, P, N, !p1, npts3(N), ptr, copy, kind, normal, own, halo, slot_group);
  return HHG_OK;
}

static int build_groups(const Mesh* m, const Prims& P, int N, bool with_bc, Groups& G, std::vector<uint8_t>& own,
                        int64_t npts, int32_t** bcn = nullptr, int32_t** gmap = nullptr) {
  std::vector<int64_t> ptr, copy, slot_group;
  std::vector<uint8_t> kind;
  std::vector<double> normal;
  host_groups(m, P, N, with_bc, npts, ptr, copy, kind, normal, own, G.halo, slot_group);
  if (bcn) {  // per stored node BC map for the fused vector kernels
    std::vector<int32_t> map((size_t)npts * m->local.size(), -1);
    for (int64_t g = 0; g < (int64_t)kind.size(); ++g) {
      if (kind[g] == HHG_BC_NONE) continue;
      for (int64_t k = ptr[g]; k < ptr[g + 1]; ++k) map[copy[k]] = kind[g] == HHG_BC_DIRICHLET0 ? -2 : (int32_t)g;
    }
    HHG_TRY(upload(bcn, map));
  }
  if (gmap) {  // per stored node: its replicated-node / BC group, -1 if none (fused interface-sum consumers)
    std::vector<int32_t> map((size_t)npts * m->local.size(), -1);
    for (int64_t g = 0; g + 1 < (int64_t)ptr.size(); ++g)
      for (int64_t k = ptr[g]; k < ptr[g + 1]; ++k) map[copy[k]] = (int32_t)g;
    HHG_TRY(upload(gmap, map));
  }
  G.n = (int64_t)ptr.size() - 1;
  G.nbc = with_bc ? (int64_t)std::count_if(kind.begin(), kind.end(), [](uint8_t k) { return k != HHG_BC_NONE; }) : 0;
  G.ncopy = (int64_t)copy.size();
  HHG_TRY(upload(&G.ptr, ptr));
  HHG_TRY(upload(&G.copy, copy));
  if (with_bc) {
    HHG_TRY(upload(&G.kind, kind));
    HHG_TRY(upload(&G.normal, normal));
  }
  Halo& H = G.halo;
  if (H.nslots > 0) {
    // CSR group -> slots
    std::vector<int64_t> gp(G.n + 1, 0), gi(H.nslots);
    for (int64_t s = 0; s < H.nslots; ++s) ++gp[slot_group[s] + 1];
    for (int64_t g = 0; g < G.n; ++g) gp[g + 1] += gp[g];
    std::vector<int64_t> fill(gp.begin(), gp.end() - 1);
    for (int64_t s = 0; s < H.nslots; ++s) gi[fill[slot_group[s]]++] = s;
    HHG_TRY(upload(&H.slot_group, slot_group));
    HHG_TRY(upload(&H.gs_ptr, gp));
    HHG_TRY(upload(&H.gs_idx, gi));
    const int nc = with_bc ? 3 : 1;
    if (cudaMalloc(&H.sbuf, nc * H.nslots * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&H.rbuf, nc * H.nslots * sizeof(double)) != cudaSuccess)
      return fail(HHG_ENOMEM, "cudaMalloc halo buffers");
  }
  return HHG_OK;
}

int ensure_level(Mesh* m, int level) {
  if (level < 0 || level > m->level_max)
    return fail(HHG_ELEVEL, "level " + std::to_string(level) + " outside [0, level_max]");
  HHG_TRY(ensure_device_geo(m));
  Level& L = m->levels[level];
  if (L.built) return HHG_OK;
  free_level(L);
  L.level = level;
  L.n1 = 1 << level;
  L.n2 = 2 * L.n1;
  L.npts1 = npts3(L.n1);
  L.npts2 = npts3(L.n2);
  const int n = L.n1;
  const int64_t nm = macro_count(m);
  // element geometry per macro and type
  const double QA = (5.0 + 3.0 * std::sqrt(5.0)) / 20.0, QB = (5.0 - std::sqrt(5.0)) / 20.0;
  std::vector<double> geo((size_t)nm * kLevelGeo, 0.0);
  for (int64_t t = 0; t < nm; ++t) {
    const MacroGeo& g = m->hgeo[t];
    double* G = &geo[(size_t)t * kLevelGeo];
    for (int ty = 0; ty < 6; ++ty) {
      double E[9], Ei[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) E[3 * r + c] = kTypeVerts[ty][c + 1][r] - kTypeVerts[ty][0][r];
      inv3(E, Ei, nullptr);
      double* JFi = G + ty * kTypeGeo;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          double s = 0;
          for (int k = 0; k < 3; ++k) s += Ei[3 * r + k] * g.Jminv[3 * k + c];
          JFi[3 * r + c] = n * s;
        }
      for (int q = 0; q < 4; ++q) {
        double lam[4] = {QB, QB, QB, QB};
        lam[q] = QA;
        double lat[3];
        for (int r = 0; r < 3; ++r) {
          lat[r] = kTypeVerts[ty][0][r];
          for (int v = 1; v < 4; ++v) lat[r] += lam[v] * (kTypeVerts[ty][v][r] - kTypeVerts[ty][0][r]);
        }
        for (int r = 0; r < 3; ++r) {
          double s = 0;
          for (int c = 0; c < 3; ++c) s += g.Jm[3 * r + c] * lat[c];
          JFi[9 + 3 * q + r] = s / n;
        }
      }
    }
    G[6 * kTypeGeo] = g.absdet / ((double)n * n * n);
  }
  HHG_TRY(upload(&L.geo, geo));
  // bricks of 4x4x4 lattice cubes whose origin cube exists (i0+j0+k0 <= n-1)
  {
    std::vector<int32_t> b;
    for (int k = 0; k <= n - 1; k += 4)
      for (int j = 0; j + k <= n - 1; j += 4)
        for (int i = 0; i + j + k <= n - 1; i += 4) b.push_back(i | (j << 10) | (k << 20));
    // dense bricks first (same relative order), then the sparse ones (delta <= 4)
    std::stable_partition(b.begin(), b.end(), [n](int32_t pk) {
      return n - ((pk & 1023) + ((pk >> 10) & 1023) + (pk >> 20)) > 4;
    });
    L.n_dense = 0;
    for (int32_t pk : b) L.n_dense += n - ((pk & 1023) + ((pk >> 10) & 1023) + (pk >> 20)) > 4;
    L.n_bricks = (int64_t)b.size();
    HHG_TRY(upload(&L.bricks, b));
    // colour classes for the deterministic mode: bricks of one colour are >= 8 cubes apart in some
    // direction, so their 9x9x9 P2 footprints are disjoint
    std::vector<int32_t> bc;
    for (int c = 0; c < 8; ++c) {
      L.col_off[c] = (int64_t)bc.size();
      for (int32_t pk : b) {
        const int bi = (pk & 1023) >> 2, bj = ((pk >> 10) & 1023) >> 2, bk = (pk >> 20) >> 2;
        if (((bi & 1) | ((bj & 1) << 1) | ((bk & 1) << 2)) == c) bc.push_back(pk);
      }
    }
    L.col_off[8] = (int64_t)bc.size();
    HHG_TRY(upload(&L.bricks_col, bc));
  }
  // row-start tables (element kernel staging / write-out)
  for (int sp = 0; sp < 2; ++sp) {
    const int N = sp == 0 ? L.n1 : L.n2;
    std::vector<int32_t> rs((size_t)(N + 1) * (N + 1), 0);
    for (int k = 0; k <= N; ++k)
      for (int j = 0; j + k <= N; ++j) rs[(size_t)k * (N + 1) + j] = (int32_t)lidx(0, j, k, N);
    HHG_TRY(upload(sp == 0 ? &L.rs1 : &L.rs2, rs));
  }
  // rows
  for (int sp = 0; sp < 2; ++sp) {
    int N = sp == 0 ? L.n1 : L.n2;
    std::vector<int32_t> rows;
    for (int k = 0; k <= N; ++k)
      for (int j = 0; j + k <= N; ++j) rows.push_back(j | (k << 16));
    if (sp == 0) {
      L.nrows1 = (int64_t)rows.size();
      HHG_TRY(upload(&L.rows1, rows));
    } else {
      L.nrows2 = (int64_t)rows.size();
      HHG_TRY(upload(&L.rows2, rows));
    }
  }
  // groups / owner masks
  Prims P;
  build_prims(m, P);
  std::vector<uint8_t> own;
  HHG_TRY(build_groups(m, P, L.n2, true, L.g2, own, L.npts2, &L.bcn2, &L.gmap2));
  HHG_TRY(upload(&L.own2, own));
  HHG_TRY(build_groups(m, P, L.n1, false, L.g1, own, L.npts1));
  HHG_TRY(upload(&L.own1, own));
  if (cudaMalloc(&L.red, (kRedBlocks + 8) * sizeof(double)) != cudaSuccess)
    return fail(HHG_ENOMEM, "cudaMalloc reduction scratch");
  HHG_CUDA(cudaMemset(L.red, 0, (kRedBlocks + 8) * sizeof(double)));  // fused-dot counter starts at 0
  // kernel tables and attributes eagerly, then a device-wide sync: a later hot call on any stream
  // (non-blocking streams included, and under graph capture) sees a finished set-up
  HHG_TRY(elem_prepare_all());
  HHG_TRY(transfer_prepare());
  HHG_CUDA(cudaDeviceSynchronize());
  L.built = true;
  return HHG_OK;
}

// ------------------------------------------------------------------ canonical numbering
// Canonical order = lexicographic order of node keys [dim, ids, weights, res].
struct Canon {
  std::vector<int32_t> verts;                    // used vertex ids, ascending
  std::map<int32_t, int64_t> vrank;
  std::vector<std::array<int32_t, 2>> edges;
  std::map<std::array<int32_t, 2>, int64_t> erank;
  std::vector<std::array<int32_t, 3>> faces;
  std::map<std::array<int32_t, 3>, int64_t> frank;
  std::vector<std::array<int32_t, 4>> cells;
  std::map<std::array<int32_t, 4>, int64_t> crank;
};

static void build_canon(const Mesh* m, Canon& C) {
  std::set<int32_t> vs;
  std::set<std::array<int32_t, 2>> es;
  std::set<std::array<int32_t, 3>> fs;
  std::set<std::array<int32_t, 4>> cs;
  for (int64_t t = 0; t < m->n_tets; ++t) {
    const int32_t* v = &m->tets[4 * t];
    cs.insert({v[0], v[1], v[2], v[3]});
    for (int a = 0; a < 4; ++a) {
      vs.insert(v[a]);
      for (int b = a + 1; b < 4; ++b) {
        es.insert({v[a], v[b]});
        for (int c = b + 1; c < 4; ++c) fs.insert({v[a], v[b], v[c]});
      }
    }
  }
  C.verts.assign(vs.begin(), vs.end());
  for (size_t i = 0; i < C.verts.size(); ++i) C.vrank[C.verts[i]] = (int64_t)i;
  C.edges.assign(es.begin(), es.end());
  for (size_t i = 0; i < C.edges.size(); ++i) C.erank[C.edges[i]] = (int64_t)i;
  C.faces.assign(fs.begin(), fs.end());
  for (size_t i = 0; i < C.faces.size(); ++i) C.frank[C.faces[i]] = (int64_t)i;
  C.cells.assign(cs.begin(), cs.end());
  for (size_t i = 0; i < C.cells.size(); ++i) C.crank[C.cells[i]] = (int64_t)i;
}

static inline int64_t n_int(int d, int64_t N) {
  if (d == 0) return 1;
  if (d == 1) return N - 1;
  if (d == 2) return (N - 1) * (N - 2) / 2;
  return (N - 1) * (N - 2) * (N - 3) / 6;
}
static inline int64_t c3(int64_t x) { return x < 3 ? 0 : x * (x - 1) * (x - 2) / 6; }
static inline int64_t face_rank(int64_t w0, int64_t w1, int64_t N) {
  return (w0 - 1) * (N - 1) - (w0 - 1) * w0 / 2 + (w1 - 1);
}

static void canon_bases(const Canon& C, int64_t N, int64_t base[5]) {
  base[0] = 0;
  base[1] = base[0] + (int64_t)C.verts.size() * n_int(0, N);
  base[2] = base[1] + (int64_t)C.edges.size() * n_int(1, N);
  base[3] = base[2] + (int64_t)C.faces.size() * n_int(2, N);
  base[4] = base[3] + (int64_t)C.cells.size() * n_int(3, N);
}

static int64_t canon_index(const Canon& C, const int64_t base[5], int N, const int32_t* ids, const int* w, int d) {
  if (d == 0) return base[0] + C.vrank.at(ids[0]);
  if (d == 1) return base[1] + C.erank.at({ids[0], ids[1]}) * n_int(1, N) + (w[0] - 1);
  if (d == 2) return base[2] + C.frank.at({ids[0], ids[1], ids[2]}) * n_int(2, N) + face_rank(w[0], w[1], N);
  int64_t r = c3(N - 1) - c3(N - w[0]) + face_rank(w[1], w[2], N - w[0]);
  return base[3] + C.crank.at({ids[0], ids[1], ids[2], ids[3]}) * n_int(3, N) + r;
}

int canonical_count(const Mesh* m, int N, int64_t* n) {
  Canon C;
  build_canon(m, C);
  int64_t base[5];
  canon_bases(C, N, base);
  *n = base[4];
  return HHG_OK;
}

int canonical_keys(const Mesh* m, int N, int64_t* keys) {
  Canon C;
  build_canon(m, C);
  int64_t r = 0;
  auto put = [&](int d, const int32_t* ids, const int* w) {
    int64_t* k = keys + 10 * r++;
    k[0] = d;
    for (int c = 0; c < 4; ++c) k[1 + c] = c <= d ? ids[c] : -1;
    for (int c = 0; c < 4; ++c) k[5 + c] = c <= d ? w[c] : 0;
    k[9] = N;
  };
  for (int32_t v : C.verts) {
    int w[1] = {N};
    put(0, &v, w);
  }
  for (auto& e : C.edges)
    for (int a = 1; a <= N - 1; ++a) {
      int w[2] = {a, N - a};
      put(1, e.data(), w);
    }
  for (auto& f : C.faces)
    for (int a = 1; a <= N - 2; ++a)
      for (int b = 1; b <= N - 1 - a; ++b) {
        int w[3] = {a, b, N - a - b};
        put(2, f.data(), w);
      }
  for (auto& c : C.cells)
    for (int a = 1; a <= N - 3; ++a)
      for (int b = 1; b <= N - 2 - a; ++b)
        for (int cc = 1; cc <= N - 1 - a - b; ++cc) {
          int w[4] = {a, b, cc, N - a - b - cc};
          put(3, c.data(), w);
        }
  return HHG_OK;
}

int ensure_canon(Mesh* m, int level, int space) {
  HHG_TRY(ensure_level(m, level));
  Level& L = m->levels[level];
  bool p1 = space == HHG_P1;
  if ((p1 && L.canon1) || (!p1 && L.canon2)) return HHG_OK;
  int N = p1 ? L.n1 : L.n2;
  int64_t np = p1 ? L.npts1 : L.npts2;
  Canon C;
  build_canon(m, C);
  int64_t base[5];
  canon_bases(C, N, base);
  std::vector<int64_t> map((size_t)np * m->local.size());
  for (size_t t = 0; t < m->local.size(); ++t) {
    const int32_t* tv = &m->tets[4 * m->local[t]];
    for (int k = 0; k <= N; ++k)
      for (int j = 0; j + k <= N; ++j)
        for (int i = 0; i + j + k <= N; ++i) {
          int W[4] = {N - i - j - k, i, j, k};
          int32_t ids[4];
          int w[4];
          int d = -1;
          for (int a = 0; a < 4; ++a)
            if (W[a] > 0) {
              ++d;
              ids[d] = tv[a];
              w[d] = W[a];
            }
          map[t * np + lidx(i, j, k, N)] = canon_index(C, base, N, ids, w, d);
        }
  }
  if (p1) {
    L.ncanon1 = base[4];
    HHG_TRY(upload(&L.canon1, map));
  } else {
    L.ncanon2 = base[4];
    HHG_TRY(upload(&L.canon2, map));
  }
  return HHG_OK;
}

int mesh_set_geometry(Mesh* m) {
  m->hgeo.resize(m->local.size());
  for (size_t t = 0; t < m->local.size(); ++t) {
    MacroGeo& g = m->hgeo[t];
    const int32_t* v = &m->tets[4 * m->local[t]];
    for (int c = 0; c < 3; ++c) g.X0[c] = m->xyz[3 * v[0] + c];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) g.Jm[3 * r + c] = m->xyz[3 * v[c + 1] + r] - m->xyz[3 * v[0] + r];
    double det;
    inv3(g.Jm, g.Jminv, &det);
    if (!(std::fabs(det) > 0)) return fail(HHG_EINVAL, "degenerate macro tet");
    g.absdet = std::fabs(det);
    g.nhat[0] = g.nhat[1] = g.nhat[2] = 0.0;
    g.cK = 0.0;
    if (m->blend == HHG_BLEND_SHELL) {
      double dirs[4][3];
      int nd = 0;
      for (int a = 0; a < 4; ++a) {
        const double* x = &m->xyz[3 * v[a]];
        double r = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
        if (!(r > 0)) return fail(HHG_EDOMAIN, "macro vertex at the origin");
        double d[3] = {x[0] / r, x[1] / r, x[2] / r};
        bool dup = false;
        for (int e = 0; e < nd; ++e) {
          double dd = std::fabs(d[0] - dirs[e][0]) + std::fabs(d[1] - dirs[e][1]) + std::fabs(d[2] - dirs[e][2]);
          if (dd < 1e-10) dup = true;
        }
        if (!dup) {
          for (int c = 0; c < 3; ++c) dirs[nd][c] = d[c];
          ++nd;
        }
      }
      if (nd != 3) return fail(HHG_EDOMAIN, "shell blending needs 3 distinct vertex directions per macro");
      double a[3], b[3], n[3];
      for (int c = 0; c < 3; ++c) {
        a[c] = dirs[1][c] - dirs[0][c];
        b[c] = dirs[2][c] - dirs[0][c];
      }
      n[0] = a[1] * b[2] - a[2] * b[1];
      n[1] = a[2] * b[0] - a[0] * b[2];
      n[2] = a[0] * b[1] - a[1] * b[0];
      double nn = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
      double h = (n[0] * dirs[0][0] + n[1] * dirs[0][1] + n[2] * dirs[0][2]) / nn;
      double sgn = h < 0 ? -1.0 : 1.0;
      for (int c = 0; c < 3; ++c) g.nhat[c] = sgn * n[c] / nn;
      g.cK = 1.0 / (sgn * h);
    }
  }
  m->dgeo_dirty = true;  // uploaded lazily (host-only calls work without a GPU)
  return HHG_OK;
}

int ensure_device_geo(Mesh* m) {
  if (!m->dgeo_dirty) return HHG_OK;
  if (!m->dgeo && cudaMalloc(&m->dgeo, std::max<size_t>(1, m->hgeo.size()) * sizeof(MacroGeo)) != cudaSuccess)
    return fail(HHG_ENOMEM, "cudaMalloc macro geometry");
  HHG_CUDA(cudaMemcpy(m->dgeo, m->hgeo.data(), m->hgeo.size() * sizeof(MacroGeo), cudaMemcpyHostToDevice));
  m->dgeo_dirty = false;
  return HHG_OK;
}

}  // namespace hhg
