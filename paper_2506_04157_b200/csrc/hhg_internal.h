// Internal data structures of libhhgstokes (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>
#include <array>
#include <cuda_runtime.h>

#include "../../include/hhg_stokes.h"

namespace hhg {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
#define HHG_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess)                                                               \
      return ::hhg::fail(HHG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)
#define HHG_TRY(expr)            \
  do {                           \
    int _r = (expr);             \
    if (_r != HHG_OK) return _r; \
  } while (0)

void count_launch(int n = 1);

// ---------------------------------------------------------------- lattice helpers
__host__ __device__ inline int64_t npts3(int64_t N) { return (N + 1) * (N + 2) * (N + 3) / 6; }
__host__ __device__ inline int64_t tri(int64_t m) { return (m + 1) * (m + 2) / 2; }
// index of (i,j,k), i+j+k <= N, ordered by k, then j, then i
__host__ __device__ inline int64_t lidx(int i, int j, int k, int N) {
  return npts3(N) - npts3(N - k) + tri(N - k) - tri(N - k - j) + i;
}

// ---------------------------------------------------------------- per-macro data
// Device POD per macro (local numbering).  Jm columns = X1-X0, X2-X0, X3-X0 (row-major
// Jm[3*r+c]); vertex order = ascending global id.
struct MacroGeo {
  double X0[3];
  double Jm[9];
  double Jminv[9];
  double absdet;    // |det Jm|
  double nhat[3];   // blending normal
  double cK;        // blending factor (0 = identity blending)
};

// per-level, per-macro, per-tet-type element geometry (device)
// 6 types x (JFinv[9] + qoff[4][3]) + absdetF
constexpr int kTypeGeo = 9 + 12;
constexpr int kLevelGeo = 6 * kTypeGeo + 2;  // + absdetF + pad

// Cross-rank part of the interface sum (multi-GPU, macro partition over ranks): the groups of
// nodes shared with other ranks, one slot per (neighbor rank, shared node) in canonical node-key
// order (identical on both sides, so no index exchange is needed).
struct Halo {
  std::vector<int> nbr;            // neighbor ranks, ascending
  std::vector<int64_t> off;        // slot offset per neighbor (size nbr.size()+1)
  int64_t nslots = 0;
  std::vector<int64_t> keys;       // host [nslots][10] node keys (tests / diagnostics)
  int64_t* slot_group = nullptr;   // device [nslots]: local group of each slot
  int64_t* gs_ptr = nullptr;       // device [n_groups+1]: CSR group -> slots
  int64_t* gs_idx = nullptr;       // device [nslots]
  double* sbuf = nullptr;          // device [nslots][nc] local partial sums to send
  double* rbuf = nullptr;          // device [nslots][nc] partial sums received
};

struct Groups {           // replicated-node groups (interface and/or boundary nodes)
  int64_t n = 0;          // number of groups
  int64_t nbc = 0;        // groups [0, nbc) carry a BC (sorted first)
  int64_t* ptr = nullptr; // [n+1] into copy
  int64_t* copy = nullptr;// scalar flat indices (macro*npts + idx)
  uint8_t* kind = nullptr;// BC kind per group (P2 only)
  double* normal = nullptr;// [n][3] (P2 only)
  int64_t ncopy = 0;
  Halo halo;
};

struct Level {
  int level = 0;
  int n1 = 0, n2 = 0;               // P1 / P2 lattice resolution
  int64_t npts1 = 0, npts2 = 0;     // per macro
  double* geo = nullptr;            // [n_macro][kLevelGeo]
  int32_t* bricks = nullptr;        // 4x4x4-cube brick origins, packed i|j<<10|k<<20; dense bricks first
  int64_t n_bricks = 0;
  int64_t n_dense = 0;              // bricks [0, n_dense): delta = n1 - (i0+j0+k0) > 4 (per-cube path); the rest
                                    // (<= 64 tets, cut by the slanted face) go to k_elem_sparse
  int32_t* bricks_col = nullptr;    // the same bricks sorted by colour (bi&1 | (bj&1)<<1 | (bk&1)<<2)
  int64_t col_off[9] = {0};         // colour c: bricks_col[col_off[c] .. col_off[c+1])
  int32_t* rs1 = nullptr;           // row starts of the P1 / P2 lattices: index of (0, j, k) at [k (N+1) + j]
  int32_t* rs2 = nullptr;
  int32_t* rows1 = nullptr;         // packed (j | k<<16) for P1 rows
  int32_t* rows2 = nullptr;         // packed rows for P2
  int64_t nrows1 = 0, nrows2 = 0;
  Groups g1, g2;                    // P1 interface groups, P2 interface+BC groups
  int32_t* bcn2 = nullptr;          // per stored P2 node: -1 none, -2 Dirichlet, g >= 0 free-slip group
  int32_t* gmap2 = nullptr;         // per stored P2 node: its group in g2 (interface and/or BC), -1 if none
  uint8_t* own1 = nullptr;          // owner mask per stored P1 node
  uint8_t* own2 = nullptr;          // owner mask per stored P2 node
  int64_t* canon1 = nullptr;        // canonical node index per stored node (lazy)
  int64_t* canon2 = nullptr;
  int64_t ncanon1 = 0, ncanon2 = 0;
  double* red = nullptr;            // reduction scratch [kRedBlocks + 8]
  double* scratch_u = nullptr;      // P2VEC scratch (divT_apply accumulate), allocated on first use
  bool built = false;
};

constexpr int kRedBlocks = 296;     // 2 x 148 SMs
constexpr int kRedScratch = kRedBlocks + 8;

struct Mesh {
  // global macro mesh (host)
  int64_t n_vert = 0, n_tets = 0;
  std::vector<double> xyz;          // [n_vert][3]
  std::vector<int32_t> tets;        // [n_tets][4] ascending
  std::vector<int32_t> vtag;
  std::vector<int32_t> tet_rank;
  int level_max = 0;
  int rank = 0, nranks = 1;
  hhg_comm* comm = nullptr;
  std::vector<int64_t> local;       // global ids of local macros
  int blend = HHG_BLEND_IDENTITY;
  bool deterministic = false;       // element kernels per brick colour, no fp64 REDs (hhg_set_deterministic)
  int dependents = 0;               // live hhg_mg / hhg_kmg / hhg_stokes / hhg_temp_solver objects on this mesh
  int bc_kind[3] = {HHG_BC_NONE, HHG_BC_NONE, HHG_BC_NONE};  // untagged, inner, outer
  std::vector<MacroGeo> hgeo;       // host copy, local macros
  MacroGeo* dgeo = nullptr;         // device
  bool dgeo_dirty = true;
  std::vector<Level> levels;
  int device = 0;
  // Side streams of the element launcher, one per caller stream: the sparse-brick launch runs on it concurrently
  // with the dense-brick launch (fork / join by events; captured into CUDA graphs as parallel branches).
  struct Side {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
  };
  mutable std::map<cudaStream_t, Side> side;
  ~Mesh();
};
// Creates the side stream of caller stream `s` if missing; call before a stream capture that launches element
// kernels (the launcher itself never creates one under capture and falls back to serial launches there).
int elem_side_prepare(const Mesh* m, cudaStream_t s);

int ensure_level(Mesh* m, int level);
int ensure_device_geo(Mesh* m);
int mesh_set_geometry(Mesh* m);
int ensure_canon(Mesh* m, int level, int space);
int canonical_count(const Mesh* m, int N, int64_t* n);
int canonical_keys(const Mesh* m, int N, int64_t* keys);
constexpr uint64_t kKPowerSeed = 7;  // K_{1/sqrt(eta)} power-iteration start vector (hhg_kmg_create)
void free_level(Level& L);
int64_t macro_count(const Mesh* m);

// ---------------------------------------------------------------- kernel launchers (hhg_kernels.cu)
// Profiling hook (hhg_mg_profile): when set, the element launcher records this event on its stream after the
// dense-brick launch (k_elem_fp) and before the sparse-brick launch (k_elem_sparse), then clears it.
extern cudaEvent_t g_elem_mid_event;
int launch_elem(const Mesh* m, const Level& L, int mode, int form, const double* eta, double gamma,
                const double* u, const double* p, double* yu, double* yp, cudaStream_t s);
// w-BFBT operators (eq:schurWBFBT): K_{1/sqrt(eta_a)} (ELEM_KP1/KP1D, P1 -> P1) and the vector
// mass M_{sqrt(eta_a)} (ELEM_VMASS/VMASSD, P2VEC -> P2VEC), eta_a = a^2 eta on micro tets touching the
// sphere of radius r_outer (D_eta), a != 1 only on shell-blended meshes
int launch_elem_surf(const Mesh* m, const Level& L, int mode, const double* eta, double a, double r_outer,
                     const double* in, double* out, cudaStream_t s);
int surf_op(const Mesh* m, int level, int mode, const double* eta, double a, const double* in, double* out,
            cudaStream_t s);  // element kernel + interface sum (+ P_v M for ELEM_VMASS)
// temperature operator of eq:WeakTemp (hhg_temp.cu): mode 0 y += L T, 1 y += P T, 2 y += diag P
typedef hhg_temp_params TempCoef;
int launch_temp(const Mesh* m, const Level& L, int mode, TempCoef cf, const double* u, const double* T, double* y,
                cudaStream_t s);
int launch_mmoc(const Mesh* m, const Level& L, double rmin, double rmax, double tau, const double* T, const double* un,
                const double* uo, double* out, int* fail_flag, cudaStream_t s);
int launch_p1_prolong(const Mesh* m, const Level& Lc, const Level& Lf, const double* xc, double* xf, cudaStream_t s);
int launch_p1_restrict(const Mesh* m, const Level& Lc, const Level& Lf, const double* rf, double* rc, cudaStream_t s);
int launch_elem_qeta(const Mesh* m, const Level& L, int mode, const double* T2, double lnC, double jump, double r_jump,
                     const double* u, double* yu, cudaStream_t s);
// Smoother / residual update fused into the A kernel's write-out (single rank, non-deterministic mode, full form):
// at the footprint-interior points of dense bricks strictly inside the macro (complete after the brick, no interface
// copy, no BC) the kernel applies the consumer's update itself instead of storing A u; every other node keeps A u in
// yu for the *_fx consumer, which skips the fused nodes (elem_fused_mask).  kind: EPI_SUB r = f - Au; EPI_CHEB0
// r = f - Au, d = D^-1 r c1; EPI_CHEBK x += d, r -= Au, d = c1 d + c2 D^-1 r (d = the apply input); EPI_CHEBK_LAST
// x += d + c1 d + c2 D^-1 (r - Au).  Same arithmetic as launch_sub_fx / launch_cheb0_fx / launch_chebk_fx /
// launch_chebk_last_fx.
enum { EPI_NONE = 0, EPI_SUB = 1, EPI_CHEB0 = 2, EPI_CHEBK = 3, EPI_CHEBK_LAST = 4 };
struct ChebEpi {
  const double* f;
  double *x, *r, *d;
  const double* dinv;
  double c1, c2;
};
int launch_elem_epi(const Mesh* m, const Level& L, int kind, const ChebEpi& e, const double* eta, const double* u,
                    double* yu, cudaStream_t s);
int elem_fused_mask(const Mesh* m, const Level& L, uint8_t** mask);  // device [stored P2 nodes], caller frees
enum { ELEM_A = 1, ELEM_BT = 2, ELEM_DIV = 4, ELEM_DIAG = 8, ELEM_MASS = 16, ELEM_MASSD = 32, ELEM_LOAD = 64,
       ELEM_KP1 = 128, ELEM_KP1D = 256, ELEM_VMASS = 512, ELEM_VMASSD = 1024 };
constexpr int ELEM_SURF = ELEM_KP1 | ELEM_KP1D | ELEM_VMASS | ELEM_VMASSD;  // w-BFBT operators (eta_a scaling)
constexpr bool elem_p_out(int mode) { return (mode & (ELEM_DIV | ELEM_MASS | ELEM_MASSD | ELEM_KP1 | ELEM_KP1D)) != 0; }
constexpr bool elem_u_out(int mode) {
  return (mode & (ELEM_A | ELEM_BT | ELEM_DIAG | ELEM_LOAD | ELEM_VMASS | ELEM_VMASSD)) != 0;
}
constexpr bool elem_need_u(int mode) { return (mode & (ELEM_A | ELEM_DIV | ELEM_VMASS)) != 0; }
constexpr bool elem_need_p(int mode) { return (mode & (ELEM_BT | ELEM_MASS | ELEM_LOAD | ELEM_KP1)) != 0; }
int launch_fixup(const Mesh* m, const Level& L, int space, bool sum, bool bc, double* v, cudaStream_t s);
// split phases of a cross-rank interface sum: pack local partial sums of shared groups into
// halo.sbuf; exchange (NCCL); final fixup adding halo.rbuf (launch_fixup does all three when the
// mesh has a communicator)
int launch_halo_pack(const Mesh* m, const Level& L, int space, const double* v, double* sbuf, cudaStream_t s);
int launch_fixup_remote(const Mesh* m, const Level& L, int space, bool bc, const double* rbuf, double* v,
                        cudaStream_t s);
int comm_exchange(hhg_comm* c, const Halo& h, int nc, const double* sbuf, double* rbuf, cudaStream_t s);
int comm_allreduce_sum(hhg_comm* c, double* buf, int64_t n, cudaStream_t s);
bool comm_capturable(const hhg_comm* c);  // false for the host-staged transport (host synchronisation)
int build_host_groups(const Mesh* m, int level, int space, std::vector<int64_t>& ptr, std::vector<int64_t>& copy,
                      std::vector<uint8_t>& kind, std::vector<double>& normal, std::vector<uint8_t>& own,
                      Halo& halo, std::vector<int64_t>& slot_group);
// reduction scratch: kRedScratch doubles (partials + a zero-initialised counter at [kRedBlocks + 4]); every
// solver object owns one (red_alloc), mesh-level calls (hhg_dot) use the level's L.red
int launch_dot(const Mesh* m, const Level& L, int space, const double* x, const double* y, double* out,
               cudaStream_t s, double* red);
int red_alloc(double** red);
int launch_prolong(const Mesh* m, const Level& Lc, const Level& Lf, const double* xc, double* xf,
                   cudaStream_t s);
int launch_restrict(const Mesh* m, const Level& Lc, const Level& Lf, const double* rf, double* rc,
                    cudaStream_t s);
int launch_coords(const Mesh* m, const Level& L, int space, double* xyz, cudaStream_t s);
int launch_gather_canon(const Level& L, int space, int64_t nstored, const double* v, double* c, bool to,
                        cudaStream_t s);
// vector kernels for smoothers
int launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s);  // y = a x + b y
int launch_cheb0(int64_t n, const double* f, const double* t, const double* dinv, double inv_theta,
                 double* r, double* d, cudaStream_t s);  // r = f - t ; d = dinv r / theta
int launch_chebk(int64_t n, const double* t, const double* dinv, double c1, double c2, double* x, double* r,
                 double* d, cudaStream_t s);            // x += d; r -= t; d = c1 d + c2 dinv r
int launch_cheb_deg1(int64_t n, const double* f, const double* t, const double* dinv, double inv_theta, double* x,
                     cudaStream_t s);                     // x += dinv (f - t) / theta  (t null: x = 0 first)
int launch_chebk_last(int64_t n, const double* t, const double* dinv, double c1, double c2, const double* r,
                      const double* d, double* x, cudaStream_t s);  // x += d + c1 d + c2 dinv (r - t)
int launch_pcg_update(int64_t n, const double* scal, double* x, double* r, const double* p, const double* q,
                      const double* dinv, double* z, cudaStream_t s);
// node-major vector kernels with the BC projection (P_v M) of the updated direction fused in
// (replaces a BC-only fixup pass); `L` supplies the per-node BC map and free-slip normals
int launch_cheb0_bc(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                    double inv_theta, double* r, double* d, cudaStream_t s);
int launch_chebk_bc(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2, double* x,
                    double* r, double* d, cudaStream_t s);
int launch_chebk_last_bc(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2,
                         const double* r, const double* d, double* x, cudaStream_t s);
int launch_cheb_deg1_bc(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                        double inv_theta, double* x, cudaStream_t s);
// PCG with ping-pong r.z scalars: scal[0]/scal[2] alternate by iteration parity, scal[1] = p.q
int launch_pcg_update_bc(const Mesh* m, const Level& L, int it, const double* scal, double* x, double* r,
                         const double* p, const double* q, const double* dinv, double* z, cudaStream_t s);
int launch_pcg_dir_zero(int64_t n, int it, const double* scal, const double* z, double* p, double* q_zero,
                        cudaStream_t s);
// Consumers of an UNSUMMED element-kernel output t (single rank; skip != nullptr: nodes with skip[i] != 0 were
// updated by the element kernel's fused epilogue, launch_elem_epi, and are left alone): each stored node reads its value as the sum
// of its group's copies with the group's BC applied (= what k_fixup would have stored), so the separate
// interface-sum pass disappears.  Same semantics as the *_bc kernels applied after launch_fixup(sum, BC).
int launch_cheb0_fx(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                    double inv_theta, double* r, double* d, cudaStream_t s, const uint8_t* skip = nullptr);
int launch_chebk_fx(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2, double* x,
                    double* r, double* d, cudaStream_t s, const uint8_t* skip = nullptr);
int launch_chebk_last_fx(const Mesh* m, const Level& L, const double* t, const double* dinv, double c1, double c2,
                         const double* r, const double* d, double* x, cudaStream_t s, const uint8_t* skip = nullptr);
int launch_cheb_deg1_fx(const Mesh* m, const Level& L, const double* f, const double* t, const double* dinv,
                        double inv_theta, double* x, cudaStream_t s);
int launch_sub_fx(const Mesh* m, const Level& L, const double* f, const double* t, double* r, cudaStream_t s, const uint8_t* skip = nullptr);  // r = f - t
// PCG update fused with the new r.z (single rank): writes r.z into the ping-pong slot of iteration `it`
int launch_pcg_update_bc_dot(const Mesh* m, const Level& L, int it, double* scal, double* x, double* r, const double* p,
                             const double* q, const double* dinv, double* z, double* red, cudaStream_t s);
// eager one-time set-up of kernel tables / attributes (never from a hot call)
int elem_prepare_all();
int transfer_prepare();
int launch_dot_fused(const Mesh* m, const Level& L, int space, const double* x, const double* y, double* out,
                     cudaStream_t s, double* red);
int launch_scalar_ops(int op, double* scal, cudaStream_t s);
// cluster-resident coarse Jacobi-PCG (hhg_coarse.cu): one kernel per coarse solve on a single-rank mesh
struct CoarseSolver;
int coarse_create(const Mesh* m, int level, int form, const double* eta, const double* T2, double lnC, double jump,
                  double rjump, const double* dinv, CoarseSolver** out);
int coarse_run(CoarseSolver* c, const double* f, double* x, double* r, double* z, double* p, double* q, int iters,
               double tol, cudaStream_t s);
int coarse_iterations(const CoarseSolver* c, int* out);  // iterations of the last run (synchronises)
void coarse_destroy(CoarseSolver* c);
int launch_fill(int64_t n, double v, double* y, cudaStream_t s);
int launch_recip(int64_t n, double* y, cudaStream_t s);                          // y = 1 / y
int launch_pcg_scale(int64_t n, const double* d, const double* x, double* y, cudaStream_t s);  // y = d x

}  // namespace hhg

struct hhg_mesh : public hhg::Mesh {};

#include <nccl.h>
struct hhg_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1, rank = 0, device = 0;
  // host-staged transport (hhg_comm_create_host)
  bool host = false;
  hhg_exchange_fn exchange_fn = nullptr;
  hhg_allreduce_fn allreduce_fn = nullptr;
  void* user = nullptr;
  double* hbuf = nullptr;   // pinned [2][hcap] send / receive staging
  size_t hcap = 0;
};
