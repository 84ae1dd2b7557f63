/*
 * hhg_stokes.h -- C-ABI of libhhgstokes.so: the B200 (sm_100a) hot path of
 * arxiv 2506.04157 (Burkhart, Kohl, Wohlmuth, Zawallich), "A robust matrix-free
 * approach for large-scale non-isothermal high-contrast viscosity Stokes flow on
 * blended domains".  Citations "P:<n>" are lines of /root/reference/PAPER.md.
 *
 * The hot path: matrix-free application of the blended P2-P1 Taylor-Hood,
 * variable-viscosity, compressible Stokes operator
 *        [ A(eta)   B^T ] [u]       A_ij = int 2 eta (eps(phi_j):eps(phi_i) - 1/3 div phi_j div phi_i)
 *        [ B + C     0  ] [p]       B_ij = -int div(phi_j) psi_i,  C_ij = -int grad ln rho . phi_j psi_i
 * (eq:SaddlePointStructure), used inside the Chebyshev-smoothed GMG
 * V-cycle of the A block (fig:ASolverStructure).
 *
 * CONVENTIONS
 *  - Every call returns int: 0 = HHG_OK, a negative HHG_E* code otherwise;
 *    hhg_last_error() returns a thread-local message for the last failure.
 *  - Handles (hhg_mesh, hhg_mg, hhg_comm) are opaque and library-owned.
 *  - VECTORS are caller-owned DEVICE pointers to contiguous fp64 arrays in the
 *    LIBRARY LAYOUT (below); their length comes from hhg_vec_len().  Per-level
 *    tables are built on the FIRST use of a (mesh, level) after hhg_mesh_create /
 *    blend_map / hhg_set_bc, or eagerly by hhg_mesh_prepare(); that build ends with a
 *    device synchronisation (so a following call on any stream, blocking or not, sees
 *    it) and must not happen under stream capture: call hhg_mesh_prepare() (or create
 *    the solver object, which builds its levels) before capturing.  Solver objects
 *    (hhg_mg, hhg_kmg, hhg_stokes, hhg_temp_solver) allocate all their workspace,
 *    including their own reduction scratch, in *_create; hot calls never allocate.
 *  - One solver object is used by one stream at a time; different objects on the same
 *    mesh may run concurrently on different streams (they share no scratch).
 *    hhg_dot uses the level's scratch: concurrent hhg_dot calls on one (mesh, level)
 *    must be ordered by the caller.
 *  - Operator applications launch their sparse-brick kernel on a library-owned side
 *    stream forked from and joined back to the caller's stream by events (one side
 *    stream per caller stream, created on the first application outside stream capture;
 *    an application captured on a stream without one launches serially).  The result
 *    is ordered on the caller's stream as if everything ran there.  Calls on one mesh
 *    from several HOST threads must be serialised by the caller.
 *  - Hot calls are asynchronous on the caller's cudaStream_t (pass NULL for the
 *    legacy default stream).  Calls that return host scalars synchronise and say so.
 *  - Outputs must not alias inputs unless stated.
 *
 * LIBRARY LAYOUT (hierarchical hybrid grid): every macro tet keeps its own
 * structured tetrahedral lattice (uniform Bey refinement to level L: 8^L micro
 * tets).  P1 lattice resolution n = 2^L, P2 lattice resolution 2n.  Points of a
 * lattice of resolution N are ordered by (k, j, i), i+j+k <= N, with barycentric
 * weights (N-i-j-k, i, j, k) w.r.t. the macro's vertices in ASCENDING global id
 * order.  Nodes on macro faces/edges/vertices are REPLICATED in every macro
 * containing them; a vector is "consistent" when all copies agree.
 *   HHG_P1    : double[n_macro][npts(n)]
 *   HHG_P2    : double[n_macro][npts(2n)]
 *   HHG_P2VEC : double[3][n_macro][npts(2n)]   (component-major, x,y,z)
 * Canonical (unique-node) order, used by hhg_to_canonical / hhg_from_canonical /
 * hhg_canonical_keys: nodes sorted by key [dim, ascending primitive vertex ids,
 * their positive integer weights, res] (dim 0 vertices, 1 edges, 2 faces, 3 cells);
 * P2VEC canonical vectors are node-major with (x,y,z) interleaved.
 *
 * Boundary conditions: HHG_BC_DIRICHLET0 zeroes the node's
 * velocity (block-row modification, surface no-slip); HHG_BC_FREESLIP applies
 * P_v: u <- u - (u.n) n with n = x/|x| (CMB).  Operators return (M P_v) A u etc.;
 * they do NOT project their input: pass constraint-consistent u (hhg_apply_bc).
 */
#ifndef HHG_STOKES_H
#define HHG_STOKES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hhg_stream_t;   /* == cudaStream_t */
typedef struct hhg_mesh hhg_mesh;
typedef struct hhg_mg hhg_mg;
typedef struct hhg_comm hhg_comm;

enum {
  HHG_OK = 0,
  HHG_EINVAL = -1,      /* bad argument (NULL, level out of range, r_min >= r_max, ...) */
  HHG_ELEVEL = -2,      /* space/level mismatch, non-adjacent levels */
  HHG_ENOTREADY = -3,   /* Chebyshev without a spectrum estimate */
  HHG_EZEROOP = -4,     /* power iteration on a zero operator */
  HHG_EDOMAIN = -5,     /* geometry outside the blending's domain */
  HHG_ECUDA = -6,
  HHG_ENCCL = -7,
  HHG_ENOMEM = -8
};

enum { HHG_P1 = 1, HHG_P2 = 2, HHG_P2VEC = 3 };
enum { HHG_BLEND_IDENTITY = 0, HHG_BLEND_SHELL = 1 };
enum { HHG_BND_ALL = 0, HHG_BND_INNER = 1, HHG_BND_OUTER = 2 };      /* vertex tags 1 / 2 */
enum { HHG_BC_NONE = 0, HHG_BC_DIRICHLET0 = 1, HHG_BC_FREESLIP = 2 };
enum { HHG_VISC_FULL = 0, HHG_VISC_EPS = 1 };

/* Thread-local message describing the last error (never NULL). */
const char* hhg_last_error(void);
/* Library version string, build flags, the sm arch compiled for. */
const char* hhg_version(void);

/* ------------------------------------------------------------------ comm
 * Multi-GPU (one process per GPU): an NCCL communicator over NVLink/NVSwitch.
 * The id is created on rank 0 and broadcast by the caller (e.g. torch.distributed).
 * comm == NULL everywhere means single GPU. */
int hhg_comm_unique_id(uint8_t id[128]);
int hhg_comm_create(const uint8_t id[128], int nranks, int rank, int device, hhg_comm** out);
int hhg_comm_destroy(hhg_comm* comm);

/* Host-staged transport (P:689-709 multi-process decomposition, without NCCL): the library drains the
 * stream, copies its send buffer to pinned host memory and calls
 *   exchange(user, n_nbr, nbr[n_nbr], off[n_nbr+1], nc, send, recv): for every neighbour rank nbr[i],
 *     send the doubles send[off[i]*nc .. off[i+1]*nc) to it and receive its block of the same length
 *     into recv[off[i]*nc ..) (both sides list the shared nodes in the same canonical order);
 *     called on EVERY rank for every interface sum (n_nbr may be 0), so it may be collective;
 *   allreduce(user, buf, n): in-place elementwise sum of n doubles over all ranks;
 * both return 0 on success.  Then the received data is copied back.  Any number of ranks may share
 * one GPU (no kernel waits on another rank).  Hot calls synchronise their stream, so objects using
 * such a communicator never capture CUDA graphs.  Errors: HHG_ENCCL if a callback fails. */
typedef int (*hhg_exchange_fn)(void* user, int n_nbr, const int* nbr, const int64_t* off, int nc, const double* send,
                               double* recv);
typedef int (*hhg_allreduce_fn)(void* user, double* buf, int64_t n);
int hhg_comm_create_host(int nranks, int rank, hhg_exchange_fn exchange, hhg_allreduce_fn allreduce, void* user,
                         hhg_comm** out);

/* ------------------------------------------------------------------ mesh
 * hhg_mesh_create: macro tets (n_tets x 4 vertex ids, any order; the
 * library sorts each row ascending), vertex coordinates (n_vert x 3, host), vertex
 * tags (0 interior, 1 inner/CMB, 2 outer/surface; host; NULL = all 0), refinement
 * up to level_max (0..8).  tet_rank (host, n_tets, NULL = all local) assigns each
 * macro to a rank of comm; this process keeps the macros with tet_rank == its rank
 * (tet_rank with nonzero entries needs comm, else HHG_EINVAL: see hhg_mesh_create_part).
 * Errors: HHG_EINVAL (NULL, n < 1, level_max out of range, degenerate tet). */
int hhg_mesh_create(const double* macro_xyz, int64_t n_vert, const int32_t* macro_tets, int64_t n_tets,
                    const int32_t* vertex_tag, int level_max, const int32_t* tet_rank, hhg_comm* comm,
                    hhg_mesh** out);
int hhg_mesh_destroy(hhg_mesh* mesh);
/* The thick spherical shell macro mesh shell(ntan, nrad) (R4): each icosahedron
 * face split into (ntan-1)^2 flat triangles normalised to the sphere, nrad spheres between r_min
 * and r_max, every layer prism split into 3 tets (sorted-id staircase rule); 60 (ntan-1)^2 (nrad-1)
 * macro tets (shell(3,2) = the paper's 240 macros).  Vertex tags 1 (r_min, CMB) / 2 (r_max,
 * surface) / 0.  hhg_icoshell_macro returns the arrays (host; pass NULL arrays to query sizes);
 * hhg_mesh_create_icoshell builds the mesh directly.  HHG_EINVAL for ntan < 2, nrad < 2, bad radii. */
int hhg_icoshell_macro(int ntan, int nrad, double r_min, double r_max, double* verts, int32_t* tets, int32_t* vtag,
                       int64_t* n_vert, int64_t* n_tets);
int hhg_mesh_create_icoshell(int ntan, int nrad, double r_min, double r_max, int level_max, const int32_t* tet_rank,
                             hhg_comm* comm, hhg_mesh** out);
/* Number of macro tets stored by this process. */
int hhg_mesh_local_macros(const hhg_mesh* mesh, int64_t* n);

/* ------------------------------------------------------------------ partitioned meshes (multi-GPU)
 * The path shards by macro tets (the paper's domain decomposition): each rank keeps
 * the lattices of its macros; nodes on macro faces/edges/vertices shared with other ranks are
 * summed by one exchange per operator (NCCL point-to-point over NVLink), dots by one allreduce.
 * hhg_partition_rcb: recursive coordinate bisection of macro centroids into nparts (radial != 0:
 *   centroids projected to the unit sphere, keeping radial macro columns on one rank) -> tet_rank
 *   (host, n_tets).  Deterministic; equal part sizes up to rounding.
 * hhg_mesh_create_part: rank `rank`'s view of a partition WITHOUT a communicator: interface sums
 *   cover local copies only; the cross-rank part is done by the caller with hhg_halo_pack ->
 *   (transport of the send buffers) -> hhg_interface_sum_remote.  hhg_mesh_create with a comm does
 *   the same internally (pack, ncclSend/ncclRecv per neighbor, remote-sum kernel).
 * Shared nodes with neighbor q are listed in canonical key order, so the receive buffer segment
 * from q matches our send segment to q slot by slot.  Buffers: device, [slots][nc] fp64, nc = 3
 *   (P2VEC) or 1 (P1), neighbor segments in ascending rank order (hhg_halo_info gives the ranks and
 *   per-neighbor counts; host-only, no GPU needed).  hhg_halo_keys: HOST int64 [slots][10] node keys.
 * Owner of a replicated node = its copy in the lowest global macro id: hhg_owned_count summed over
 *   ranks equals hhg_canonical_len (host-only).  Errors: HHG_EINVAL (bad rank, NULL, bad space). */
int hhg_partition_rcb(const double* macro_xyz, int64_t n_vert, const int32_t* macro_tets, int64_t n_tets,
                      int nparts, int radial, int32_t* tet_rank);
int hhg_mesh_create_part(const double* macro_xyz, int64_t n_vert, const int32_t* macro_tets, int64_t n_tets,
                         const int32_t* vertex_tag, int level_max, const int32_t* tet_rank, int nranks, int rank,
                         hhg_mesh** out);
int hhg_mesh_rank(const hhg_mesh* mesh, int* rank, int* nranks);
int hhg_halo_info(const hhg_mesh* mesh, int level, int space, int* n_nbr, int32_t* nbr_ranks, int64_t* counts);
int hhg_halo_keys(const hhg_mesh* mesh, int level, int space, int64_t* keys_host);
int hhg_owned_count(const hhg_mesh* mesh, int level, int space, int64_t* n_owned);
int hhg_halo_pack(const hhg_mesh* mesh, int level, int space, const double* v, double* sendbuf,
                  hhg_stream_t stream);
int hhg_interface_sum_remote(const hhg_mesh* mesh, int level, int space, const double* recvbuf, double* v,
                             hhg_stream_t stream);

/* blend_map: HHG_BLEND_SHELL = origin-centred thick spherical
 * shell: per macro, B(x) = c_K x (n_K . x)/|x| with n_K the unit normal of the plane
 * through the macro's 3 distinct vertex directions and c_K = 1/(n_K . p); it maps
 * every flat layer triangle onto its sphere and is C^0 across macros.
 * Errors: HHG_EDOMAIN if a macro does not have exactly 3 distinct directions. */
int blend_map(hhg_mesh* mesh, int kind);

/* hhg_set_bc: boundary faces = macro faces of exactly one macro tet; a face's tag
 * is the common tag of its 3 vertices.  tag = HHG_BND_ALL sets every boundary face.
 * blend_map / hhg_set_bc / hhg_set_deterministic invalidate the per-level tables and
 * return HHG_EINVAL while solver objects built on the mesh are alive (their diagonals,
 * spectrum estimates and captured CUDA graphs depend on the old tables). */
int hhg_set_bc(hhg_mesh* mesh, int tag, int kind);

/* hhg_set_deterministic (on != 0): every element kernel (A, diag, B, B^T, C, mass, load,
 * w-BFBT operators) runs as 8 launches, one per brick colour (bricks of one colour share
 * no lattice point), accumulating brick borders with plain load-add-store instead of fp64
 * atomics, so applies, dots, V-cycles and solves are bitwise reproducible run to run.
 * Off by default (the atomic single-launch path is faster).  The temperature operator
 * (hhg_temp_apply) keeps its atomics.  Errors: HHG_EINVAL with live solver objects. */
int hhg_set_deterministic(hhg_mesh* mesh, int on);

/* hhg_mesh_prepare: build the per-level tables of every level 0..level_max now (host work
 * + uploads + one device synchronisation), so that no later call builds them lazily. */
int hhg_mesh_prepare(hhg_mesh* mesh);

/* Length (doubles) of a vector of `space` at `level` in the library layout. */
int hhg_vec_len(const hhg_mesh* mesh, int level, int space, int64_t* n);
/* Number of unique nodes (HHG_P1/HHG_P2) or unique dofs (HHG_P2VEC) in canonical order. */
int hhg_canonical_len(const hhg_mesh* mesh, int level, int space, int64_t* n_unique);
/* Canonical node keys, HOST int64 array [n_unique_nodes][10] =
 * [dim, id0..id3 (-1 padded), w0..w3 (0 padded), res].  space: HHG_P1 or HHG_P2. */
int hhg_canonical_keys(const hhg_mesh* mesh, int level, int space, int64_t* keys_host);
/* Gather a CONSISTENT library-layout vector into canonical order (device -> device). */
int hhg_to_canonical(const hhg_mesh* mesh, int level, int space, const double* v_dev, double* c_dev,
                     hhg_stream_t stream);
/* Scatter a canonical vector to all copies in the library layout (device -> device). */
int hhg_from_canonical(const hhg_mesh* mesh, int level, int space, const double* c_dev, double* v_dev,
                       hhg_stream_t stream);
/* Blended physical coordinates of every stored node of a scalar space (HHG_P1 or
 * HHG_P2): xyz_dev = double[n_stored][3]. */
int hhg_node_coords(const hhg_mesh* mesh, int level, int space, double* xyz_dev, hhg_stream_t stream);

/* ------------------------------------------------------------------ constraints / consistency
 * hhg_apply_bc: u <- P_v M u in place (P2VEC).  hhg_interface_sum: turn a vector of
 * per-macro partial sums into the consistent assembled vector (sum of all copies,
 * written to every copy); for HHG_P2VEC the BCs are applied afterwards. */
int hhg_apply_bc(const hhg_mesh* mesh, int level, double* u, hhg_stream_t stream);
int hhg_interface_sum(const hhg_mesh* mesh, int level, int space, double* v, hhg_stream_t stream);

/* ------------------------------------------------------------------ operators
 * Results are interface-summed (consistent) and, for velocity outputs, BC-masked
 * (M P_v ...).  eta_p1: P1 viscosity at level's vertices, NULL = 1.
 * Quadrature: 4-point degree-2 rule on every micro tet (R6); the blending
 * Jacobian is evaluated at each quadrature point on the fly.
 *
 * epsilon_apply: y = (M P_v) A(eta) u.  form HHG_VISC_FULL = the paper's A
 *   (P:277-278 with eta on both terms, R1); HHG_VISC_EPS = int 2 eta eps:eps.
 * div_apply:  q = (B + C) u, grad ln rho = -gamma x/|x|; gamma 0 -> B.
 * divT_apply: y_u = (M P_v) B^T p   (accumulate != 0: y_u += ..., y_u consistent).
 * stokes_apply: y_u = (M P_v)(A u + B^T p), y_p = (B + C) u.
 * hhg_diag: diag(A(eta)) WITHOUT P_v, consistent, all dofs. */
int epsilon_apply(const hhg_mesh* mesh, int level, int form, const double* eta_p1, const double* u,
                  double* y, hhg_stream_t stream);
int div_apply(const hhg_mesh* mesh, int level, double gamma, const double* u, double* q,
              hhg_stream_t stream);
int divT_apply(const hhg_mesh* mesh, int level, const double* p, double* y_u, int accumulate,
               hhg_stream_t stream);
int stokes_apply(const hhg_mesh* mesh, int level, const double* eta_p1, double gamma, const double* u,
                 const double* p, double* y_u, double* y_p, hhg_stream_t stream);
int hhg_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double* diag, hhg_stream_t stream);
/* hhg_mass_apply: y = M_{1/eta} p, the P1 pressure mass matrix weighted by 1/eta (the Schur
 * complement approximation S_M of eq:schurMass): M_vw = int (1/eta) psi_v psi_w with
 * eta P1-interpolated at the quadrature points, blended geometry.  hhg_mass_diag: its diagonal.
 * Both consistent (interface-summed) P1 vectors; eta_p1 NULL = 1 (plain pressure mass). */
int hhg_mass_apply(const hhg_mesh* mesh, int level, const double* eta_p1, const double* p, double* y,
                   hhg_stream_t stream);
int hhg_mass_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double* diag, hhg_stream_t stream);
/* hhg_buoyancy_load: f = (M P_v) b, b_i = int (T - 1/2) (x/|x|) . phi_i  -- the buoyancy right-hand
 * side of config 4 (P:282 with rho' = -alpha (T - 1/2), alpha = 1, gravity g = -x/|x|; DESIGN.md
 * R21).  T_p1: consistent P1 temperature at the level's vertices; f: P2VEC, consistent. */
int hhg_buoyancy_load(const hhg_mesh* mesh, int level, const double* T_p1, double* f, hhg_stream_t stream);
/* epsilon_apply_partial: the element half of epsilon_apply only -- per-copy partial sums of
 * A(eta) u, NO interface sum and NO BC (first phase of a split-phase exchange). */
int epsilon_apply_partial(const hhg_mesh* mesh, int level, int form, const double* eta_p1, const double* u,
                          double* y, hhg_stream_t stream);

/* Inner product over UNIQUE dofs of two consistent vectors (each replicated node
 * counted once), allreduced over ranks; result written to out_dev (1 double). */
int hhg_dot(const hhg_mesh* mesh, int level, int space, const double* x, const double* y, double* out_dev,
            hhg_stream_t stream);

/* ------------------------------------------------------------------ multigrid
 * p2_prolong: x_fine += (M P_v) P x_coarse, P = nodal P2 interpolation (exact embedding).
 * p2_restrict: r_coarse = (M P_v) P^T r_fine  (r_fine consistent). */
int p2_restrict(const hhg_mesh* mesh, int fine_level, const double* r_fine, double* r_coarse,
                hhg_stream_t stream);
int p2_prolong(const hhg_mesh* mesh, int coarse_level, const double* x_coarse, double* x_fine,
               hhg_stream_t stream);

/* chebyshev_smooth: one degree-`degree` Chebyshev sweep on D^-1 A over
 * [lmin, lmax]: theta=(lmax+lmin)/2, delta=(lmax-lmin)/2, sigma=theta/delta, rho=1/sigma;
 * r = rhs - A x; d = PM dinv r/theta; for k=1..deg: x += d; if k<deg: r -= A d;
 * rho' = 1/(2 sigma - rho); d = rho' rho d + (2 rho'/delta) PM dinv r; rho = rho'.
 * work: >= 3 P2VEC vectors.  dinv = 1/diag(A).  HHG_ENOTREADY if lmax <= 0. */
int chebyshev_smooth(const hhg_mesh* mesh, int level, const double* eta_p1, const double* dinv, int degree,
                     double lmin, double lmax, const double* rhs, double* x, double* work, hhg_stream_t stream);

/* Power iteration for lambda_max(D^-1 A): v = PM v0; iters x { w = PM dinv A v;
 * lambda = |w|; v = w/lambda }.  v0 (device, consistent) is overwritten.
 * Synchronises; lambda returned on the host.  HHG_EZEROOP on a zero operator. */
int hhg_power_iteration(const hhg_mesh* mesh, int level, const double* eta_p1, const double* dinv, int iters,
                        double* v0, double* lambda_host, hhg_stream_t stream);

typedef struct {
  int l_min, l_max;          /* coarsest / finest level */
  int pre, post, degree;     /* Chebyshev steps and degree (BASELINE config 3: 3, 3, 3) */
  int power_iters;           /* 20 */
  int coarse_iters;          /* Jacobi-PCG iterations on l_min (50) */
  double cheb_hi_factor;     /* 1.1  (b = 1.1 lambda_hat) */
  double cheb_lo_ratio;      /* 0.1  (a = b/10)           */
  int visc_form;             /* HHG_VISC_FULL */
  int use_graph;             /* capture the V-cycle in a CUDA graph */
  int l_eta;                 /* levels <= l_eta evaluate eta at the quadrature points (NEXT-2; -1: none) */
  double qeta_lnC, qeta_jump, qeta_rjump;  /* eta_q = exp(lnC (1/2 - T_q)) (jump if r_q < rjump else 1) */
  int coarse_redundant;      /* multi-rank meshes: gather the l_min problem of ALL macros (one allreduce of the
                                zero-padded global vector) and solve it redundantly on every rank -- the analogue
                                of the paper's coarse-grid agglomeration; 0: distributed PCG
                                (an interface exchange + 2 allreduces per coarse iteration) */
  double coarse_tol;         /* 0: exactly coarse_iters Jacobi-PCG iterations (BASELINE config 3).  > 0: stop as soon
                                as sqrt(r.z) <= coarse_tol sqrt(r0.z0), at most coarse_iters iterations -- the paper's
                                coarse solve "up to a relative tolerance tol_coarse" (Table 1: 1e-2; DESIGN.md
                                R29).  Needs the cluster-resident coarse solver (single-rank mesh or
                                coarse_redundant): HHG_EINVAL otherwise. */
} hhg_mg_params;

/* hhg_mg_create: builds per-level workspaces, diag(A) and D^-1, and lambda_hat per
 * level by power iteration from the consistent start vectors power_v0[l] (device,
 * P2VEC, may be NULL entries for l_min).  eta_per_level[l] (device P1 vectors) must
 * stay alive while the hierarchy is used.  Synchronises. */
int hhg_mg_create(hhg_mesh* mesh, const hhg_mg_params* params, const double* const* eta_per_level,
                  double* const* power_v0, hhg_mg** out);
/* hhg_mg_create_qeta: as hhg_mg_create, and on levels l <= params->l_eta the A operator (apply,
 * diag, lambda) evaluates the viscosity at the quadrature points from the P2 temperature
 * T2_per_level[l] (consistent P2 vectors, kept alive by the caller): the two-tier viscosity of
 * P:451-453 (the paper's order-6 exp surrogate is a CPU-vectorisation device; the fp64 exp is used). */
int hhg_mg_create_qeta(hhg_mesh* mesh, const hhg_mg_params* params, const double* const* eta_per_level,
                       const double* const* T2_per_level, double* const* power_v0, hhg_mg** out);
/* epsilon_apply_qeta / hhg_diag_qeta: A(eta) u and diag(A) with eta evaluated at the quadrature
 * points: eta_q = exp(lnC (1/2 - T_q)) * (jump if |x_q| < r_jump else 1), T_q the P2 interpolant of
 * T_p2 (NEXT-2 tier).  Results consistent; apply BC-masked (M P_v), diag without P_v. */
int epsilon_apply_qeta(const hhg_mesh* mesh, int level, const double* T_p2, double lnC, double jump, double r_jump,
                       const double* u, double* y, hhg_stream_t stream);
int hhg_diag_qeta(const hhg_mesh* mesh, int level, const double* T_p2, double lnC, double jump, double r_jump,
                  double* diag, hhg_stream_t stream);
/* Iterations taken by the most recent coarse solve of the hierarchy (coarse_tol > 0: data dependent).
 * Synchronises the device.  HHG_EINVAL if the coarse level does not run the cluster-resident solver. */
int hhg_mg_coarse_iterations(const hhg_mg* mg, int* iters_out);
int hhg_mg_lambda(const hhg_mg* mg, int level, double* lambda_host);
/* One V-cycle (fig:ASolverStructure) from x = 0: x = V(rhs). */
int vcycle(hhg_mg* mg, const double* rhs, double* x, hhg_stream_t stream);
/* hhg_ablock_cg (the A-block solver of the Uzawa preconditioners): CG preconditioned by one
 * V-cycle (this hierarchy) per iteration, from x = 0, until |r|_2 <= tol |rhs|_2 (unique dofs) or
 * max_iters.  rhs: consistent, BC-projected P2VEC on l_max; x overwritten.  Synchronises once per
 * iteration (convergence check); iterations / final relative residual returned on the host. */
int hhg_ablock_cg(hhg_mg* mg, const double* rhs, double* x, double tol, int max_iters, int* iters,
                  double* rel_res, hhg_stream_t stream);
/* Same with HOST (pinned or pageable) rhs / x: H2D copy, V-cycle, D2H copy on `stream`. */
int vcycle_host(hhg_mg* mg, const double* rhs_host, double* x_host, hhg_stream_t stream);
/* nsteps V-cycles on HOST buffers, pipelined: step k's H2D copy, V-cycle and D2H copy each run on their own
 * stream so that the H2D of step k+1 and the D2H of step k-1 overlap V-cycle k (two device staging
 * pairs, event-ordered reuse).  rhs_host[k] / x_host[k]: pinned host pointers (repeats allowed).
 * Asynchronous: `stream` is complete once every x_host[k] is written. */
int vcycle_host_batch(hhg_mg* mg, const double* const* rhs_host, double* const* x_host, int nsteps,
                      hhg_stream_t stream);
/* Kernel timing of the fine-level element kernel inside vcycle (CUDA events on the
 * launching stream; disables graph capture while on).  get: sum of ms and count. */
int hhg_mg_profile(hhg_mg* mg, int enable);
int hhg_mg_profile_get(hhg_mg* mg, double* apply_ms_sum, int64_t* apply_count, double* cycle_ms_sum,
                       int64_t* cycle_count);
/* Of apply_ms_sum, the part spent in the dense-brick launch (k_elem_fp, the dominant kernel of the path:
 * P:275-287 evaluated brick by brick) -- an event is recorded between it and the sparse-brick launch
 * (k_elem_sparse).  Same count as apply_count.  dense_ms_sum: host pointer. */
int hhg_mg_profile_get_dense(hhg_mg* mg, double* dense_ms_sum);
int hhg_mg_destroy(hhg_mg* mg);

/* ------------------------------------------------------------------ Stokes solve
 * FGMRES (restarted every `restart` iterations) for the projected system
 * P [[A, B^T], [B+C, 0]] P [u; p] = P [f; g] (P_p = pressure mean zero),
 * right-preconditioned by the symmetric Uzawa block preconditioner (eq:SymmetricUzawaStep1,
 * P:427-437, B -> B+C in the pressure update) with A^-1 = V-cycle-preconditioned CG to tol_A
 * (hhg_ablock_cg on the hierarchy `mg`) and S^-1 = M_{1/eta}^-1 by Jacobi-CG to tol_mass
 * (eq:schurMass) or S^-1 = the V-cycle BFBT of eq:schurV (A_C = the cheap
 * hierarchy mg_cheap, e.g. V(1,1) with degree-1 Chebyshev; B A_C^-1 B^T inverted by CG
 * preconditioned by M_{1/eta} to tol_vbfbt).
 * Vectors: [u (P2VEC) | p (P1)] contiguous, device, on the hierarchy's finest level.  Stops at
 * |r| <= tol |P rhs| (2-norm over unique dofs) or max_iters.  Synchronises (host Arnoldi). */
typedef struct {
  int restart, max_iters;      /* FGMRES restart length and iteration cap */
  double tol;                  /* relative residual target of FGMRES */
  double sigma, omega;         /* Uzawa scalings (Table 1: 1, 0.3) */
  double tol_A;                /* A-block CG relative tolerance (Table 1: 1e-2) */
  int ablock_max_iters;
  double tol_mass;             /* M_{1/eta} CG relative tolerance (Table 1: 1e-10) */
  int mass_max_iters;
  int schur;                   /* 0: S = M_{1/eta} (eq:schurMass); 1: V-cycle BFBT (eq:schurV) */
  double tol_vbfbt;            /* CG tolerance for B A_C^-1 B^T (Table 1: 1e-1), M_{1/eta}-preconditioned */
  int vbfbt_max_iters;
  int uzawa;                   /* 0 symmetric (default), 1 inexact, 2 adjoint inexact */
  /* schur = 2: weighted BFBT (eq:schurWBFBT with the a_l / a_r surface scaling) */
  double a_l, a_r;             /* eta_l = a_l^2 eta, eta_r = a_r^2 eta on D_eta (1, 1: plain w-BFBT) */
  double tol_wbfbt;            /* K_{1/sqrt(eta)} GMG-CG: relative tolerance ... */
  double tol_wbfbt_abs;        /* ... or absolute residual 2-norm, whichever is met first */
  int wbfbt_max_iters;
  double tol_vmass;            /* M_{sqrt(eta)} Jacobi-CG relative tolerance (reading R24) */
  int vmass_max_iters;
} hhg_stokes_params;
typedef struct hhg_stokes hhg_stokes;
int hhg_stokes_create(hhg_mg* mg, hhg_mg* mg_cheap /*NULL unless schur = 1*/, const double* eta_p1, double gamma,
                      const hhg_stokes_params* params, hhg_stokes** out);
int hhg_stokes_solve(hhg_stokes* solver, const double* rhs, double* x, int* iters, double* rel_res,
                     hhg_stream_t stream);
int hhg_stokes_destroy(hhg_stokes* solver);
/* z = S^-1 t for the solver's Schur approximation (schur 0: M_{1/eta}^-1, 1: S_V^-1, 2: S_w^-1), without
 * the -omega of the Uzawa step; t: P1 on the finest level, projected to mean zero first; z mean zero.
 * Synchronises (inner CG stopping tests). */
int hhg_stokes_schur_apply(hhg_stokes* solver, const double* t, double* z, hhg_stream_t stream);

/* ------------------------------------------------------------------ weighted BFBT pieces (NEXT-3)
 * eq:schurWBFBT: S_w^-1 ~ K_{1/sqrt(eta_l)}^-1 (B M_{sqrt(eta_l)}^-1 A M_{sqrt(eta_r)}^-1 B^T)
 * K_{1/sqrt(eta_r)}^-1 with eta_a = a^2 eta on D_eta = the micro tets with a vertex on the outer sphere
 * (the radius of the HHG_BND_OUTER-tagged macro vertices; a != 1 needs a shell-blended mesh -> HHG_EINVAL).
 * hhg_kp1_apply: y = K_{1/sqrt(eta_a)} p, the P1 Laplacian weighted by 1/sqrt(eta_a) (P1 eta interpolated
 *   at the quadrature points), Neumann (no constraints); p consistent P1, y consistent P1 (overwritten).
 * hhg_kp1_diag: its diagonal.  hhg_vmass_apply: y = (P_v M) M_{sqrt(eta_a)} u, the P2 vector mass weighted
 *   by sqrt(eta_a) (u consistent, BC-projected P2VEC); hhg_vmass_diag: its diagonal (no P_v, like diag A).
 * eta_p1 NULL means eta = 1.  Asynchronous on `stream`. */
int hhg_kp1_apply(const hhg_mesh* mesh, int level, const double* eta_p1, double a, const double* p, double* y,
                  hhg_stream_t stream);
int hhg_kp1_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double a, double* diag, hhg_stream_t stream);
int hhg_vmass_apply(const hhg_mesh* mesh, int level, const double* eta_p1, double a, const double* u, double* y,
                    hhg_stream_t stream);
int hhg_vmass_diag(const hhg_mesh* mesh, int level, const double* eta_p1, double a, double* diag,
                   hhg_stream_t stream);
/* P1 transfers of the K multigrid: x_fine += P x_coarse (linear interpolation; consistent in, consistent
 * out); r_coarse = P^T r_fine over unique fine nodes, then the coarse interface sum (overwritten). */
int p1_prolong(const hhg_mesh* mesh, int coarse_level, const double* x_coarse, double* x_fine, hhg_stream_t stream);
int p1_restrict(const hhg_mesh* mesh, int fine_level, const double* r_fine, double* r_coarse, hhg_stream_t stream);
/* K_{1/sqrt(eta_a)}^-1 by CG preconditioned by a P1 GMG V-cycle ("a CG solver preconditioned by a
 * GMG approach"): Chebyshev(D^-1 K) smoothing, P1 transfers, coarse Jacobi-PCG, the smoother / level /
 * power-iteration settings of `params`; eta_per_level[l] P1 eta on level l (NULL entries: 1).
 * hhg_kmg_solve: from x = 0, rhs projected to mean zero, until |r| <= tol |r0| or |r| <= tol_abs or
 * max_iters; x mean zero.  Synchronises once per iteration. */
typedef struct hhg_kmg hhg_kmg;
int hhg_kmg_create(hhg_mesh* mesh, const hhg_mg_params* params, const double* const* eta_per_level, double a,
                   hhg_kmg** out);
int hhg_kmg_solve(hhg_kmg* kmg, const double* rhs, double* x, double tol, double tol_abs, int max_iters, int* iters,
                  double* rel_res, hhg_stream_t stream);
int hhg_kmg_destroy(hhg_kmg* kmg);

/* ------------------------------------------------------------------ temperature operator (NEXT-4, part)
 * eq:WeakTemp without the MMOC advection step: for P2 scalar T and test w
 *   L(T, w) = s int T w + tau [ int (u . grad T) w + int kappa grad T . grad(w / rho) - int beta T (u . g) w ]
 * with rho = exp(gamma (1 - |x|)) (grad ln rho = -gamma x/|x|), g = -x/|x|, u a P2VEC velocity;
 *   P(T, w) = s int T w + tau int (kappa / rho) grad T . grad w   (the symmetric mass + diffusion part).
 * s = s^{n+1} of the BDF2 step, tau = tau^{n+1}, kappa = k/(Pe C_p), beta = Di alpha / C_p. */
typedef struct {
  double s, tau, kappa, beta, gamma;
} hhg_temp_params;
/* y = L T (which 0), P T (1) or diag(P) (2, T ignored); unconstrained, interface-summed, overwritten.
 * u: consistent P2VEC (which 0 only), T / y: consistent P2 scalars on `level`. */
int hhg_temp_apply(const hhg_mesh* mesh, int level, const hhg_temp_params* prm, const double* u, const double* T,
                   double* y, int which, hhg_stream_t stream);
/* The temperature solve of P:548: FGMRES (restarted, right-preconditioned by CG on P with the inverse
 * diagonal, to tol_cg) for L T = b at interior nodes with T fixed on the boundary nodes that carry a
 * velocity BC (surface and CMB for the shell).  T: in = Dirichlet values on those nodes (interior entries
 * ignored), out = solution.  Stops at |r| <= tol |r0| or |r| <= tol_abs (2-norm over unique interior
 * nodes) or max_iters.  Workspace allocated in create.  Synchronises (host Arnoldi). */
typedef struct hhg_temp_solver hhg_temp_solver;
int hhg_temp_solver_create(hhg_mesh* mesh, int level, const hhg_temp_params* prm, int restart, hhg_temp_solver** out);
int hhg_temp_solve(hhg_temp_solver* S, const double* u, const double* b, double* T, double tol, double tol_abs,
                   int max_iters, double tol_cg, int cg_max_iters, int* iters, double* rel_res, hhg_stream_t stream);
int hhg_temp_solver_destroy(hhg_temp_solver* S);
/* MMOC step: T_hat(x) = T(X(x)) at every P2 node x, X = RK4 back-tracking over tau along
 * u(y, th) = (1 - th) u_new(y) + th u_old(y) (linear in time between t^{n+1} and t^n); fields evaluated
 * at located points (inverse blending, macro, lattice cube, micro tet, P2 basis); points leaving the
 * shell are moved radially onto it.  T, T_hat: consistent P2 scalars; u_*: consistent P2VEC.
 * Synchronises; HHG_EINVAL if a point cannot be located (non-shell meshes: a point left the domain) or the
 * mesh is partitioned over several ranks (particles would need the neighbours' macros). */
int hhg_mmoc(const hhg_mesh* mesh, int level, const double* T, const double* u_new, const double* u_old, double tau,
             double* T_hat, hhg_stream_t stream);

/* Number of kernels launched by the library on this thread since the last reset. */
int64_t hhg_launch_count(int reset);

#ifdef __cplusplus
}
#endif
#endif /* HHG_STOKES_H */
