// Element kernel of the hot path (sm_100a, fp64 DFMA pipe -- the operator is not a dense
// contraction, and B200's fp64 tensor path runs at the DFMA rate, so no tensor cores).
//
// Work decomposition ("brick"): the P1 lattice of a macro (resolution n = 2^L) is cut into
// 4x4x4 blocks of lattice cubes; one CTA of 64 threads owns one block.  A cube holds up to 6
// micro tets (Bey/Freudenthal refinement):
//   type 0 up {000,100,010,001}, 1-4 octahedron around diagonal 010-101, 5 down {011,101,110,111};
// a cube with anchor sum s has 6 tets if s <= n-3, 5 if s == n-2, 1 if s == n-1.
//  * k_elem_fp (v6): the brick's 9x9x9-point P2 footprint of u (and eta / p on the 5x5x5 P1
//    footprint, and the macro's element geometry) is staged in shared memory with cp.async; one
//    thread per cube loops over its tets, all lanes of a warp on the same type; element outputs are
//    added into a per-warp output footprint in 4 conflict-free rounds (the 6 edge midpoints of a tet
//    have pairwise different parity classes, the 4 vertices take one round each; sm_100a has no
//    native fp64 shared atomics), then the CTA writes the footprint: plain stores inside, one fp64
//    RED per footprint-border point (shared with neighbouring bricks).
//  * sparse bricks (those cut by the macro's slanted face with <= 64 tets): one thread per tet,
//    outputs go straight to global memory with fp64 REDs (the dense loop would run 6 iterations
//    for 1 tet per thread on these bricks).
//  History (v1 thread-per-tet, v2 private slots, v5 slot gather): DESIGN.md §6.
//
// Per tet (tet_body): gather 30 velocity dofs (+4 eta, +4 p), evaluate the blending map at the 4
// quadrature points on the fly, and form 2 eta dev(eps(u)),
// -p I (B^T) and -(div u + grad ln rho . u) (B+C).  Arithmetic layout:
//   * reference gradients in barycentric form: D_m(q) = Dt_m + 4 x_m(q) (scaled by 1/(a-b)),
//     Dt_m = (sqrt5-1) sum_j u_mj - u_m, x_m(q) = u_m if m == q else u_mq;
//   * blending: with s = |x|^2, t = n.x, the physical gradient is grad_ref . K / (c alpha) with
//     K = J_F^-1 - (J_F^-1 x) z^T, z = n/t - x/s, alpha = t/sqrt(s)  (rank-one closed form of
//     J_B^-1, one rsqrt + one reciprocal per point, both MUFU-seeded + Newton);
//   * the transposed map scatters R = S K^T through Sbar_m = sum_q Db_m(q) (vertex: -Sbar/4 +
//     Db_m(m), edge: (sqrt5-1)/4 (Sbar_m + Sbar_j) + Db_m(j) + Db_j(m)), all constant factors
//     folded into the per-point weight.
#include <algorithm>

#include "hhg_internal.h"
#include "hhg_device.cuh"
#include "hhg_tet.cuh"

namespace hhg {

constexpr int kBT = 64;  // threads per CTA of k_elem_sparse (one thread per tet of a sparse brick)
// k_elem_fp: one CTA per brick of 4x4x4 lattice cubes, kWT thread groups of 64 (one thread per cube each); group g
// evaluates tet types [g 6/kWT, (g+1) 6/kWT) of every cube into its own pair of per-warp output footprints, so more
// warps share one staged u footprint.  kWT = 2 (4 warps, 3 CTAs = 12 warps per SM instead of 5 x 2) measured SLOWER
// on B200 (L5 0.691 vs 0.644 ms, profiles/r02_tsplit_elem.jsonl: twice the footprint zeroing and write-out sums), so
// the default stays kWT = 1; -DHHG_TSPLIT=2 builds the variant.
#ifndef HHG_TSPLIT
#define HHG_TSPLIT 1
#endif
constexpr int kWT = HHG_TSPLIT;
static_assert(6 % kWT == 0, "type groups");
constexpr int kBTD = 64 * kWT;

// 32-bit lattice helpers (N <= 512 keeps (N+1)(N+2)(N+3) < 2^31)
__device__ __forceinline__ int kbase32(int N, int k) {  // first index of plane k
  const int M = N - k;
  return ((N + 1) * (N + 2) * (N + 3) - (M + 1) * (M + 2) * (M + 3)) / 6;
}
__device__ __forceinline__ int rowstart32(int N, int j, int k) {  // index of (0, j, k)
  const int m = N - k;
  return kbase32(N, k) + (j * (2 * m + 3 - j)) / 2;
}


// ---------------------------------------------------------------- tables (uploaded once)
// Per tet type t and local node a: cube-local P2 slot sl = dx + 3dy + 9dz of the doubled offset,
// packed load index (row (dy + 3dz) << 2 | dx), first-touch flags in type order 0..5 (the first
// touch of a cube slot stores, later touches add), P1 corner slots; sparse-brick item lists.
constexpr int kNS2 = 81;  // P2 slots per cube (27 nodes x 3)
constexpr int kNS1 = 8;   // P1 slots per cube
__constant__ int eSlot[6][10];
__constant__ int eLd[6][10];
__constant__ int ePSlot[6][4];
__constant__ int eFirst[6];
__constant__ int ePFirst[6];
__device__ int eItems[5][64];  // delta = n - (i0+j0+k0) in 1..4: item = cube | type << 6
__device__ int eNItems[5];

constexpr int kGeoSm = 6 * kTypeGeo + 2;  // staged per-macro element geometry (doubles)

// Array accessor for tet_body
struct RegU {
  const double (&u)[10][3];
  __device__ __forceinline__ double operator()(int a, int c) const { return u[a][c]; }
};

// ================================================================ element kernel v6 ("footprint")
// The brick's u footprint (9x9x9 doubled-lattice points x 3 comps) and P1 footprint (eta, p) are
// staged in shared memory with cp.async; every tet reads its dofs with LDS at table offsets.
// Outputs accumulate in a PER-WARP output footprint (warp w owns cube layers z = 2w, 2w+1, i.e.
// points Z in [4w, 4w+4]) with plain load-add-store in 4 rounds separated by __syncwarp: in one
// round all lanes (same tet type, different cubes) update the same local node index, hence
// distinct points; the 6 edge midpoints of a tet have pairwise different parity classes (host-
// checked), so they share one round with vertex 0, and vertices 1-3 take one round each.  No atomics and no
// per-cube slots.  After __syncthreads the CTA writes the footprint: plain stores inside, fp64 RED
// on the footprint border (shared with neighbouring bricks), the two warps' Z = 4 planes summed.
// Layout word(X,Y,Z) = xs(X) + kPY*Y + kPZ*Z, xs(X) = X/2 (even X) or 5 + X/2 (odd X): lanes
// (x,y) of a half-warp then hit x + 20y + const -> 16 distinct 8-byte bank pairs.
constexpr int kPY = 10, kPZ = 9 * kPY;     // row / plane pitch (words)
constexpr int kFU = 9 * kPZ;               // u footprint words per component (810)
constexpr int kFY = 5 * kPZ;               // per-warp output footprint words per component (450)
constexpr int kF1 = 125, kF1Y = 75;        // P1 footprints: brick 5x5x5, per warp 5x5x3
__host__ __device__ constexpr int xs(int X) { return (X & 1) ? 5 + (X >> 1) : (X >> 1); }
__host__ __device__ constexpr int fword(int X, int Y, int Z) { return xs(X) + kPY * Y + kPZ * Z; }
__constant__ int eOffU[6][10];  // footprint word offset of each local node from its cube's base word
__constant__ int eOffB[6][10];  // the same in bytes (LDS/STS [reg + uniform] addressing)
__constant__ int eOffP[6][4];   // P1 footprint offset of each vertex from the cube's P1 base

struct FootU {
  const char* b;    // su + cube base word, as a byte address
  const int* off;   // eOffB[t] (bytes)
  __device__ __forceinline__ double operator()(int a, int c) const {
    return *reinterpret_cast<const double*>(b + off[a] + c * (kFU * 8));
  }
};

struct FootT {  // scalar P2 footprint (temperature) for the quadrature-point viscosity tier
  const char* b;
  const int* off;
  __device__ __forceinline__ double operator()(int a) const { return *reinterpret_cast<const double*>(b + off[a]); }
};

template <int MODE, bool ETAQ = false>
__host__ __device__ constexpr int fp_smem_words() {
  return (elem_need_u(MODE) ? 3 * kFU : 0) + (elem_u_out(MODE) ? 2 * kWT * 3 * kFY : 0) +
         kF1 + (elem_need_p(MODE) ? kF1 : 0) + (elem_p_out(MODE) ? 2 * kWT * kF1Y : 0) + kGeoSm +
         (ETAQ ? kFU : 0);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

constexpr int kMG = 26;  // MacroGeo (doubles)
static_assert(sizeof(MacroGeo) == kMG * sizeof(double), "MacroGeo layout");

// k_elem_fp (v6): one CTA per (brick of `bricks` = blockIdx.x, macro = blockIdx.y).  det != 0
// (deterministic mode, one launch per brick colour -- bricks of one colour share no footprint point):
// border points use plain load-add-store instead of fp64 REDs and sparse bricks take the dense path, so
// the result is bitwise reproducible.
template <bool BLEND, int MODE, bool FULL, bool ETAQ = false, int EPI = EPI_NONE>
#ifndef HHG_FP_MINB
#define HHG_FP_MINB (kWT == 1 ? 5 : 2)  // kWT = 2: (128, 3) makes ptxas spill at 168 registers; (128, 2) fits in <= 170 = 3 CTAs/SM
#endif
__global__ void __launch_bounds__(kBTD, HHG_FP_MINB)
    k_elem_fp(const MacroGeo* __restrict__ mgeo, const double* __restrict__ lgeo, const int32_t* __restrict__ bricks,
              int nb, int n1, double inv_n1, int64_t npts1, int64_t npts2, int64_t cstride,
              const double* __restrict__ eta, const double* u, const double* __restrict__ p,
              double* __restrict__ yu, double* __restrict__ yp, double gamma, const double* __restrict__ T2, EtaQ eq,
              int det, ChebEpi ep) {
  (void)nb;
  constexpr bool NEED_U = elem_need_u(MODE);
  constexpr bool NEED_P = elem_need_p(MODE);
  constexpr bool HAS_P_OUT = elem_p_out(MODE);
  constexpr bool HAS_U_OUT = elem_u_out(MODE);
  extern __shared__ double sm[];
  double* su = sm;                                   // [3][kFU]
  double* sy = su + (NEED_U ? 3 * kFU : 0);          // [kWT groups][2 warps][3][kFY]
  double* se = sy + (HAS_U_OUT ? 2 * kWT * 3 * kFY : 0);  // [kF1]
  double* sp = se + kF1;                             // [kF1]
  double* syp = sp + (NEED_P ? kF1 : 0);             // [kWT groups][2 warps][kF1Y]
  double* sgeo = syp + (HAS_P_OUT ? 2 * kWT * kF1Y : 0);  // [kGeoSm]
  double* stt = sgeo + kGeoSm;                       // [kFU] temperature footprint (ETAQ)

  const int mac = blockIdx.y;
  const int32_t bpk = __ldg(bricks + blockIdx.x);
  const int i0 = bpk & 1023, j0 = (bpk >> 10) & 1023, k0 = bpk >> 20;
  const int delta = n1 - (i0 + j0 + k0);
  const int tid = threadIdx.x;
  const int n2 = 2 * n1;
  const int64_t mb2 = (int64_t)mac * npts2, mb1 = (int64_t)mac * npts1;

  // ---- row starts of the brick's footprint rows (P2: 9x9 rows (Y, Z), P1: 5x5), computed once per CTA and
  // shared by the staging and write-out loops (rows outside the lattice hold garbage and are never used)
#ifndef HHG_EXP_NOSROW
  __shared__ int srow2[81], srow1[25];
  for (int r = tid; r < 81 + 25; r += kBTD) {
    if (r < 81) srow2[r] = rowstart32(n2, 2 * j0 + r % 9, 2 * k0 + r / 9);
    else srow1[r - 81] = rowstart32(n1, j0 + (r - 81) % 5, k0 + (r - 81) / 5);
  }
  __syncthreads();
#define HHG_ROW2(gy, gz, Y, Z) srow2[(Y) + 9 * (Z)]
#define HHG_ROW1(gy, gz, Y, Z) srow1[(Y) + 5 * (Z)]
#else
#define HHG_ROW2(gy, gz, Y, Z) rowstart32(n2, gy, gz)
#define HHG_ROW1(gy, gz, Y, Z) rowstart32(n1, gy, gz)
#endif
  // ---- stage: u footprint (cp.async), eta / p footprints, geometry; zero the output footprints
  const double* Gm = lgeo + (int64_t)mac * kLevelGeo;
  for (int r = tid; r < kGeoSm; r += kBTD) cp_async8(sgeo + r, Gm + r);
#ifdef HHG_EXP_ROWSTAGE
  // one (row, component) item per thread: 2 row-start evaluations per thread, 9 cp.async per item
  if (NEED_U || ETAQ) {
    constexpr int NI = (NEED_U ? 243 : 0) + (ETAQ ? 81 : 0);
#pragma unroll 1
    for (int it = tid; it < NI; it += kBTD) {
      const int c = it / 81, r = it - 81 * c;
      const int Y = r % 9, Z = r / 9;
      const int gy = 2 * j0 + Y, gz = 2 * k0 + Z;
      const int len = min(9, n2 - 2 * i0 - gy - gz + 1);
      if (len <= 0) continue;
      const int o = rowstart32(n2, gy, gz) + 2 * i0;
      const double* sr = (NEED_U && c < 3) ? u + mb2 + c * cstride + o : T2 + mb2 + o;
      double* d = ((NEED_U && c < 3) ? su + c * kFU : stt) + kPY * Y + kPZ * Z;
#pragma unroll
      for (int X = 0; X < 9; ++X)
        if (X < len) cp_async8(d + xs(X), sr + X);
    }
  }
#else
  if (NEED_U) {
#pragma unroll 1
    for (int L = tid; L < 729; L += kBTD) {
      const int X = L % 9, Y = (L / 9) % 9, Z = L / 81;
      const int gx = 2 * i0 + X, gy = 2 * j0 + Y, gz = 2 * k0 + Z;
      if (gx + gy + gz > n2) continue;
      const double* src = u + mb2 + HHG_ROW2(gy, gz, Y, Z) + gx;
      HHG_CHECK(src - u >= mb2 && src - u < mb2 + npts2 && mb2 + npts2 <= cstride, "u stage", src - u, cstride);
      const int w = fword(X, Y, Z);
#pragma unroll
      for (int c = 0; c < 3; ++c) cp_async8(su + c * kFU + w, src + c * cstride);
    }
  }
  if (ETAQ) {
#pragma unroll 1
    for (int L = tid; L < 729; L += kBTD) {
      const int X = L % 9, Y = (L / 9) % 9, Z = L / 81;
      const int gx = 2 * i0 + X, gy = 2 * j0 + Y, gz = 2 * k0 + Z;
      if (gx + gy + gz > n2) continue;
      cp_async8(stt + fword(X, Y, Z), T2 + mb2 + HHG_ROW2(gy, gz, Y, Z) + gx);
    }
  }
#endif
#ifdef HHG_EXP_PF
  // warm L2 for the brick whose CTA is dispatched after this one's wave (CTA index + resident CTAs):
  // its cp.async staging then hits L2 instead of DRAM
  if (NEED_U) {
    const unsigned nbx = gridDim.x, b2 = blockIdx.y * nbx + blockIdx.x + HHG_EXP_PF;
    if (b2 < nbx * gridDim.y) {
      const int mac2 = b2 / nbx;
      const int32_t bp2 = __ldg(bricks + (b2 - mac2 * nbx));
      const int a2 = bp2 & 1023, c2 = (bp2 >> 10) & 1023, d2 = bp2 >> 20;
      const double* ub2 = u + (int64_t)mac2 * npts2;
      for (int it = tid; it < 243; it += kBTD) {
        const int c = it / 81, r = it - 81 * c;
        const int gy = 2 * c2 + r % 9, gz = 2 * d2 + r / 9;
        const int len = min(9, n2 - 2 * a2 - gy - gz + 1);
        if (len <= 0) continue;
        const double* rp = ub2 + c * cstride + rowstart32(n2, gy, gz) + 2 * a2;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(rp));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + len - 1));
      }
    }
  }
#endif
  if (HAS_U_OUT)
    for (int r = tid; r < 2 * kWT * 3 * kFY; r += kBTD) sy[r] = 0.0;
  if (HAS_P_OUT)
    for (int r = tid; r < 2 * kWT * kF1Y; r += kBTD) syp[r] = 0.0;
  for (int L = tid; L < kF1; L += kBTD) {  // P1 footprint (points outside the lattice are never read)
    const int X = L % 5, Y = (L / 5) % 5, Z = L / 25;
    const int gx = i0 + X, gy = j0 + Y, gz = k0 + Z;
    if (gx + gy + gz > n1) continue;
    const int64_t ix = mb1 + HHG_ROW1(gy, gz, Y, Z) + gx;
    HHG_CHECK(ix >= mb1 && ix < mb1 + npts1 && ix < (int64_t)gridDim.y * npts1, "P1 stage", ix, npts1);
    if (eta != nullptr) cp_async8(se + L, eta + ix);
    else se[L] = 1.0;
    if (NEED_P) cp_async8(sp + L, p + ix);
  }
  const MacroGeo& g = mgeo[mac];
  double nh[3] = {0, 0, 0}, cK = 1.0;
  if (BLEND) {
    nh[0] = g.nhat[0];
    nh[1] = g.nhat[1];
    nh[2] = g.nhat[2];
    cK = g.cK;
  }
  cp_async_wait_all();
  __syncthreads();
  const double wdet = EWQ * sgeo[6 * kTypeGeo];

  auto anchor = [&](int x, int y, int z, double (&xa)[3]) {
    const double fa = (i0 + x) * inv_n1, fb = (j0 + y) * inv_n1, fc = (k0 + z) * inv_n1;  // exact: n1 = 2^L
#pragma unroll
    for (int r = 0; r < 3; ++r) xa[r] = g.X0[r] + g.Jm[3 * r] * fa + g.Jm[3 * r + 1] * fb + g.Jm[3 * r + 2] * fc;
  };

  if (delta <= 4 && !det) {
#ifdef HHG_EXP_NOSPARSE
    return;
#endif
    // ---------------- sparse brick (<= 64 tets, mixed types per warp): one tet per thread, REDs
    if (tid >= eNItems[delta]) return;
    const int item = eItems[delta][tid];
    const int cube = item & 63, t = item >> 6;
    const int x = cube & 3, y = (cube >> 2) & 3, z = cube >> 4;
    double xa[3];
    anchor(x, y, z, xa);
    const int cb2 = x + 2 * kPY * y + 2 * kPZ * z, cb1 = x + 5 * y + 25 * z;
    double et[4], pp[4] = {0, 0, 0, 0}, acc[10][3], gy[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      et[v] = se[cb1 + eOffP[t][v]];
      if (NEED_P) pp[v] = sp[cb1 + eOffP[t][v]];
    }
    tet_body<BLEND, MODE, FULL, FootU, ETAQ, FootT>(sgeo + t * kTypeGeo, wdet, xa, nh, cK, gamma,
                                                    FootU{reinterpret_cast<const char*>(su + cb2), eOffB[t]}, et, pp,
                                                    acc, gy, FootT{reinterpret_cast<const char*>(stt + cb2), eOffB[t]}, eq);
    if (HAS_U_OUT) {
#pragma unroll
      for (int a = 0; a < 10; ++a) {
        const int o = eOffU[t][a];  // decode the footprint point of node a
        const int Z = o / kPZ, Y = (o % kPZ) / kPY, xw = o % kPY;
        const int X = xw >= 5 ? 2 * (xw - 5) + 1 : 2 * xw;
        double* dst = yu + mb2 + rowstart32(n2, 2 * (j0 + y) + Y, 2 * (k0 + z) + Z) + 2 * (i0 + x) + X;
        HHG_CHECK(dst - yu >= mb2 && dst - yu < mb2 + npts2, "sparse RED", dst - yu, mb2 + npts2);
#pragma unroll
        for (int c = 0; c < 3; ++c) atomicAdd(dst + c * cstride, acc[a][c]);
      }
    }
    if (HAS_P_OUT) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int o = eOffP[t][v];
        const int X = o % 5, Y = (o / 5) % 5, Z = o / 25;
        atomicAdd(yp + mb1 + rowstart32(n1, j0 + y + Y, k0 + z + Z) + i0 + x + X, gy[v]);
      }
    }
    return;
  }

  // ---------------- dense brick: thread = cube, all lanes of a warp on the same tet type
  const int x = tid & 3, y = (tid >> 2) & 3, z = (tid >> 4) & 3;
  const int wz = z >> 1, grp = tid >> 6;  // cube-layer pair of this warp, type group
  const int s = i0 + j0 + k0 + x + y + z;
  const int ntypes = (s <= n1 - 3) ? 6 : ((s == n1 - 2) ? 5 : ((s == n1 - 1) ? 1 : 0));
  double xa[3];
  anchor(x, y, z, xa);
  const int cb2 = x + 2 * kPY * y + 2 * kPZ * z, cb1 = x + 5 * y + 25 * z;
  const int fw = 2 * grp + wz;  // this warp's output footprints
  double* yw = sy + fw * 3 * kFY + (x + 2 * kPY * y + 2 * kPZ * (z - 2 * wz));
  double* ypw = syp + fw * kF1Y + (x + 5 * y + 25 * (z - 2 * wz));
  constexpr int kTPG = 6 / kWT;
#pragma unroll 1
  for (int t = grp * kTPG; t < (grp + 1) * kTPG; ++t) {
    const bool act = t < ntypes;
    double acc[10][3], gy[4];
    if (act) {
      double et[4], pp[4] = {0, 0, 0, 0};
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        et[v] = se[cb1 + eOffP[t][v]];
        if (NEED_P) pp[v] = sp[cb1 + eOffP[t][v]];
      }
#ifdef HHG_EXP_NOBODY
      {
        FootU fu{reinterpret_cast<const char*>(su + cb2), eOffB[t]};
#pragma unroll
        for (int a = 0; a < 10; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[a][c] = fu(a, c) * et[0];
#pragma unroll
        for (int v = 0; v < 4; ++v) gy[v] = pp[v];
      }
#else
      tet_body<BLEND, MODE, FULL, FootU, ETAQ, FootT>(sgeo + t * kTypeGeo, wdet, xa, nh, cK, gamma,
                                                      FootU{reinterpret_cast<const char*>(su + cb2), eOffB[t]}, et, pp,
                                                      acc, gy, FootT{reinterpret_cast<const char*>(stt + cb2), eOffB[t]}, eq);
#endif
    }
    const int* off = eOffB[t];
    char* ywb = reinterpret_cast<char*>(yw);
    auto Y = [&](int a, int c) -> double& { return *reinterpret_cast<double*>(ywb + off[a] + c * (kFY * 8)); };
    // round 0: the 6 edge midpoints (pairwise different parity classes, none even-even-even) and
    // vertex 0 (parity 000) -- 7 nodes of pairwise different parity; rounds 1..3: one vertex each
    if (act) {
      if (HAS_U_OUT) {
        double old[7][3];
#pragma unroll
        for (int e = 0; e < 7; ++e)
#pragma unroll
          for (int c = 0; c < 3; ++c) old[e][c] = Y(e < 6 ? 4 + e : 0, c);
#pragma unroll
        for (int e = 0; e < 7; ++e)
#pragma unroll
          for (int c = 0; c < 3; ++c) Y(e < 6 ? 4 + e : 0, c) = old[e][c] + acc[e < 6 ? 4 + e : 0][c];
      }
      if (HAS_P_OUT) ypw[eOffP[t][0]] += gy[0];
    }
    __syncwarp();
#pragma unroll
    for (int a = 1; a < 4; ++a) {
      if (act) {
        if (HAS_U_OUT) {
#pragma unroll
          for (int c = 0; c < 3; ++c) Y(a, c) += acc[a][c];
        }
        if (HAS_P_OUT) ypw[eOffP[t][a]] += gy[a];
      }
      __syncwarp();
    }
  }
  __syncthreads();

  // ---- write the brick's output footprint: plain stores inside, fp64 RED (deterministic mode: plain
  // load-add-store) on the footprint border shared with neighbouring bricks; the two warps' Z = 4 planes
  // are summed first
  if (HAS_U_OUT) {
#pragma unroll 1
    for (int L = tid; L < 729; L += kBTD) {
      const int X = L % 9, Y = (L / 9) % 9, Z = L / 81;
      const int gx = 2 * i0 + X, gy = 2 * j0 + Y, gz = 2 * k0 + Z;
      if (gx + gy + gz > n2) continue;
      const int wxy = xs(X) + kPY * Y;
      double* dst = yu + mb2 + HHG_ROW2(gy, gz, Y, Z) + gx;
      HHG_CHECK(dst - yu >= mb2 && dst - yu < mb2 + npts2, "write-out", dst - yu, mb2 + npts2);
      const bool border = X == 0 || Y == 0 || Z == 0 || X == 8 || Y == 8 || Z == 8;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < kWT; ++g2) {  // type groups in fixed order
          const double* f = sy + g2 * 6 * kFY + c * kFY + wxy;
          if (Z < 4) v += f[kPZ * Z];
          else if (Z > 4) v += f[3 * kFY + kPZ * (Z - 4)];
          else v += f[kPZ * 4] + f[3 * kFY];
        }
        if (EPI != EPI_NONE && !border && !det && gx + gy + gz < n2) {
          // fused consumer update (launch_elem_epi): this point is complete, inside the macro, BC-free
          const int64_t j = (dst - yu) + c * cstride;
          if (EPI == EPI_SUB) {
            ep.r[j] = ep.f[j] - v;
          } else if (EPI == EPI_CHEB0) {
            const double ri = ep.f[j] - v;
            ep.r[j] = ri;
            ep.d[j] = ep.dinv[j] * ri * ep.c1;
          } else {
            const double di = su[c * kFU + xs(X) + kPY * Y + kPZ * Z];  // the apply input d at this point
            if (EPI == EPI_CHEBK) {
              ep.x[j] += di;
              const double ri = ep.r[j] - v;
              ep.r[j] = ri;
              ep.d[j] = ep.c1 * di + ep.c2 * ep.dinv[j] * ri;
            } else {
              const double dn = ep.c1 * di + ep.c2 * ep.dinv[j] * (ep.r[j] - v);
              ep.x[j] += di + dn;
            }
          }
        } else if (!border) {
          dst[c * cstride] = v;
        } else if (v != 0.0) {
          if (det) dst[c * cstride] += v;
          else atomicAdd(dst + c * cstride, v);
        }
      }
    }
  }
  if (HAS_P_OUT) {
    for (int L = tid; L < kF1; L += kBTD) {
      const int X = L % 5, Y = (L / 5) % 5, Z = L / 25;
      const int gx = i0 + X, gy = j0 + Y, gz = k0 + Z;
      if (gx + gy + gz > n1) continue;
      double v = 0.0;
#pragma unroll
      for (int g2 = 0; g2 < kWT; ++g2) {
        const double* f = syp + g2 * 2 * kF1Y + X + 5 * Y;
        if (Z < 2) v += f[25 * Z];
        else if (Z > 2) v += f[kF1Y + 25 * (Z - 2)];
        else v += f[50] + f[kF1Y];
      }
      double* dst = yp + mb1 + HHG_ROW1(gy, gz, Y, Z) + gx;
      const bool border = X == 0 || Y == 0 || Z == 0 || X == 4 || Y == 4 || Z == 4;
      if (!border) *dst = v;
      else if (v != 0.0) {
        if (det) *dst += v;
        else atomicAdd(dst, v);
      }
    }
  }
#undef HHG_ROW2
#undef HHG_ROW1
}

// ================================================================ sparse bricks without staging
// The bricks cut by the macro's slanted face (delta <= 4, <= 64 tets: 30 % of the bricks at L5, all of them on
// levels <= 2) hold few tets, so staging their 9x9x9 footprint in 43 KB of shared memory costs more than the
// tets themselves.  k_elem_sparse runs them in a launch of their own without shared memory: one thread per tet
// reads its 30 velocity dofs (+ eta, p, T at the nodes) straight from global memory (L1/L2 resident: the
// brick's tets share their nodes) and adds its outputs with fp64 REDs, as the sparse path of k_elem_fp did.
struct GlobU {  // u(a, c) = u[base + ix[a] + c * cs]
  const double* b;
  const int (&ix)[10];
  int64_t cs;
  __device__ __forceinline__ double operator()(int a, int c) const { return __ldg(b + ix[a] + c * cs); }
};
struct GlobT {
  const double* b;
  const int (&ix)[10];
  __device__ __forceinline__ double operator()(int a) const { return __ldg(b + ix[a]); }
};

template <bool BLEND, int MODE, bool FULL, bool ETAQ = false>
__global__ void __launch_bounds__(kBT)
    k_elem_sparse(const MacroGeo* __restrict__ mgeo, const double* __restrict__ lgeo, const int32_t* __restrict__ bricks,
                  int n1, double inv_n1, int64_t npts1, int64_t npts2, int64_t cstride, const double* __restrict__ eta,
                  const double* __restrict__ u, const double* __restrict__ p, double* __restrict__ yu,
                  double* __restrict__ yp, double gamma, const double* __restrict__ T2, EtaQ eq) {
  constexpr bool NEED_P = elem_need_p(MODE);
  const int mac = blockIdx.y;
  const int32_t bpk = __ldg(bricks + blockIdx.x);
  const int i0 = bpk & 1023, j0 = (bpk >> 10) & 1023, k0 = bpk >> 20;
  const int delta = n1 - (i0 + j0 + k0);
  const int tid = threadIdx.x;
  if (tid >= eNItems[delta]) return;
  const int item = eItems[delta][tid];
  const int cube = item & 63, t = item >> 6;
  const int x = i0 + (cube & 3), y = j0 + ((cube >> 2) & 3), z = k0 + (cube >> 4);
  const int n2 = 2 * n1;
  const int64_t mb2 = (int64_t)mac * npts2, mb1 = (int64_t)mac * npts1;
  const MacroGeo& g = mgeo[mac];
  const double* G = lgeo + (int64_t)mac * kLevelGeo;
  double nh[3] = {0, 0, 0}, cK = 1.0;
  if (BLEND) {
    nh[0] = g.nhat[0];
    nh[1] = g.nhat[1];
    nh[2] = g.nhat[2];
    cK = g.cK;
  }
  double xa[3];
  {
    const double fa = x * inv_n1, fb = y * inv_n1, fc = z * inv_n1;  // exact: n1 = 2^L
#pragma unroll
    for (int r = 0; r < 3; ++r) xa[r] = g.X0[r] + g.Jm[3 * r] * fa + g.Jm[3 * r + 1] * fb + g.Jm[3 * r + 2] * fc;
  }
  int ix[10];  // P2 node indices within the macro
#pragma unroll
  for (int a = 0; a < 10; ++a) {
    const int sl = eSlot[t][a];
    const int dx = sl % 3, dy = (sl / 3) % 3, dz = sl / 9;
    ix[a] = rowstart32(n2, 2 * y + dy, 2 * z + dz) + 2 * x + dx;
    HHG_CHECK(ix[a] >= 0 && ix[a] < npts2, "sparse node", ix[a], npts2);
  }
  int iv[4];  // P1 vertex indices within the macro
  double et[4], pp[4] = {0, 0, 0, 0};
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int ps = ePSlot[t][v];
    iv[v] = rowstart32(n1, y + ((ps >> 1) & 1), z + (ps >> 2)) + x + (ps & 1);
    HHG_CHECK(iv[v] >= 0 && iv[v] < npts1, "sparse vertex", iv[v], npts1);
    et[v] = eta != nullptr ? __ldg(eta + mb1 + iv[v]) : 1.0;
    if (NEED_P) pp[v] = __ldg(p + mb1 + iv[v]);
  }
  double acc[10][3], gy[4];
  tet_body<BLEND, MODE, FULL, GlobU, ETAQ, GlobT>(G + t * kTypeGeo, EWQ * __ldg(G + 6 * kTypeGeo), xa, nh, cK, gamma,
                                                  GlobU{u ? u + mb2 : u, ix, cstride}, et, pp, acc, gy,
                                                  GlobT{T2 ? T2 + mb2 : T2, ix}, eq);
  if (elem_u_out(MODE)) {
#pragma unroll
    for (int a = 0; a < 10; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) atomicAdd(yu + mb2 + ix[a] + c * cstride, acc[a][c]);
  }
  if (elem_p_out(MODE)) {
#pragma unroll
    for (int v = 0; v < 4; ++v) atomicAdd(yp + mb1 + iv[v], gy[v]);
  }
}

// Launch of one element-kernel instantiation: one CTA per (macro, brick) item, one launch over the dense bricks
// plus one k_elem_sparse launch over the sparse ones -- or, in deterministic mode, one launch per brick colour
// (sparse bricks on the dense path).
// A/B switch: HHG_NO_SPLIT=1 runs the sparse bricks inside k_elem_fp (staged path) as before
cudaEvent_t g_elem_mid_event = nullptr;
// The dense and the sparse launch of one operator application touch common points only through fp64 REDs (brick
// borders), so they are order-independent: the sparse launch (latency-bound, 12 warps/SM of 165 registers, no shared
// memory) runs on a side stream and its CTAs fill the register space the shared-memory-limited dense CTAs leave free.
// A/B switch: HHG_NO_CONC=1 launches them one after the other on the caller's stream.
static const bool g_no_conc = [] {
  const char* e = getenv("HHG_NO_CONC");
  return e && e[0] == '1';
}();
int elem_side_prepare(const Mesh* m, cudaStream_t s) {
  if (g_no_conc || m->side.count(s)) return HHG_OK;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  HHG_CUDA(cudaStreamIsCapturing(s, &st));
  if (st != cudaStreamCaptureStatusNone) return HHG_OK;  // never create under capture
  Mesh::Side sd;
  HHG_CUDA(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
  HHG_CUDA(cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming));
  HHG_CUDA(cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming));
  m->side[s] = sd;
  return HHG_OK;
}
static const bool g_no_split = [] {
  const char* e = getenv("HHG_NO_SPLIT");
  return e && e[0] == '1';
}();

template <bool BLEND, int MODE, bool FULL, bool ETAQ, int EPI = EPI_NONE>
struct ElemKernel {
  static constexpr size_t smem = fp_smem_words<MODE, ETAQ>() * sizeof(double);
  static bool ready;
  static int prepare() {  // host-side attributes (eager: never under stream capture)
    if (ready) return HHG_OK;
    auto k = k_elem_fp<BLEND, MODE, FULL, ETAQ, EPI>;
    HHG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
    HHG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ready = true;
    return HHG_OK;
  }
  static int launch(const Mesh* m, const Level& L, const double* eta, double gamma, const double* u, const double* p,
                    double* yu, double* yp, const double* T2, EtaQ eq, cudaStream_t s, ChebEpi ep = ChebEpi{}) {
    HHG_TRY(prepare());
    const int64_t nm = macro_count(m);
    auto go = [&](const int32_t* list, int64_t nb, int det) {
      if (nm * nb == 0) return;
      k_elem_fp<BLEND, MODE, FULL, ETAQ, EPI><<<dim3((unsigned)nb, (unsigned)nm), kBTD, smem, s>>>(
          m->dgeo, L.geo, list, (int)nb, L.n1, 1.0 / L.n1, L.npts1, L.npts2, nm * L.npts2, eta, u, p, yu, yp, gamma, T2,
          eq, det, ep);
      count_launch();
    };
    if (!m->deterministic && !g_no_split) {
      const int64_t ns = L.n_bricks - L.n_dense;
      // fork: the sparse launch on the side stream, concurrent with the dense one (serial when profiling times the
      // dense kernel alone, when one of the two is empty, or when no side stream exists for s yet under capture)
      const Mesh::Side* sd = nullptr;
      if (nm * ns && nm * L.n_dense && !g_elem_mid_event && !g_no_conc) {
        HHG_TRY(elem_side_prepare(m, s));
        auto it = m->side.find(s);
        if (it != m->side.end()) sd = &it->second;
      }
      if (sd) {
        HHG_CUDA(cudaEventRecord(sd->fork, s));
        HHG_CUDA(cudaStreamWaitEvent(sd->s, sd->fork, 0));
      }
      go(L.bricks, L.n_dense, 0);
      if (g_elem_mid_event) {  // profiling: the dense-brick kernel is timed alone
        HHG_CUDA(cudaEventRecord(g_elem_mid_event, s));
        g_elem_mid_event = nullptr;
      }
      if (nm * ns) {
        k_elem_sparse<BLEND, MODE, FULL, ETAQ><<<dim3((unsigned)ns, (unsigned)nm), kBT, 0, sd ? sd->s : s>>>(
            m->dgeo, L.geo, L.bricks + L.n_dense, L.n1, 1.0 / L.n1, L.npts1, L.npts2, nm * L.npts2, eta, u, p, yu, yp,
            gamma, T2, eq);
        count_launch();
      }
      if (sd) {  // join
        HHG_CUDA(cudaEventRecord(sd->join, sd->s));
        HHG_CUDA(cudaStreamWaitEvent(s, sd->join, 0));
      }
    } else if (!m->deterministic) {
      go(L.bricks, L.n_bricks, 0);
    } else {
      for (int c = 0; c < 8; ++c) go(L.bricks_col + L.col_off[c], L.col_off[c + 1] - L.col_off[c], 1);
    }
    HHG_CUDA(cudaGetLastError());
    return HHG_OK;
  }
};
template <bool BLEND, int MODE, bool FULL, bool ETAQ, int EPI>
bool ElemKernel<BLEND, MODE, FULL, ETAQ, EPI>::ready = false;

static bool g_slots_ready = false;
static int ensure_slots() {
  if (g_slots_ready) return HHG_OK;
  const int TV[6][4][3] = {
      {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}}};
  const int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  int slot[6][10], ld[6][10], pslot[6][4], first[6] = {0}, pfirst[6] = {0};
  long long seen2 = 0;
  int seen1 = 0;
  for (int t = 0; t < 6; ++t) {
    int off[10][3];
    for (int v = 0; v < 4; ++v) {
      for (int r = 0; r < 3; ++r) off[v][r] = 2 * TV[t][v][r];
      pslot[t][v] = TV[t][v][0] + 2 * TV[t][v][1] + 4 * TV[t][v][2];
    }
    for (int e = 0; e < 6; ++e)
      for (int r = 0; r < 3; ++r) off[4 + e][r] = TV[t][ep[e][0]][r] + TV[t][ep[e][1]][r];
    for (int a = 0; a < 10; ++a) {
      slot[t][a] = off[a][0] + 3 * off[a][1] + 9 * off[a][2];
      ld[t][a] = ((off[a][1] + 3 * off[a][2]) << 2) | off[a][0];
      if (!((seen2 >> slot[t][a]) & 1)) {
        first[t] |= 1 << a;
        seen2 |= 1LL << slot[t][a];
      }
    }
    for (int v = 0; v < 4; ++v)
      if (!((seen1 >> pslot[t][v]) & 1)) {
        pfirst[t] |= 1 << v;
        seen1 |= 1 << pslot[t][v];
      }
  }
  int items[5][64] = {{0}}, nitems[5] = {0};
  for (int delta = 1; delta <= 4; ++delta)
    for (int cube = 0; cube < 64; ++cube) {
      const int ts = (cube & 3) + ((cube >> 2) & 3) + (cube >> 4);
      const int nt = (ts <= delta - 3) ? 6 : (ts == delta - 2 ? 5 : (ts == delta - 1 ? 1 : 0));
      for (int t = 0; t < nt; ++t) {
        if (nitems[delta] >= 64) return fail(HHG_EINVAL, "sparse brick item table overflow");
        items[delta][nitems[delta]++] = cube | (t << 6);
      }
    }
  int offU[6][10], offP[6][4];
  for (int t = 0; t < 6; ++t) {
    int seen = 0;
    for (int a = 0; a < 10; ++a) {
      const int sl = slot[t][a];  // doubled offset (sl%3, (sl/3)%3, sl/9)
      offU[t][a] = fword(sl % 3, (sl / 3) % 3, sl / 9);
      if (a >= 4) {  // k_elem_fp's round E relies on distinct edge parity classes
        const int par = (sl % 3) % 2 | (((sl / 3) % 3) % 2) << 1 | ((sl / 9) % 2) << 2;
        if ((seen >> par) & 1) return fail(HHG_EINVAL, "edge parity classes collide");
        seen |= 1 << par;
      }
    }
    for (int v = 0; v < 4; ++v) offP[t][v] = TV[t][v][0] + 5 * TV[t][v][1] + 25 * TV[t][v][2];
  }
  HHG_CUDA(cudaMemcpyToSymbol(eOffU, offU, sizeof(offU)));
  int offB[6][10];
  for (int t = 0; t < 6; ++t)
    for (int a = 0; a < 10; ++a) offB[t][a] = 8 * offU[t][a];
  HHG_CUDA(cudaMemcpyToSymbol(eOffB, offB, sizeof(offB)));
  HHG_CUDA(cudaMemcpyToSymbol(eOffP, offP, sizeof(offP)));
  HHG_CUDA(cudaMemcpyToSymbol(eSlot, slot, sizeof(slot)));
  HHG_CUDA(cudaMemcpyToSymbol(eLd, ld, sizeof(ld)));
  HHG_CUDA(cudaMemcpyToSymbol(ePSlot, pslot, sizeof(pslot)));
  HHG_CUDA(cudaMemcpyToSymbol(eFirst, first, sizeof(first)));
  HHG_CUDA(cudaMemcpyToSymbol(ePFirst, pfirst, sizeof(pfirst)));
  HHG_CUDA(cudaMemcpyToSymbol(eItems, items, sizeof(items)));
  HHG_CUDA(cudaMemcpyToSymbol(eNItems, nitems, sizeof(nitems)));
  g_slots_ready = true;
  return HHG_OK;
}

int launch_elem_surf(const Mesh* m, const Level& L, int mode, const double* eta, double a, double r_outer,
                     const double* in, double* out, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;  // a rank without macros (empty partition)
  HHG_TRY(ensure_slots());
  const bool bl = m->blend == HHG_BLEND_SHELL;
  if (a != 1.0 && !bl) return fail(HHG_EINVAL, "w-BFBT surface scaling a != 1 needs a shell-blended mesh");
  if (!(a > 0.0)) return fail(HHG_EINVAL, "w-BFBT surface scaling a must be > 0");
  // a in the gamma slot, the outer radius in eq.r_jump
  const EtaQ eq{0.0, 1.0, r_outer};
#define HHG_SURF(MODE, U, P, YU, YP)                                                                     \
  return bl ? ElemKernel<true, MODE, true, false>::launch(m, L, eta, a, U, P, YU, YP, nullptr, eq, s)    \
            : ElemKernel<false, MODE, true, false>::launch(m, L, eta, a, U, P, YU, YP, nullptr, eq, s);
  switch (mode) {
    case ELEM_KP1: HHG_SURF(ELEM_KP1, nullptr, in, nullptr, out);
    case ELEM_KP1D: HHG_SURF(ELEM_KP1D, nullptr, nullptr, nullptr, out);
    case ELEM_VMASS: HHG_SURF(ELEM_VMASS, in, nullptr, out, nullptr);
    case ELEM_VMASSD: HHG_SURF(ELEM_VMASSD, nullptr, nullptr, out, nullptr);
    default: return fail(HHG_EINVAL, "bad w-BFBT element mode");
  }
#undef HHG_SURF
}

// A (mode ELEM_A) or diag(A) (ELEM_DIAG) with the viscosity evaluated at the quadrature points from the
// P2 temperature T2 (NEXT-2 tier); full form only
int launch_elem_qeta(const Mesh* m, const Level& L, int mode, const double* T2, double lnC, double jump, double r_jump,
                     const double* u, double* yu, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;  // a rank without macros (empty partition)
  HHG_TRY(ensure_slots());
  const EtaQ eq{lnC, jump, r_jump};
  const bool bl = m->blend == HHG_BLEND_SHELL;
  if (mode == ELEM_A)
    return bl ? ElemKernel<true, ELEM_A, true, true>::launch(m, L, nullptr, 0.0, u, nullptr, yu, nullptr, T2, eq, s)
              : ElemKernel<false, ELEM_A, true, true>::launch(m, L, nullptr, 0.0, u, nullptr, yu, nullptr, T2, eq, s);
  if (mode == ELEM_DIAG)
    return bl ? ElemKernel<true, ELEM_DIAG, true, true>::launch(m, L, nullptr, 0.0, u, nullptr, yu, nullptr, T2, eq, s)
              : ElemKernel<false, ELEM_DIAG, true, true>::launch(m, L, nullptr, 0.0, u, nullptr, yu, nullptr, T2, eq, s);
  return fail(HHG_EINVAL, "quadrature-point viscosity: mode must be A or diag");
}

int launch_elem(const Mesh* m, const Level& L, int mode, int form, const double* eta, double gamma,
                const double* u, const double* p, double* yu, double* yp, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;  // a rank without macros (empty partition)
  HHG_TRY(ensure_slots());
  const bool bl = m->blend == HHG_BLEND_SHELL;
  const bool full = form == HHG_VISC_FULL;
  const EtaQ eq{0.0, 1.0, 0.0};
#define HHG_DISPATCH(MODE)                                                                                           \
  return bl ? (full ? ElemKernel<true, MODE, true, false>::launch(m, L, eta, gamma, u, p, yu, yp, nullptr, eq, s)   \
                    : ElemKernel<true, MODE, false, false>::launch(m, L, eta, gamma, u, p, yu, yp, nullptr, eq, s)) \
            : (full ? ElemKernel<false, MODE, true, false>::launch(m, L, eta, gamma, u, p, yu, yp, nullptr, eq, s)  \
                    : ElemKernel<false, MODE, false, false>::launch(m, L, eta, gamma, u, p, yu, yp, nullptr, eq, s));
  switch (mode) {
    case ELEM_A: HHG_DISPATCH(ELEM_A);
    case ELEM_BT: HHG_DISPATCH(ELEM_BT);
    case ELEM_DIV: HHG_DISPATCH(ELEM_DIV);
    case ELEM_A | ELEM_BT | ELEM_DIV: HHG_DISPATCH(ELEM_A | ELEM_BT | ELEM_DIV);
    case ELEM_DIAG: HHG_DISPATCH(ELEM_DIAG);
    case ELEM_MASS: HHG_DISPATCH(ELEM_MASS);
    case ELEM_MASSD: HHG_DISPATCH(ELEM_MASSD);
    case ELEM_LOAD: HHG_DISPATCH(ELEM_LOAD);
    default: return fail(HHG_EINVAL, "bad element mode");
  }
#undef HHG_DISPATCH
}

int launch_elem_epi(const Mesh* m, const Level& L, int kind, const ChebEpi& e, const double* eta, const double* u,
                    double* yu, cudaStream_t s) {
  if (macro_count(m) == 0) return HHG_OK;
  if (m->deterministic || m->nranks != 1) return fail(HHG_EINVAL, "fused epilogue: single rank, non-deterministic only");
  HHG_TRY(ensure_slots());
  const bool bl = m->blend == HHG_BLEND_SHELL;
  const EtaQ eq{0.0, 1.0, 0.0};
#define HHG_EPI(K)                                                                                              \
  return bl ? ElemKernel<true, ELEM_A, true, false, K>::launch(m, L, eta, 0.0, u, nullptr, yu, nullptr, nullptr, eq, s, e) \
            : ElemKernel<false, ELEM_A, true, false, K>::launch(m, L, eta, 0.0, u, nullptr, yu, nullptr, nullptr, eq, s, e);
  switch (kind) {
    case EPI_SUB: HHG_EPI(EPI_SUB);
    case EPI_CHEB0: HHG_EPI(EPI_CHEB0);
    case EPI_CHEBK: HHG_EPI(EPI_CHEBK);
    case EPI_CHEBK_LAST: HHG_EPI(EPI_CHEBK_LAST);
    default: return fail(HHG_EINVAL, "bad fused epilogue");
  }
#undef HHG_EPI
}

// Nodes the fused epilogue updates: footprint-interior points (X, Y, Z in 1..7) of the dense bricks (delta > 4,
// the ones k_elem_fp runs on the per-cube path), strictly inside the macro (i + j + k < n2).  Host-built, once.
int elem_fused_mask(const Mesh* m, const Level& L, uint8_t** mask) {
  const int64_t nm = macro_count(m), ns = nm * L.npts2;
  std::vector<int32_t> br(L.n_bricks);
  if (L.n_bricks) HHG_CUDA(cudaMemcpy(br.data(), L.bricks, L.n_bricks * sizeof(int32_t), cudaMemcpyDeviceToHost));
  std::vector<uint8_t> h(ns, 0), one(L.npts2, 0);
  const int n1 = L.n1, n2 = L.n2;
  for (int32_t bpk : br) {
    const int i0 = bpk & 1023, j0 = (bpk >> 10) & 1023, k0 = bpk >> 20;
    if (n1 - (i0 + j0 + k0) <= 4) continue;  // sparse brick: REDs only
    for (int Z = 1; Z < 8; ++Z)
      for (int Y = 1; Y < 8; ++Y)
        for (int X = 1; X < 8; ++X) {
          const int gx = 2 * i0 + X, gy = 2 * j0 + Y, gz = 2 * k0 + Z;
          if (gx + gy + gz < n2) one[lidx(gx, gy, gz, n2)] = 1;
        }
  }
  for (int64_t mc = 0; mc < nm; ++mc) std::copy(one.begin(), one.end(), h.begin() + mc * L.npts2);
  HHG_CUDA(cudaMalloc(mask, std::max<int64_t>(ns, 1)));
  if (ns) HHG_CUDA(cudaMemcpy(*mask, h.data(), ns, cudaMemcpyHostToDevice));
  return HHG_OK;
}

// Eager one-time set-up of the element kernels (tables in __constant__ memory, kernel attributes,
// occupancy): called from mesh/level construction so that no hot call -- in particular none under
// CUDA-graph capture -- runs a synchronous host API.
int elem_prepare_all() {
  HHG_TRY(ensure_slots());
#define HHG_PREP(B, MODE, F, E) HHG_TRY((ElemKernel<B, MODE, F, E>::prepare()));
#define HHG_PREP4(MODE) HHG_PREP(true, MODE, true, false) HHG_PREP(true, MODE, false, false) \
  HHG_PREP(false, MODE, true, false) HHG_PREP(false, MODE, false, false)
  HHG_PREP4(ELEM_A)
  HHG_PREP4(ELEM_BT)
  HHG_PREP4(ELEM_DIV)
  HHG_PREP4(ELEM_A | ELEM_BT | ELEM_DIV)
  HHG_PREP4(ELEM_DIAG)
  HHG_PREP4(ELEM_MASS)
  HHG_PREP4(ELEM_MASSD)
  HHG_PREP4(ELEM_LOAD)
  HHG_PREP(true, ELEM_KP1, true, false) HHG_PREP(false, ELEM_KP1, true, false)
  HHG_PREP(true, ELEM_KP1D, true, false) HHG_PREP(false, ELEM_KP1D, true, false)
  HHG_PREP(true, ELEM_VMASS, true, false) HHG_PREP(false, ELEM_VMASS, true, false)
  HHG_PREP(true, ELEM_VMASSD, true, false) HHG_PREP(false, ELEM_VMASSD, true, false)
  HHG_PREP(true, ELEM_A, true, true) HHG_PREP(false, ELEM_A, true, true)
#define HHG_PREPE(K) HHG_TRY((ElemKernel<true, ELEM_A, true, false, K>::prepare())); \
  HHG_TRY((ElemKernel<false, ELEM_A, true, false, K>::prepare()));
  HHG_PREPE(EPI_SUB) HHG_PREPE(EPI_CHEB0) HHG_PREPE(EPI_CHEBK) HHG_PREPE(EPI_CHEBK_LAST)
#undef HHG_PREPE
  HHG_PREP(true, ELEM_DIAG, true, true) HHG_PREP(false, ELEM_DIAG, true, true)
#undef HHG_PREP4
#undef HHG_PREP
  return HHG_OK;
}

}  // namespace hhg
