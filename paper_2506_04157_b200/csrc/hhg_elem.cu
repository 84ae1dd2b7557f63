// Element kernel of the hot path (sm_100a, fp64 DFMA pipe -- the operator is not a dense
// contraction, so no tensor cores).
//
// Work decomposition ("brick"): the P1 lattice of a macro (resolution n = 2^L) is cut into
// 4x4x4 blocks of lattice cubes; one CTA of 64 threads owns one block, one thread owns one cube
// and evaluates the (up to) 6 micro tets of that cube (Bey/Freudenthal refinement):
//   type 0 up {000,100,010,001}, 1-4 octahedron around diagonal 010-101, 5 down {011,101,110,111}.
// Per tet: gather 30 velocity dofs (+4 eta, +4 p), evaluate the blending Jacobian at the 4
// quadrature points on the fly, form 2 eta dev(eps(u)), -p I (B^T) and
// -(div u + grad ln rho . u) (B+C), and scatter through the transpose of the barycentric
// gradient map.  Outputs are accumulated in thread-private shared-memory slots (27 P2 nodes x 3
// comps of the cube, + 8 P1 corners): no shared-memory atomics (sm_100a has no native fp64
// ATOMS add).  After one __syncthreads the CTA gathers every node of the block footprint once:
// nodes strictly inside the footprint get a plain store, footprint-border nodes one fp64 RED.
#include "hhg_internal.h"

namespace hhg {

constexpr double EQA = 0.58541019662496845446;  // Q4 (5 + 3 sqrt 5)/20
constexpr double EQB = 0.13819660112501051518;  // Q4 (5 - sqrt 5)/20
constexpr double EQAB = EQA - EQB;
constexpr double EWQ = 1.0 / 24.0;

constexpr int kB = 4;          // cubes per brick edge
constexpr int kBT = 64;        // threads per CTA (one per cube)
constexpr int kFP = 2 * kB + 1;  // P2 footprint points per edge (9)
constexpr int kFP1 = kB + 1;     // P1 footprint points per edge (5)

__constant__ int eTV[6][4][3] = {
    {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
    {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}},
    {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}},
    {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}},
};
// cube-local P2 slot (a + 3b + 9c of the doubled offset) of each tet's 10 local nodes, and
// cube-local P1 slot (a + 2b + 4c) of its 4 vertices; filled from eTV on the host side below.
__constant__ int eSlot[6][10];
__constant__ int ePSlot[6][4];

// 32-bit lattice helpers (N <= 512 keeps (N+1)(N+2)(N+3) < 2^31)
__device__ __forceinline__ int kbase32(int N, int k) {  // first index of plane k
  const int M = N - k;
  return ((N + 1) * (N + 2) * (N + 3) - (M + 1) * (M + 2) * (M + 3)) / 6;
}
__device__ __forceinline__ int rowstart32(int N, int j, int k) {  // index of (0, j, k)
  const int m = N - k;
  return kbase32(N, k) + (j * (2 * m + 3 - j)) / 2;
}

#define EEI(m, j) (((m) == 0) ? (3 + (j)) : (((m) == 1) ? (((j) == 0) ? 4 : 5 + (j)) : (((m) == 2) ? (((j) == 0) ? 5 : ((j) == 1 ? 7 : 9)) : (((j) == 0) ? 6 : ((j) == 1 ? 8 : 9)))))

// One micro tet.  G: [JFinv(9) | qoff(4x3)] of the tet's type; xa: unblended anchor position.
// acc[10][3]: velocity outputs (local P2 order v0..v3, e01..e23); gy[4]: P1 outputs.
template <bool BLEND, int MODE, bool FULL>
__device__ __forceinline__ void tet_body(const double* __restrict__ G, double absdetF, const double (&xa)[3],
                                         const double (&nh)[3], double cK, double gamma, const double (&uu)[10][3],
                                         const double (&et)[4], const double (&pp)[4], double (&acc)[10][3],
                                         double (&gy)[4]) {
  constexpr bool DO_A = (MODE & ELEM_A) != 0;
  constexpr bool DO_BT = (MODE & ELEM_BT) != 0;
  constexpr bool DO_DIV = (MODE & ELEM_DIV) != 0;
  constexpr bool DO_DIAG = (MODE & ELEM_DIAG) != 0;
  constexpr bool NEED_U = DO_A || DO_DIV;
  double JFi[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) JFi[r] = __ldg(G + r);
  const double etaS = EQB * (et[0] + et[1] + et[2] + et[3]);
  const double pS = EQB * (pp[0] + pp[1] + pp[2] + pp[3]);
  // D_m(lambda) = sum_j lambda_j C_mj, C_mm = 3u_m, C_mj = 4u_mj - u_m; at the Q4 point q:
  // D_m(q) = Sb_m + (a-b) C_mq with Sb_m = 4 b sum_{j!=m} u_mj;  grad_xi u = D_k - D_0.
  double Sb[4][3];
  if (NEED_U) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Sb[0][c] = 4.0 * EQB * (uu[4][c] + uu[5][c] + uu[6][c]);
      Sb[1][c] = 4.0 * EQB * (uu[4][c] + uu[7][c] + uu[8][c]);
      Sb[2][c] = 4.0 * EQB * (uu[5][c] + uu[7][c] + uu[9][c]);
      Sb[3][c] = 4.0 * EQB * (uu[6][c] + uu[8][c] + uu[9][c]);
    }
  }
  double Sbar[4][3];
#pragma unroll
  for (int a = 0; a < 10; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[a][c] = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int c = 0; c < 3; ++c) Sbar[m][c] = 0.0;
  double gq[4] = {0, 0, 0, 0}, gsum = 0.0;

#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double xq[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) xq[r] = xa[r] + __ldg(G + 9 + 3 * q + r);
    // blending at x_q: d = x/|x|, alpha = n.d, J_B^-1 = (I - d w^T)/(c alpha), w = n/alpha - d
    double d[3] = {0, 0, 0}, wh[3] = {0, 0, 0}, ca = 1.0;
    if (BLEND || DO_DIV) {
      const double ri = rsqrt(xq[0] * xq[0] + xq[1] * xq[1] + xq[2] * xq[2]);
      d[0] = xq[0] * ri;
      d[1] = xq[1] * ri;
      d[2] = xq[2] * ri;
    }
    if (BLEND) {
      const double alpha = nh[0] * d[0] + nh[1] * d[1] + nh[2] * d[2];
      const double ia = 1.0 / alpha;
      wh[0] = nh[0] * ia - d[0];
      wh[1] = nh[1] * ia - d[1];
      wh[2] = nh[2] * ia - d[2];
      ca = cK * alpha;
    }
    const double etaq = etaS + EQAB * et[q];
    // 2 eta w |det J_F| |det J_B| / (c alpha)^2 = 2 eta w |det J_F| c alpha
    const double sA = 2.0 * etaq * EWQ * absdetF * ca;

    if (DO_DIAG) {
#pragma unroll
      for (int a = 0; a < 10; ++a) {
        double gh[3];
        if (a < 4) {
          const double lam = (a == q) ? EQA : EQB;
          const double f = 4.0 * lam - 1.0;
          gh[0] = (a == 0) ? -f : (a == 1 ? f : 0.0);
          gh[1] = (a == 0) ? -f : (a == 2 ? f : 0.0);
          gh[2] = (a == 0) ? -f : (a == 3 ? f : 0.0);
        } else {
          const int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
          const int i0 = ep[a - 4][0], j0 = ep[a - 4][1];
          const double li = (i0 == q) ? EQA : EQB, lj = (j0 == q) ? EQA : EQB;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double gi = (i0 == 0) ? -1.0 : (i0 == k + 1 ? 1.0 : 0.0);
            const double gj = (j0 == 0) ? -1.0 : (j0 == k + 1 ? 1.0 : 0.0);
            gh[k] = 4.0 * (li * gj + lj * gi);
          }
        }
        double gx[3];
#pragma unroll
        for (int l = 0; l < 3; ++l) gx[l] = gh[0] * JFi[l] + gh[1] * JFi[3 + l] + gh[2] * JFi[6 + l];
        if (BLEND) {
          const double gd = gx[0] * d[0] + gx[1] * d[1] + gx[2] * d[2];
          gx[0] -= gd * wh[0];
          gx[1] -= gd * wh[1];
          gx[2] -= gd * wh[2];
        }
        const double n2g = gx[0] * gx[0] + gx[1] * gx[1] + gx[2] * gx[2];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double gc2 = gx[c] * gx[c];
          acc[a][c] += sA * (FULL ? (0.5 * (n2g + gc2) - gc2 * (1.0 / 3.0)) : 0.5 * (n2g + gc2));
        }
      }
      continue;
    }

    double H[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (NEED_U) {
      double gh[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double D[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double Cmq = (m == q) ? 3.0 * uu[m][c] : 4.0 * uu[EEI(m, q)][c] - uu[m][c];
          D[m] = Sb[m][c] + EQAB * Cmq;
        }
        gh[c][0] = D[1] - D[0];
        gh[c][1] = D[2] - D[0];
        gh[c][2] = D[3] - D[0];
      }
      // G = gh J_F^-1 ;  H = G - (G d) w^T   (grad_x u = H / (c alpha))
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int l = 0; l < 3; ++l) H[c][l] = gh[c][0] * JFi[l] + gh[c][1] * JFi[3 + l] + gh[c][2] * JFi[6 + l];
        if (BLEND) {
          const double gd = H[c][0] * d[0] + H[c][1] * d[1] + H[c][2] * d[2];
          H[c][0] -= gd * wh[0];
          H[c][1] -= gd * wh[1];
          H[c][2] -= gd * wh[2];
        }
      }
    }
    if (DO_DIV) {
      // g_q = -W (div u + grad ln rho . u),  div u = tr(H)/(c alpha),  grad ln rho = -gamma d
      double uq[3];
      const double phv = EQB * (2.0 * EQB - 1.0), phq = EQA * (2.0 * EQA - 1.0);
      const double peq = 4.0 * EQA * EQB, pen = 4.0 * EQB * EQB;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) s += ((a == q) ? phq : phv) * uu[a][c];
        const int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
        for (int e = 0; e < 6; ++e) s += ((ep[e][0] == q || ep[e][1] == q) ? peq : pen) * uu[4 + e][c];
        uq[c] = s;
      }
      const double W = EWQ * absdetF * ca * ca * ca;
      const double div = (H[0][0] + H[1][1] + H[2][2]) / ca;
      const double gg = -W * (div - gamma * (d[0] * uq[0] + d[1] * uq[1] + d[2] * uq[2]));
      gq[q] = gg;
      gsum += gg;
    }
    if (DO_A || DO_BT) {
      double S[3][3];
      if (DO_A) {
        const double tr3 = (H[0][0] + H[1][1] + H[2][2]) * (1.0 / 3.0);
        if (FULL) {
          S[0][0] = sA * (H[0][0] - tr3);
          S[1][1] = sA * (H[1][1] - tr3);
          S[2][2] = sA * (H[2][2] - tr3);
        } else {
          S[0][0] = sA * H[0][0];
          S[1][1] = sA * H[1][1];
          S[2][2] = sA * H[2][2];
        }
        S[0][1] = S[1][0] = 0.5 * sA * (H[0][1] + H[1][0]);
        S[0][2] = S[2][0] = 0.5 * sA * (H[0][2] + H[2][0]);
        S[1][2] = S[2][1] = 0.5 * sA * (H[1][2] + H[2][1]);
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int l = 0; l < 3; ++l) S[c][l] = 0.0;
      }
      if (DO_BT) {
        // B^T p: isotropic stress -p_q W I, scaled by 1/(c alpha)
        const double pq = pS + EQAB * pp[q];
        const double wb = EWQ * absdetF * ca * ca * pq;
        S[0][0] -= wb;
        S[1][1] -= wb;
        S[2][2] -= wb;
      }
      // M = S - (S w) d^T ; R = M J_F^-T
      double R[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double Mr[3] = {S[c][0], S[c][1], S[c][2]};
        if (BLEND) {
          const double sw = S[c][0] * wh[0] + S[c][1] * wh[1] + S[c][2] * wh[2];
          Mr[0] -= sw * d[0];
          Mr[1] -= sw * d[1];
          Mr[2] -= sw * d[2];
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) R[c][k] = Mr[0] * JFi[3 * k] + Mr[1] * JFi[3 * k + 1] + Mr[2] * JFi[3 * k + 2];
      }
      // transpose of the barycentric gradient map
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double Db[4];
        Db[1] = R[c][0];
        Db[2] = R[c][1];
        Db[3] = R[c][2];
        Db[0] = -(Db[1] + Db[2] + Db[3]);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          Sbar[m][c] += Db[m];
          if (m == q) {
            acc[m][c] += 3.0 * EQAB * Db[m];
          } else {
            acc[EEI(m, q)][c] += 4.0 * EQAB * Db[m];
            acc[m][c] -= EQAB * Db[m];
          }
        }
      }
    }
  }
  if (DO_A || DO_BT) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      acc[4][c] += 4.0 * EQB * (Sbar[0][c] + Sbar[1][c]);
      acc[5][c] += 4.0 * EQB * (Sbar[0][c] + Sbar[2][c]);
      acc[6][c] += 4.0 * EQB * (Sbar[0][c] + Sbar[3][c]);
      acc[7][c] += 4.0 * EQB * (Sbar[1][c] + Sbar[2][c]);
      acc[8][c] += 4.0 * EQB * (Sbar[1][c] + Sbar[3][c]);
      acc[9][c] += 4.0 * EQB * (Sbar[2][c] + Sbar[3][c]);
    }
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) gy[v] = EQB * gsum + EQAB * gq[v];
}

template <bool BLEND, int MODE, bool FULL>
#ifndef HHG_ELEM_MINB
#define HHG_ELEM_MINB 4
#endif
__global__ void __launch_bounds__(kBT, HHG_ELEM_MINB) k_elem_brick(const MacroGeo* __restrict__ mgeo, const double* __restrict__ lgeo,
                                                    const int32_t* __restrict__ bricks, int n1, int64_t npts1,
                                                    int64_t npts2, int64_t cstride, const double* __restrict__ eta,
                                                    const double* __restrict__ u, const double* __restrict__ p,
                                                    double* __restrict__ yu, double* __restrict__ yp, double gamma) {
  constexpr bool DO_DIV = (MODE & ELEM_DIV) != 0;
  constexpr bool HAS_U_OUT = (MODE & (ELEM_A | ELEM_BT | ELEM_DIAG)) != 0;
  constexpr bool NEED_U = (MODE & (ELEM_A | ELEM_DIV)) != 0;
  constexpr bool NEED_ETA = (MODE & (ELEM_A | ELEM_DIAG)) != 0;
  constexpr bool NEED_P = (MODE & ELEM_BT) != 0;
  constexpr int NSU = HAS_U_OUT ? 81 : 0;
  constexpr int NS = NSU + (DO_DIV ? 8 : 0);
  extern __shared__ double sm[];  // [NS][kBT]

  const int mac = blockIdx.y;
  const int32_t bpk = __ldg(bricks + blockIdx.x);
  const int i0 = bpk & 1023, j0 = (bpk >> 10) & 1023, k0 = bpk >> 20;
  const int tid = threadIdx.x;
  const int ti = tid & 3, tj = (tid >> 2) & 3, tk = tid >> 4;
  const int ai = i0 + ti, aj = j0 + tj, ak = k0 + tk;
  const int s = ai + aj + ak;
  const int n2 = 2 * n1;
#pragma unroll 1
  for (int sl = 0; sl < NS; ++sl) sm[sl * kBT + tid] = 0.0;

  if (s <= n1 - 1) {
    const MacroGeo& g = mgeo[mac];
    double nh[3] = {0, 0, 0}, cK = 1.0;
    if (BLEND) {
      nh[0] = g.nhat[0];
      nh[1] = g.nhat[1];
      nh[2] = g.nhat[2];
      cK = g.cK;
    }
    const double fa = (double)ai / n1, fb = (double)aj / n1, fc = (double)ak / n1;
    double xa[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) xa[r] = g.X0[r] + g.Jm[3 * r] * fa + g.Jm[3 * r + 1] * fb + g.Jm[3 * r + 2] * fc;
    const double* Gm = lgeo + (int64_t)mac * kLevelGeo;
    const double absdetF = __ldg(Gm + 6 * kTypeGeo);
    // per-cube row starts: P2 rows (2aj+b, 2ak+c), b,c in 0..2 ; P1 rows (aj+b, ak+c), b,c in 0..1
    // (kept in per-thread shared-memory slots: the tet loop indexes them with runtime values)
    int* rs2 = reinterpret_cast<int*>(sm + NS * kBT) + tid;  // stride kBT
    int* rs1 = rs2 + 9 * kBT;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int b = 0; b < 3; ++b) rs2[(b + 3 * c) * kBT] = rowstart32(n2, 2 * aj + b, 2 * ak + c) + 2 * ai;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int b = 0; b < 2; ++b) rs1[(b + 2 * c) * kBT] = rowstart32(n1, aj + b, ak + c) + ai;
    const double* um = u + (int64_t)mac * npts2;
    const double* em = eta ? eta + (int64_t)mac * npts1 : nullptr;
    const double* pm = p ? p + (int64_t)mac * npts1 : nullptr;
    const int ntypes = (s <= n1 - 3) ? 6 : ((s <= n1 - 2) ? 5 : 1);
#pragma unroll 1
    for (int t = 0; t < ntypes; ++t) {  // s <= n-1: up only; s <= n-2: + octahedron (1-4); s <= n-3: + down
      double uu[10][3];
      if (NEED_U) {
#pragma unroll
        for (int a = 0; a < 10; ++a) {
          const int sl = eSlot[t][a];  // doubled offset (sl%3, (sl/3)%3, sl/9) inside the cube
          const int ix = rs2[(sl / 3) * kBT] + sl % 3;
#pragma unroll
          for (int c = 0; c < 3; ++c) uu[a][c] = __ldg(um + c * cstride + ix);
        }
      }
      double et[4] = {1.0, 1.0, 1.0, 1.0}, pp[4] = {0, 0, 0, 0};
      if ((NEED_ETA && eta != nullptr) || NEED_P) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int ps = ePSlot[t][v];  // (ps&1, (ps>>1)&1, ps>>2)
          const int ix = rs1[(ps >> 1) * kBT] + (ps & 1);
          if (NEED_ETA && eta != nullptr) et[v] = __ldg(em + ix);
          if (NEED_P) pp[v] = __ldg(pm + ix);
        }
      }
      double acc[10][3], gy[4];
      tet_body<BLEND, MODE, FULL>(Gm + t * kTypeGeo, absdetF, xa, nh, cK, gamma, uu, et, pp, acc, gy);
      if (HAS_U_OUT) {
#pragma unroll
        for (int a = 0; a < 10; ++a) {
          const int sl = eSlot[t][a];
#pragma unroll
          for (int c = 0; c < 3; ++c) sm[(3 * sl + c) * kBT + tid] += acc[a][c];
        }
      }
      if (DO_DIV) {
#pragma unroll
        for (int v = 0; v < 4; ++v) sm[(NSU + ePSlot[t][v]) * kBT + tid] += gy[v];
      }
    }
  }
  __syncthreads();

  // gather the brick footprint: each node once (sum over the <= 8 cubes of the brick containing it)
  if (HAS_U_OUT) {
    const int64_t mbase2 = (int64_t)mac * npts2;
#pragma unroll 1
    for (int pt = tid; pt < kFP * kFP * kFP; pt += kBT) {
      const int px = pt % kFP, py = (pt / kFP) % kFP, pz = pt / (kFP * kFP);
      const int gx = 2 * i0 + px, gy_ = 2 * j0 + py, gz = 2 * k0 + pz;
      if (gx + gy_ + gz > n2) continue;
      const int lx0 = (px & 1) ? (px >> 1) : (px >> 1) - 1, lx1 = min(px >> 1, kB - 1);
      const int ly0 = (py & 1) ? (py >> 1) : (py >> 1) - 1, ly1 = min(py >> 1, kB - 1);
      const int lz0 = (pz & 1) ? (pz >> 1) : (pz >> 1) - 1, lz1 = min(pz >> 1, kB - 1);
      double v[3] = {0.0, 0.0, 0.0};
      for (int lz = max(lz0, 0); lz <= lz1; ++lz)
        for (int ly = max(ly0, 0); ly <= ly1; ++ly)
          for (int lx = max(lx0, 0); lx <= lx1; ++lx) {
            const int sl = (px - 2 * lx) + 3 * (py - 2 * ly) + 9 * (pz - 2 * lz);
            const int cube = lx + kB * ly + kB * kB * lz;
#pragma unroll
            for (int c = 0; c < 3; ++c) v[c] += sm[(3 * sl + c) * kBT + cube];
          }
      const int64_t idx = mbase2 + rowstart32(n2, gy_, gz) + gx;
      const bool border = px == 0 || py == 0 || pz == 0 || px == kFP - 1 || py == kFP - 1 || pz == kFP - 1;
      if (border) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (v[c] != 0.0) atomicAdd(yu + c * cstride + idx, v[c]);
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) yu[c * cstride + idx] = v[c];
      }
    }
  }
  if (DO_DIV) {
    const int64_t mbase1 = (int64_t)mac * npts1;
#pragma unroll 1
    for (int pt = tid; pt < kFP1 * kFP1 * kFP1; pt += kBT) {
      const int px = pt % kFP1, py = (pt / kFP1) % kFP1, pz = pt / (kFP1 * kFP1);
      const int gx = i0 + px, gy_ = j0 + py, gz = k0 + pz;
      if (gx + gy_ + gz > n1) continue;
      double v = 0.0;
      for (int lz = max(pz - 1, 0); lz <= min(pz, kB - 1); ++lz)
        for (int ly = max(py - 1, 0); ly <= min(py, kB - 1); ++ly)
          for (int lx = max(px - 1, 0); lx <= min(px, kB - 1); ++lx) {
            const int sl = (px - lx) + 2 * (py - ly) + 4 * (pz - lz);
            v += sm[(NSU + sl) * kBT + lx + kB * ly + kB * kB * lz];
          }
      const int64_t idx = mbase1 + rowstart32(n1, gy_, gz) + gx;
      const bool border = px == 0 || py == 0 || pz == 0 || px == kFP1 - 1 || py == kFP1 - 1 || pz == kFP1 - 1;
      if (border) {
        if (v != 0.0) atomicAdd(yp + idx, v);
      } else {
        yp[idx] = v;
      }
    }
  }
}

static bool g_slots_ready = false;
static int ensure_slots() {
  if (g_slots_ready) return HHG_OK;
  const int TV[6][4][3] = {
      {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}}};
  const int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  int slot[6][10], pslot[6][4];
  for (int t = 0; t < 6; ++t) {
    for (int v = 0; v < 4; ++v) {
      slot[t][v] = 2 * TV[t][v][0] + 3 * 2 * TV[t][v][1] + 9 * 2 * TV[t][v][2];
      pslot[t][v] = TV[t][v][0] + 2 * TV[t][v][1] + 4 * TV[t][v][2];
    }
    for (int e = 0; e < 6; ++e) {
      const int a = ep[e][0], b = ep[e][1];
      slot[t][4 + e] = (TV[t][a][0] + TV[t][b][0]) + 3 * (TV[t][a][1] + TV[t][b][1]) + 9 * (TV[t][a][2] + TV[t][b][2]);
    }
  }
  HHG_CUDA(cudaMemcpyToSymbol(eSlot, slot, sizeof(slot)));
  HHG_CUDA(cudaMemcpyToSymbol(ePSlot, pslot, sizeof(pslot)));
  g_slots_ready = true;
  return HHG_OK;
}

template <bool BLEND, int MODE, bool FULL>
static void elem_launch(const Mesh* m, const Level& L, const double* eta, double gamma, const double* u,
                        const double* p, double* yu, double* yp, cudaStream_t s) {
  const int64_t nm = macro_count(m);
  constexpr int NS = ((MODE & (ELEM_A | ELEM_BT | ELEM_DIAG)) ? 81 : 0) + ((MODE & ELEM_DIV) ? 8 : 0);
  dim3 grid((unsigned)L.n_bricks, (unsigned)nm);
  k_elem_brick<BLEND, MODE, FULL><<<grid, kBT, NS * kBT * sizeof(double) + 13 * kBT * sizeof(int), s>>>(
      m->dgeo, L.geo, L.bricks, L.n1, L.npts1, L.npts2, nm * L.npts2, eta, u, p, yu, yp, gamma);
}

int launch_elem(const Mesh* m, const Level& L, int mode, int form, const double* eta, double gamma,
                const double* u, const double* p, double* yu, double* yp, cudaStream_t s) {
  HHG_TRY(ensure_slots());
  const bool bl = m->blend == HHG_BLEND_SHELL;
  const bool full = form == HHG_VISC_FULL;
#define HHG_DISPATCH(MODE)                                                            \
  if (bl) {                                                                           \
    if (full) elem_launch<true, MODE, true>(m, L, eta, gamma, u, p, yu, yp, s);       \
    else elem_launch<true, MODE, false>(m, L, eta, gamma, u, p, yu, yp, s);           \
  } else {                                                                            \
    if (full) elem_launch<false, MODE, true>(m, L, eta, gamma, u, p, yu, yp, s);      \
    else elem_launch<false, MODE, false>(m, L, eta, gamma, u, p, yu, yp, s);          \
  }
  switch (mode) {
    case ELEM_A: HHG_DISPATCH(ELEM_A); break;
    case ELEM_BT: HHG_DISPATCH(ELEM_BT); break;
    case ELEM_DIV: HHG_DISPATCH(ELEM_DIV); break;
    case ELEM_A | ELEM_BT | ELEM_DIV: HHG_DISPATCH(ELEM_A | ELEM_BT | ELEM_DIV); break;
    case ELEM_DIAG: HHG_DISPATCH(ELEM_DIAG); break;
    default: return fail(HHG_EINVAL, "bad element mode");
  }
#undef HHG_DISPATCH
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

}  // namespace hhg
