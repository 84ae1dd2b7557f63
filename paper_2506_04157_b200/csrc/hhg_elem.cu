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

namespace hhg {

constexpr double EQA = 0.58541019662496845446;  // Q4 (5 + 3 sqrt 5)/20
constexpr double EQB = 0.13819660112501051518;  // Q4 (5 - sqrt 5)/20
constexpr double EQAB = EQA - EQB;              // 1/sqrt 5
constexpr double EWQ = 1.0 / 24.0;              // Q4 weight (reference volume 1/6, 4 points)
constexpr double C_SB = 1.2360679774997896964;  // 4b/(a-b) = sqrt5 - 1
constexpr double F_R = 4.0 * EQAB;              // prescale of R (folds 4(a-b) of the scatter)
constexpr double C_V = -0.25;                   // (4b-1)/F_R
constexpr double C_E = 0.30901699437494742410;  // 4b/F_R = (sqrt5-1)/4

constexpr int kBT = 64;  // threads per CTA; one CTA per brick of 4x4x4 lattice cubes

// 32-bit lattice helpers (N <= 512 keeps (N+1)(N+2)(N+3) < 2^31)
__device__ __forceinline__ int kbase32(int N, int k) {  // first index of plane k
  const int M = N - k;
  return ((N + 1) * (N + 2) * (N + 3) - (M + 1) * (M + 2) * (M + 3)) / 6;
}
__device__ __forceinline__ int rowstart32(int N, int j, int k) {  // index of (0, j, k)
  const int m = N - k;
  return kbase32(N, k) + (j * (2 * m + 3 - j)) / 2;
}

// local edge index of edge (m, j), m != j (edges 01,02,03,12,13,23 -> 4..9)
__host__ __device__ constexpr int EEI(int m, int j) {
  return (m + j == 1) ? 4 : (m + j == 2) ? 5 : (m * j == 0) ? 6 : (m + j == 3) ? 7 : (m + j == 4) ? 8 : 9;
}

// fp64 reciprocal / reciprocal square root: MUFU seed (rcp/rsqrt.approx.ftz.f64) + Newton.
// Arguments are positive normal numbers here (|x|^2 >= 0.3, n.x >= 0.5 on the shell).
__device__ __forceinline__ double rcp_nr(double t) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(t));
  double e = fma(-t, r, 1.0);
  r = fma(r, e, r);
  e = fma(-t, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double s) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double hs = 0.5 * s;
  y = y * fma(-hs * y, y, 1.5);
  y = y * fma(-hs * y, y, 1.5);
  return y;
}

// Element outputs of one micro tet.  G: [JFinv(9) | qoff(4x3)] of the tet's type;
// wdet = w |det J_F| of the level; xa: unblended anchor position.
// acc[10][3]: velocity outputs (v0..v3, e01..e23); gy[4]: P1 outputs.
// Quadrature-point viscosity tier (NEXT-2): eta_q = exp(lnC (1/2 - T_q)) * (jump if
// r_q < r_jump else 1) with T_q the P2 interpolant of the nodal temperature (R22).
struct EtaQ {
  double lnC, jump, r_jump;
};
struct NoT {
  __device__ __forceinline__ double operator()(int) const { return 0.0; }
};

template <bool BLEND, int MODE, bool FULL, class UA, bool ETAQ = false, class TA = NoT>
__device__ __forceinline__ void tet_body(const double* G, double wdet, const double (&xa)[3],
                                         const double (&nh)[3], double cK, double gamma, const UA& uu,
                                         const double (&et)[4], const double (&pp)[4], double (&acc)[10][3],
                                         double (&gy)[4], const TA& tt = TA{}, EtaQ eq = EtaQ{0.0, 1.0, 0.0}) {
  constexpr bool DO_A = (MODE & ELEM_A) != 0;
  constexpr bool DO_BT = (MODE & ELEM_BT) != 0;
  constexpr bool DO_DIV = (MODE & ELEM_DIV) != 0;
  constexpr bool DO_DIAG = (MODE & ELEM_DIAG) != 0;
  constexpr bool NEED_U = DO_A || DO_DIV;
  constexpr bool SCATTER = DO_A || DO_BT;

  const double etaS = EQB * (et[0] + et[1] + et[2] + et[3]);
  const double pS = EQB * (pp[0] + pp[1] + pp[2] + pp[3]);
  // per-macro constant factors of the point weights
  const double cwA = (DO_DIAG ? 2.0 : 2.0 * F_R * EQAB) * wdet * cK;  // x eta_q alpha
  const double cwB = F_R * wdet * cK * cK;                            // x alpha^2 p_q
  const double cwD = wdet * cK * cK;                                  // x alpha^2 (div rows)

  // Delta_k = Dt_k - Dt_0 (k = 1..3), Dt_m = C_SB sum_{j != m} u_mj - u_m
  double Dl[3][3];
  if (NEED_U) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double d0 = fma(C_SB, uu(4, c) + uu(5, c) + uu(6, c), -uu(0, c));
      const double d1 = fma(C_SB, uu(4, c) + uu(7, c) + uu(8, c), -uu(1, c));
      const double d2 = fma(C_SB, uu(5, c) + uu(7, c) + uu(9, c), -uu(2, c));
      const double d3 = fma(C_SB, uu(6, c) + uu(8, c) + uu(9, c), -uu(3, c));
      Dl[0][c] = d1 - d0;
      Dl[1][c] = d2 - d0;
      Dl[2][c] = d3 - d0;
    }
  }
  // u at the quadrature points (div rows): u_q = B0 + (phq-phv) u_q + (peq-pen) sum_{e ∋ q} u_e
  constexpr double phv = EQB * (2.0 * EQB - 1.0), phq = EQA * (2.0 * EQA - 1.0);
  constexpr double peq = 4.0 * EQA * EQB, pen = 4.0 * EQB * EQB;
  double B0[3] = {0, 0, 0};
  if (DO_DIV) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      B0[c] = phv * (uu(0, c) + uu(1, c) + uu(2, c) + uu(3, c)) +
              pen * (uu(4, c) + uu(5, c) + uu(6, c) + uu(7, c) + uu(8, c) + uu(9, c));
  }
  double Sbar[4][3];
  double gq[4] = {0, 0, 0, 0}, gsum = 0.0;
  if (DO_DIAG) {
#pragma unroll
    for (int a = 0; a < 10; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[a][c] = 0.0;
  }

  // ---- geometry of the 4 quadrature points first, written point-parallel (4 independent
  // chains through the rsqrt/rcp Newton iterations): K_q = JFi - (JFi x_q) z_q^T,
  // z_q = n/t_q - x_q/s_q, alpha_q = t_q/sqrt(s_q)  (rank-one J_B^-1)
  double JFi[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) JFi[r] = G[r];
  double Kq[4][9], al[4] = {1.0, 1.0, 1.0, 1.0}, dq[4][3], etv[4] = {1.0, 1.0, 1.0, 1.0};
  double sfac = 1.0;  // w-BFBT modes: a on D_eta (gamma carries a, eq.r_jump the outer radius)
  {
    double xq[4][3], sq[4], yq[4], tq[4], rq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int r = 0; r < 3; ++r) xq[q][r] = xa[r] + G[9 + 3 * q + r];
    if (ETAQ) {
      constexpr double phv = EQB * (2.0 * EQB - 1.0), phq = EQA * (2.0 * EQA - 1.0);
      constexpr double peq = 4.0 * EQA * EQB, pen = 4.0 * EQB * EQB;
      double tv[10];
#pragma unroll
      for (int a = 0; a < 10; ++a) tv[a] = tt(a);
      const double sv = phv * (tv[0] + tv[1] + tv[2] + tv[3]) + pen * (tv[4] + tv[5] + tv[6] + tv[7] + tv[8] + tv[9]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double es = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (m != q) es += tv[EEI(m, q)];
        const double Tq = fma(peq - pen, es, fma(phq - phv, tv[q], sv));
        const double s2 = fma(xq[q][0], xq[q][0], fma(xq[q][1], xq[q][1], xq[q][2] * xq[q][2]));
        // radius of the blended point: |B(x)| = c (n.x)
        const double rr = BLEND ? cK * fma(nh[0], xq[q][0], fma(nh[1], xq[q][1], nh[2] * xq[q][2])) : sqrt(s2);
        etv[q] = exp(eq.lnC * (0.5 - Tq)) * (rr < eq.r_jump ? eq.jump : 1.0);
      }
    }
    if (BLEND || DO_DIV) {
#pragma unroll
      for (int q = 0; q < 4; ++q) sq[q] = fma(xq[q][0], xq[q][0], fma(xq[q][1], xq[q][1], xq[q][2] * xq[q][2]));
#pragma unroll
      for (int q = 0; q < 4; ++q) yq[q] = rsqrt_nr(sq[q]);
    }
    if (DO_DIV) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int r = 0; r < 3; ++r) dq[q][r] = xq[q][r] * yq[q];
    }
    if (BLEND) {
#pragma unroll
      for (int q = 0; q < 4; ++q) tq[q] = fma(nh[0], xq[q][0], fma(nh[1], xq[q][1], nh[2] * xq[q][2]));
#pragma unroll
      for (int q = 0; q < 4; ++q) rq[q] = rcp_nr(tq[q]);
      if ((MODE & ELEM_SURF) && gamma != 1.0) {
        // D_eta: a vertex on the outer sphere.  Vertex m from its quadrature point,
        // x_q(m) = EQAB x_m + EQB sum_v x_v, and the blended radius |B(x)| = c (n.x) is linear in x.
        const double ts = EQB * (tq[0] + tq[1] + tq[2] + tq[3]);
        const double tmax = fmax(fmax(tq[0], tq[1]), fmax(tq[2], tq[3]));
        if (cK * (tmax - ts) * (1.0 / EQAB) >= eq.r_jump * (1.0 - 1e-9)) sfac = gamma;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        al[q] = tq[q] * yq[q];
        const double y2 = yq[q] * yq[q];
        double z[3], v[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) z[r] = fma(rq[q], nh[r], -xq[q][r] * y2);
#pragma unroll
        for (int k = 0; k < 3; ++k)
          v[k] = fma(JFi[3 * k], xq[q][0], fma(JFi[3 * k + 1], xq[q][1], JFi[3 * k + 2] * xq[q][2]));
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int l = 0; l < 3; ++l) Kq[q][3 * k + l] = fma(-v[k], z[l], JFi[3 * k + l]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int r = 0; r < 9; ++r) Kq[q][r] = JFi[r];
    }
  }

  if (MODE & ELEM_LOAD) {
    // buoyancy load (P:282 with rho' = -alpha (T - 1/2), alpha = 1, g = -x/|x|; R21):
    // f_a,c = sum_q w |det J_F| |det J_B| (T_q - 1/2) (x_q/|x_q|)_c phi_a(q), T P1-interpolated (pp)
#pragma unroll
    for (int a = 0; a < 10; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[a][c] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double xq[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) xq[r] = xa[r] + G[9 + 3 * q + r];
      const double ri = rsqrt_nr(fma(xq[0], xq[0], fma(xq[1], xq[1], xq[2] * xq[2])));
      const double cq = cK * al[q];
      const double sq = wdet * cq * cq * cq * (fma(EQAB, pp[q], pS) - 0.5) * ri;
      constexpr double phv = EQB * (2.0 * EQB - 1.0), phq = EQA * (2.0 * EQA - 1.0);
      constexpr double peq = 4.0 * EQA * EQB, pen = 4.0 * EQB * EQB;
#pragma unroll
      for (int a = 0; a < 10; ++a) {
        double phi;
        if (a < 4) phi = (a == q) ? phq : phv;
        else {
          constexpr int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
          phi = (ep[a - 4][0] == q || ep[a - 4][1] == q) ? peq : pen;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[a][c] = fma(sq * phi, xq[c], acc[a][c]);
      }
    }
    return;
  }
  if (MODE & (ELEM_KP1 | ELEM_KP1D)) {
    // K_{1/sqrt(eta_a)} (w-BFBT Poisson replacement of B M^-1 B^T):
    // K_vw = sum_q w |det J| omega_q grad lam_v . grad lam_w,  omega = 1/sqrt(eta_a),
    // grad lam_{k+1} = row k of K_q / (c alpha_q)  =>  weight w |det J_F| c alpha_q omega_q
#pragma unroll
    for (int v = 0; v < 4; ++v) gy[v] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double* K = Kq[q];
      const double Wq = wdet * cK * al[q] / (sfac * sqrt(fma(EQAB, et[q], etaS)));
      const double R0[3] = {K[0], K[1], K[2]}, R1[3] = {K[3], K[4], K[5]}, R2[3] = {K[6], K[7], K[8]};
      if (MODE & ELEM_KP1) {
        double G[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) G[r] = (pp[1] - pp[0]) * R0[r] + (pp[2] - pp[0]) * R1[r] + (pp[3] - pp[0]) * R2[r];
        const double d1 = R0[0] * G[0] + R0[1] * G[1] + R0[2] * G[2];
        const double d2 = R1[0] * G[0] + R1[1] * G[1] + R1[2] * G[2];
        const double d3 = R2[0] * G[0] + R2[1] * G[1] + R2[2] * G[2];
        gy[1] += Wq * d1;
        gy[2] += Wq * d2;
        gy[3] += Wq * d3;
        gy[0] -= Wq * (d1 + d2 + d3);
      } else {
        double S0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double t0 = R0[r] + R1[r] + R2[r];
          S0 += t0 * t0;
          s1 += R0[r] * R0[r];
          s2 += R1[r] * R1[r];
          s3 += R2[r] * R2[r];
        }
        gy[0] += Wq * S0;
        gy[1] += Wq * s1;
        gy[2] += Wq * s2;
        gy[3] += Wq * s3;
      }
    }
    return;
  }
  if (MODE & (ELEM_VMASS | ELEM_VMASSD)) {
    // vector mass M_{sqrt(eta_a)}: y_(a,c) = sum_q w |det J| sqrt(eta_a,q) phi_a(q) u_c(q)
    constexpr double phv = EQB * (2.0 * EQB - 1.0), phq = EQA * (2.0 * EQA - 1.0);
    constexpr double peq = 4.0 * EQA * EQB, pen = 4.0 * EQB * EQB;
    constexpr int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
    for (int a = 0; a < 10; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[a][c] = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double cq = cK * al[q];
      const double Wq = wdet * cq * cq * cq * sfac * sqrt(fma(EQAB, et[q], etaS));
      double phi[10];
#pragma unroll
      for (int a = 0; a < 10; ++a)
        phi[a] = a < 4 ? ((a == q) ? phq : phv) : ((ep[a - 4][0] == q || ep[a - 4][1] == q) ? peq : pen);
      if (MODE & ELEM_VMASS) {
        double uq[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < 10; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) uq[c] = fma(phi[a], uu(a, c), uq[c]);
#pragma unroll
        for (int a = 0; a < 10; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[a][c] = fma(Wq * phi[a], uq[c], acc[a][c]);
      } else {
#pragma unroll
        for (int a = 0; a < 10; ++a) {
          const double d = Wq * phi[a] * phi[a];
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[a][c] += d;
        }
      }
    }
    return;
  }
  if (MODE & (ELEM_MASS | ELEM_MASSD)) {
    // pressure mass weighted by 1/eta (Schur approximation M_{1/eta}, eq:schurMass P:457-461):
    // M_vw = sum_q w |det J_F| |det J_B| / eta_q  lambda_v(q) lambda_w(q),  |det J_B| = (c alpha)^3
    double gs = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double cq = cK * al[q];
      const double Wq = wdet * cq * cq * cq / fma(EQAB, et[q], etaS);
      if (MODE & ELEM_MASS) {
        gq[q] = Wq * fma(EQAB, pp[q], pS);
        gs += gq[q];
      } else {
        gq[q] = Wq;
        gs += Wq;
      }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v)
      gy[v] = (MODE & ELEM_MASS) ? fma(EQB, gs, EQAB * gq[v]) : fma(EQB * EQB, gs, (EQA * EQA - EQB * EQB) * gq[v]);
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double* K = Kq[q];
    const double alpha = al[q];
    const double* d = dq[q];
    const double etaq = ETAQ ? etv[q] : fma(EQAB, et[q], etaS);

    if (DO_DIAG) {
      // diag(A): sum_q 2 eta w|det J| [eps(phi_a e_c) : eps(phi_a e_c) - 1/3 (div)^2]
      const double sA = cwA * etaq * alpha;
#pragma unroll
      for (int a = 0; a < 10; ++a) {
        double gh[3];
        if (a < 4) {
          const double f = 4.0 * ((a == q) ? EQA : EQB) - 1.0;
          gh[0] = (a == 0) ? -f : (a == 1 ? f : 0.0);
          gh[1] = (a == 0) ? -f : (a == 2 ? f : 0.0);
          gh[2] = (a == 0) ? -f : (a == 3 ? f : 0.0);
        } else {
          constexpr int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
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
        for (int l = 0; l < 3; ++l) gx[l] = gh[0] * K[l] + gh[1] * K[3 + l] + gh[2] * K[6 + l];
        const double n2g = gx[0] * gx[0] + gx[1] * gx[1] + gx[2] * gx[2];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double gc2 = gx[c] * gx[c];
          acc[a][c] += sA * (FULL ? (0.5 * (n2g + gc2) - gc2 * (1.0 / 3.0)) : 0.5 * (n2g + gc2));
        }
      }
      continue;
    }

    // Ht = grad_ref(u)/(a-b) . K   (physical gradient = (a-b) Ht / (c alpha))
    double H[3][3];
    if (NEED_U) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double x0 = (q == 0) ? uu(0, c) : uu(EEI(0, q), c);
        double gh[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double xk = (q == k + 1) ? uu(k + 1, c) : uu(EEI(k + 1, q), c);
          gh[k] = fma(4.0, xk - x0, Dl[k][c]);
        }
#pragma unroll
        for (int l = 0; l < 3; ++l) H[c][l] = fma(gh[0], K[l], fma(gh[1], K[3 + l], gh[2] * K[6 + l]));
      }
    }
    if (DO_DIV) {
      // g_q = -w|det J_F| (c alpha)^2 [ (a-b) tr Ht - gamma c alpha d.u_q ]   (grad ln rho = -gamma d)
      double du = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double es = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (m != q) es += uu(EEI(m, q), c);
        const double uqc = fma(peq - pen, es, fma(phq - phv, uu(q, c), B0[c]));
        du = fma(d[c], uqc, du);
      }
      const double trH = H[0][0] + H[1][1] + H[2][2];
      const double gg = -cwD * alpha * alpha * fma(EQAB, trH, -gamma * cK * alpha * du);
      gq[q] = gg;
      gsum += gg;
    }
    if (SCATTER) {
      // S = F_R * (stress at q) * weight, symmetric
      double S[3][3];
      if (DO_A) {
        const double sA = cwA * etaq * alpha;
        if (FULL) {
          const double m3 = sA * (1.0 / 3.0) * (H[0][0] + H[1][1] + H[2][2]);
          S[0][0] = fma(sA, H[0][0], -m3);
          S[1][1] = fma(sA, H[1][1], -m3);
          S[2][2] = fma(sA, H[2][2], -m3);
        } else {
          S[0][0] = sA * H[0][0];
          S[1][1] = sA * H[1][1];
          S[2][2] = sA * H[2][2];
        }
        const double hs = 0.5 * sA;
        S[0][1] = S[1][0] = hs * (H[0][1] + H[1][0]);
        S[0][2] = S[2][0] = hs * (H[0][2] + H[2][0]);
        S[1][2] = S[2][1] = hs * (H[1][2] + H[2][1]);
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int l = 0; l < 3; ++l) S[c][l] = 0.0;
      }
      if (DO_BT) {  // B^T p: isotropic stress -p_q W I / (c alpha)
        const double wb = cwB * alpha * alpha * fma(EQAB, pp[q], pS);
        S[0][0] -= wb;
        S[1][1] -= wb;
        S[2][2] -= wb;
      }
      // R = S K^T ; Db_k = R[c][k-1], Db_0 = -(sum)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double Db[4];
#pragma unroll
        for (int k = 0; k < 3; ++k) Db[k + 1] = fma(S[c][0], K[3 * k], fma(S[c][1], K[3 * k + 1], S[c][2] * K[3 * k + 2]));
        Db[0] = -(Db[1] + Db[2] + Db[3]);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          if (q == 0) Sbar[m][c] = Db[m];
          else Sbar[m][c] += Db[m];
          if (m == q) {
            acc[m][c] = Db[m];
          } else {
            if (q < m) acc[EEI(m, q)][c] = Db[m];  // edge (q,m), q < m: first contribution
            else acc[EEI(m, q)][c] += Db[m];
          }
        }
      }
    }
  }
  if (SCATTER) {
    constexpr int ep[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[m][c] = fma(C_V, Sbar[m][c], acc[m][c]);
#pragma unroll
      for (int e = 0; e < 6; ++e) acc[4 + e][c] = fma(C_E, Sbar[ep[e][0]][c] + Sbar[ep[e][1]][c], acc[4 + e][c]);
    }
  }
  if (DO_DIV) {
#pragma unroll
    for (int v = 0; v < 4; ++v) gy[v] = fma(EQB, gsum, EQAB * gq[v]);
  }
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
// points Z in [4w, 4w+4]) with plain load-add-store in 5 rounds separated by __syncwarp: in one
// round all lanes (same tet type, different cubes) update the same local node index, hence
// distinct points; the 6 edge midpoints of a tet have pairwise different parity classes (host-
// checked), so they share one round, and the 4 vertices take one round each.  No atomics and no
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
  return (elem_need_u(MODE) ? 3 * kFU : 0) + (elem_u_out(MODE) ? 2 * 3 * kFY : 0) +
         kF1 + (elem_need_p(MODE) ? kF1 : 0) + (elem_p_out(MODE) ? 2 * kF1Y : 0) + kGeoSm +
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
template <bool BLEND, int MODE, bool FULL, bool ETAQ = false>
#ifndef HHG_FP_MINB
#define HHG_FP_MINB 5
#endif
__global__ void __launch_bounds__(kBT, HHG_FP_MINB)
    k_elem_fp(const MacroGeo* __restrict__ mgeo, const double* __restrict__ lgeo, const int32_t* __restrict__ bricks,
              int nb, int n1, double inv_n1, int64_t npts1, int64_t npts2, int64_t cstride,
              const double* __restrict__ eta, const double* __restrict__ u, const double* __restrict__ p,
              double* __restrict__ yu, double* __restrict__ yp, double gamma, const double* __restrict__ T2, EtaQ eq,
              int det) {
  (void)nb;
  constexpr bool NEED_U = elem_need_u(MODE);
  constexpr bool NEED_P = elem_need_p(MODE);
  constexpr bool HAS_P_OUT = elem_p_out(MODE);
  constexpr bool HAS_U_OUT = elem_u_out(MODE);
  extern __shared__ double sm[];
  double* su = sm;                                   // [3][kFU]
  double* sy = su + (NEED_U ? 3 * kFU : 0);          // [2 warps][3][kFY]
  double* se = sy + (HAS_U_OUT ? 6 * kFY : 0);       // [kF1]
  double* sp = se + kF1;                             // [kF1]
  double* syp = sp + (NEED_P ? kF1 : 0);             // [2 warps][kF1Y]
  double* sgeo = syp + (HAS_P_OUT ? 2 * kF1Y : 0);   // [kGeoSm]
  double* stt = sgeo + kGeoSm;                       // [kFU] temperature footprint (ETAQ)

  const int mac = blockIdx.y;
  const int32_t bpk = __ldg(bricks + blockIdx.x);
  const int i0 = bpk & 1023, j0 = (bpk >> 10) & 1023, k0 = bpk >> 20;
  const int delta = n1 - (i0 + j0 + k0);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int n2 = 2 * n1;
  const int64_t mb2 = (int64_t)mac * npts2, mb1 = (int64_t)mac * npts1;

  // ---- stage: u footprint (cp.async), eta / p footprints, geometry; zero the output footprints
  const double* Gm = lgeo + (int64_t)mac * kLevelGeo;
  for (int r = tid; r < kGeoSm; r += kBT) cp_async8(sgeo + r, Gm + r);
#ifdef HHG_EXP_ROWSTAGE
  // one (row, component) item per thread: 2 row-start evaluations per thread, 9 cp.async per item
  if (NEED_U || ETAQ) {
    constexpr int NI = (NEED_U ? 243 : 0) + (ETAQ ? 81 : 0);
#pragma unroll 1
    for (int it = tid; it < NI; it += kBT) {
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
    for (int L = tid; L < 729; L += kBT) {
      const int X = L % 9, Y = (L / 9) % 9, Z = L / 81;
      const int gx = 2 * i0 + X, gy = 2 * j0 + Y, gz = 2 * k0 + Z;
      if (gx + gy + gz > n2) continue;
      const double* src = u + mb2 + rowstart32(n2, gy, gz) + gx;
      HHG_CHECK(src - u >= mb2 && src - u < mb2 + npts2 && mb2 + npts2 <= cstride, "u stage", src - u, cstride);
      const int w = fword(X, Y, Z);
#pragma unroll
      for (int c = 0; c < 3; ++c) cp_async8(su + c * kFU + w, src + c * cstride);
    }
  }
  if (ETAQ) {
#pragma unroll 1
    for (int L = tid; L < 729; L += kBT) {
      const int X = L % 9, Y = (L / 9) % 9, Z = L / 81;
      const int gx = 2 * i0 + X, gy = 2 * j0 + Y, gz = 2 * k0 + Z;
      if (gx + gy + gz > n2) continue;
      cp_async8(stt + fword(X, Y, Z), T2 + mb2 + rowstart32(n2, gy, gz) + gx);
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
      for (int it = tid; it < 243; it += kBT) {
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
    for (int r = tid; r < 6 * kFY; r += kBT) sy[r] = 0.0;
  if (HAS_P_OUT)
    for (int r = tid; r < 2 * kF1Y; r += kBT) syp[r] = 0.0;
  for (int L = tid; L < kF1; L += kBT) {  // P1 footprint (points outside the lattice are never read)
    const int X = L % 5, Y = (L / 5) % 5, Z = L / 25;
    const int gx = i0 + X, gy = j0 + Y, gz = k0 + Z;
    if (gx + gy + gz > n1) continue;
    const int64_t ix = mb1 + rowstart32(n1, gy, gz) + gx;
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
  const int x = tid & 3, y = (tid >> 2) & 3, z = tid >> 4;
  const int s = i0 + j0 + k0 + x + y + z;
  const int ntypes = (s <= n1 - 3) ? 6 : ((s == n1 - 2) ? 5 : ((s == n1 - 1) ? 1 : 0));
  double xa[3];
  anchor(x, y, z, xa);
  const int cb2 = x + 2 * kPY * y + 2 * kPZ * z, cb1 = x + 5 * y + 25 * z;
  double* yw = sy + warp * 3 * kFY + (x + 2 * kPY * y + 2 * kPZ * (z - 2 * warp));
  double* ypw = syp + warp * kF1Y + (x + 5 * y + 25 * (z - 2 * warp));
#pragma unroll 1
  for (int t = 0; t < 6; ++t) {
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
    for (int L = tid; L < 729; L += kBT) {
      const int X = L % 9, Y = (L / 9) % 9, Z = L / 81;
      const int gx = 2 * i0 + X, gy = 2 * j0 + Y, gz = 2 * k0 + Z;
      if (gx + gy + gz > n2) continue;
      const int wxy = xs(X) + kPY * Y;
      double* dst = yu + mb2 + rowstart32(n2, gy, gz) + gx;
      HHG_CHECK(dst - yu >= mb2 && dst - yu < mb2 + npts2, "write-out", dst - yu, mb2 + npts2);
      const bool border = X == 0 || Y == 0 || Z == 0 || X == 8 || Y == 8 || Z == 8;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v;
        if (Z < 4) v = sy[c * kFY + wxy + kPZ * Z];
        else if (Z > 4) v = sy[3 * kFY + c * kFY + wxy + kPZ * (Z - 4)];
        else v = sy[c * kFY + wxy + kPZ * 4] + sy[3 * kFY + c * kFY + wxy];
        if (!border) dst[c * cstride] = v;
        else if (v != 0.0) {
          if (det) dst[c * cstride] += v;
          else atomicAdd(dst + c * cstride, v);
        }
      }
    }
  }
  if (HAS_P_OUT) {
    for (int L = tid; L < kF1; L += kBT) {
      const int X = L % 5, Y = (L / 5) % 5, Z = L / 25;
      const int gx = i0 + X, gy = j0 + Y, gz = k0 + Z;
      if (gx + gy + gz > n1) continue;
      double v;
      if (Z < 2) v = syp[X + 5 * Y + 25 * Z];
      else if (Z > 2) v = syp[kF1Y + X + 5 * Y + 25 * (Z - 2)];
      else v = syp[X + 5 * Y + 50] + syp[kF1Y + X + 5 * Y];
      double* dst = yp + mb1 + rowstart32(n1, gy, gz) + gx;
      const bool border = X == 0 || Y == 0 || Z == 0 || X == 4 || Y == 4 || Z == 4;
      if (!border) *dst = v;
      else if (v != 0.0) {
        if (det) *dst += v;
        else atomicAdd(dst, v);
      }
    }
  }
}

// Launch of one element-kernel instantiation: one CTA per (macro, brick) item, one launch over all bricks --
// or, in deterministic mode, one launch per brick colour.
template <bool BLEND, int MODE, bool FULL, bool ETAQ>
struct ElemKernel {
  static constexpr size_t smem = fp_smem_words<MODE, ETAQ>() * sizeof(double);
  static bool ready;
  static int prepare() {  // host-side attributes (eager: never under stream capture)
    if (ready) return HHG_OK;
    auto k = k_elem_fp<BLEND, MODE, FULL, ETAQ>;
    HHG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
    HHG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ready = true;
    return HHG_OK;
  }
  static int launch(const Mesh* m, const Level& L, const double* eta, double gamma, const double* u, const double* p,
                    double* yu, double* yp, const double* T2, EtaQ eq, cudaStream_t s) {
    HHG_TRY(prepare());
    const int64_t nm = macro_count(m);
    auto go = [&](const int32_t* list, int64_t nb, int det) {
      if (nm * nb == 0) return;
      k_elem_fp<BLEND, MODE, FULL, ETAQ><<<dim3((unsigned)nb, (unsigned)nm), kBT, smem, s>>>(m->dgeo, L.geo, list, (int)nb, L.n1,
                                                                           1.0 / L.n1, L.npts1, L.npts2, nm * L.npts2,
                                                                           eta, u, p, yu, yp, gamma, T2, eq, det);
      count_launch();
    };
    if (!m->deterministic) {
      go(L.bricks, L.n_bricks, 0);
    } else {
      for (int c = 0; c < 8; ++c) go(L.bricks_col + L.col_off[c], L.col_off[c + 1] - L.col_off[c], 1);
    }
    HHG_CUDA(cudaGetLastError());
    return HHG_OK;
  }
};
template <bool BLEND, int MODE, bool FULL, bool ETAQ>
bool ElemKernel<BLEND, MODE, FULL, ETAQ>::ready = false;

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
  HHG_PREP(true, ELEM_DIAG, true, true) HHG_PREP(false, ELEM_DIAG, true, true)
#undef HHG_PREP4
#undef HHG_PREP
  return HHG_OK;
}

}  // namespace hhg
