// Per-micro-tet arithmetic of the blended P2-P1 Stokes operator (tet_body) and its helpers, shared by
// the brick element kernel (hhg_elem.cu) and the cluster-resident coarse solver (hhg_coarse.cu).
// See hhg_elem.cu for the arithmetic layout and its paper citations.
#pragma once
#include "hhg_internal.h"

namespace hhg {

constexpr double EQA = 0.58541019662496845446;  // Q4 (5 + 3 sqrt 5)/20
constexpr double EQB = 0.13819660112501051518;  // Q4 (5 - sqrt 5)/20
constexpr double EQAB = EQA - EQB;              // 1/sqrt 5
constexpr double EWQ = 1.0 / 24.0;              // Q4 weight (reference volume 1/6, 4 points)
constexpr double C_SB = 1.2360679774997896964;  // 4b/(a-b) = sqrt5 - 1
constexpr double F_R = 4.0 * EQAB;              // prescale of R (folds 4(a-b) of the scatter)
constexpr double C_V = -0.25;                   // (4b-1)/F_R
constexpr double C_E = 0.30901699437494742410;  // 4b/F_R = (sqrt5-1)/4

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

}  // namespace hhg
