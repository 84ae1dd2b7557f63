// Temperature operator of eq:WeakTemp (SURVEY §8(f) NEXT-4 without the MMOC step):
//   L(T, w) = s int T w + tau [ int (u . grad T) w + int kappa grad T . grad(w / rho) - int beta T (u . g) w ]
// rho = exp(gamma (1 - r)) (grad ln rho = -gamma x/|x|), g = -x/|x|, so
// grad(w / rho) = (grad w + gamma w x/|x|) / rho and -beta T (u . g) w = +beta T (u . x/|x|) w.
// P(T, w) = s int T w + tau int (kappa / rho) grad T . grad w is the symmetric mass + diffusion part the
// paper's FGMRES is preconditioned with.  Q4 rule, blended geometry (J = J_B J_F) as for A.
// Not the hot path of the Stokes solve: one thread per micro tet, generic 3x3 algebra, fp64 REDs into
// the scalar P2 output, then the interface sum.
#include <cmath>

#include "hhg_internal.h"

namespace hhg {
namespace {
constexpr double TQA = 0.58541019662496845446, TQB = 0.13819660112501051518;  // Q4 barycentric
__constant__ int kTV[6][4][3] = {
    {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
    {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}}};
__constant__ int kEP[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

__device__ __forceinline__ int rs32(int N, int j, int k) {
  const int M = N - k;
  return ((N + 1) * (N + 2) * (N + 3) - (M + 1) * (M + 2) * (M + 3)) / 6 + (j * (2 * M + 3 - j)) / 2;
}

// MODE 0: y = L T, 1: y = P T, 2: y = diag(P)
template <int MODE>
__global__ void k_temp(const MacroGeo* __restrict__ mgeo, int n1, int64_t npts2, int64_t cstride, bool blend,
                       TempCoef cf, const double* __restrict__ u, const double* __restrict__ T, double* __restrict__ y) {
  const int mac = blockIdx.z;
  const int j = blockIdx.y % n1, k = blockIdx.y / n1;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int sc = i + j + k;
  if (sc > n1 - 1) return;
  const MacroGeo& g = mgeo[mac];
  const int n2 = 2 * n1;
  const int64_t mb = (int64_t)mac * npts2;
  const double inv = 1.0 / n1;
  for (int t = 0; t < 6; ++t) {
    if ((t == 0 && sc > n1 - 1) || (t >= 1 && t <= 4 && sc > n1 - 2) || (t == 5 && sc > n1 - 3)) continue;
    // vertices (unblended), P2 node indices
    double X[4][3];
    int idx[10];
    for (int v = 0; v < 4; ++v) {
      const double f[3] = {(i + kTV[t][v][0]) * inv, (j + kTV[t][v][1]) * inv, (k + kTV[t][v][2]) * inv};
      for (int r = 0; r < 3; ++r) X[v][r] = g.X0[r] + g.Jm[3 * r] * f[0] + g.Jm[3 * r + 1] * f[1] + g.Jm[3 * r + 2] * f[2];
      idx[v] = rs32(n2, 2 * (j + kTV[t][v][1]), 2 * (k + kTV[t][v][2])) + 2 * (i + kTV[t][v][0]);
    }
    for (int e = 0; e < 6; ++e) {
      const int a = kEP[e][0], b = kEP[e][1];
      idx[4 + e] = rs32(n2, 2 * j + kTV[t][a][1] + kTV[t][b][1], 2 * k + kTV[t][a][2] + kTV[t][b][2]) + 2 * i +
                   kTV[t][a][0] + kTV[t][b][0];
    }
    double Tv[10] = {0}, Uv[10][3] = {{0}};
    for (int a = 0; a < 10; ++a) {
      if (MODE != 2) Tv[a] = T[mb + idx[a]];
      if (MODE == 0)
        for (int c = 0; c < 3; ++c) Uv[a][c] = u[c * cstride + mb + idx[a]];
    }
    double JF[3][3];  // columns X_v - X_0
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) JF[r][c] = X[c + 1][r] - X[0][r];
    double out[10] = {0};
    for (int q = 0; q < 4; ++q) {
      double lam[4];
      for (int v = 0; v < 4; ++v) lam[v] = v == q ? TQA : TQB;
      double x[3];
      for (int r = 0; r < 3; ++r) x[r] = lam[0] * X[0][r] + lam[1] * X[1][r] + lam[2] * X[2][r] + lam[3] * X[3][r];
      const double rr = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
      double J[3][3], rphys = rr;
      if (blend) {
        const double nx = g.nhat[0] * x[0] + g.nhat[1] * x[1] + g.nhat[2] * x[2];
        const double ph = nx / rr;
        double gp[3];
        for (int r = 0; r < 3; ++r) gp[r] = g.nhat[r] / rr - nx * x[r] / (rr * rr * rr);
        double JB[3][3];
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) JB[r][c] = g.cK * ((r == c ? ph : 0.0) + x[r] * gp[c]);
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) J[r][c] = JB[r][0] * JF[0][c] + JB[r][1] * JF[1][c] + JB[r][2] * JF[2][c];
        rphys = g.cK * nx;
      } else {
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) J[r][c] = JF[r][c];
      }
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      double Ji[3][3];  // J^-1 = adj(J) / det
      Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
      const double W = fabs(det) / 24.0;
      // P2 basis values and physical gradients: grad phi = J^-T grad_xi phi
      const double DL[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
      double ph[10], gr[10][3];
      for (int a = 0; a < 10; ++a) {
        double gx[3];
        if (a < 4) {
          ph[a] = lam[a] * (2.0 * lam[a] - 1.0);
          for (int m = 0; m < 3; ++m) gx[m] = (4.0 * lam[a] - 1.0) * DL[a][m];
        } else {
          const int p = kEP[a - 4][0], r = kEP[a - 4][1];
          ph[a] = 4.0 * lam[p] * lam[r];
          for (int m = 0; m < 3; ++m) gx[m] = 4.0 * (lam[p] * DL[r][m] + lam[r] * DL[p][m]);
        }
        for (int d = 0; d < 3; ++d) gr[a][d] = Ji[0][d] * gx[0] + Ji[1][d] * gx[1] + Ji[2][d] * gx[2];
      }
      const double rho_i = exp(-cf.gamma * (1.0 - rphys));  // 1 / rho
      double xh[3] = {x[0] / rr, x[1] / rr, x[2] / rr};
      if (MODE == 2) {
        for (int a = 0; a < 10; ++a)
          out[a] += W * (cf.s * ph[a] * ph[a] +
                         cf.tau * cf.kappa * rho_i * (gr[a][0] * gr[a][0] + gr[a][1] * gr[a][1] + gr[a][2] * gr[a][2]));
        continue;
      }
      double Tq = 0.0, gT[3] = {0, 0, 0}, uq[3] = {0, 0, 0};
      for (int a = 0; a < 10; ++a) {
        Tq += ph[a] * Tv[a];
        for (int d = 0; d < 3; ++d) gT[d] += Tv[a] * gr[a][d];
        if (MODE == 0)
          for (int d = 0; d < 3; ++d) uq[d] += ph[a] * Uv[a][d];
      }
      const double adv = uq[0] * gT[0] + uq[1] * gT[1] + uq[2] * gT[2];
      const double ux = uq[0] * xh[0] + uq[1] * xh[1] + uq[2] * xh[2];
      const double xg = xh[0] * gT[0] + xh[1] * gT[1] + xh[2] * gT[2];
      for (int a = 0; a < 10; ++a) {
        const double dg = gr[a][0] * gT[0] + gr[a][1] * gT[1] + gr[a][2] * gT[2];
        double v = cf.s * ph[a] * Tq + cf.tau * cf.kappa * rho_i * dg;
        if (MODE == 0) v += cf.tau * (ph[a] * adv + cf.kappa * rho_i * cf.gamma * ph[a] * xg + cf.beta * ph[a] * Tq * ux);
        out[a] += W * v;
      }
    }
    for (int a = 0; a < 10; ++a) atomicAdd(y + mb + idx[a], out[a]);
  }
}
}  // namespace

int launch_temp(const Mesh* m, const Level& L, int mode, TempCoef cf, const double* u, const double* T, double* y,
                cudaStream_t s) {
  const int64_t nm = macro_count(m);
  if (nm == 0) return HHG_OK;
  HHG_TRY(ensure_device_geo(const_cast<Mesh*>(m)));
  const int n1 = L.n1;
  dim3 grid((unsigned)((n1 + 31) / 32), (unsigned)(n1 * n1), (unsigned)nm);
  const bool bl = m->blend == HHG_BLEND_SHELL;
  const int64_t cs = nm * L.npts2;
  if (mode == 0) k_temp<0><<<grid, 32, 0, s>>>(m->dgeo, n1, L.npts2, cs, bl, cf, u, T, y);
  else if (mode == 1) k_temp<1><<<grid, 32, 0, s>>>(m->dgeo, n1, L.npts2, cs, bl, cf, u, T, y);
  else k_temp<2><<<grid, 32, 0, s>>>(m->dgeo, n1, L.npts2, cs, bl, cf, u, T, y);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}
}  // namespace hhg
