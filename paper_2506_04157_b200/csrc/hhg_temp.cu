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

// ------------------------------------------------------------------ MMOC
// Per owned stored P2 node: RK4 back-tracking along u(y, th) = (1 - th) u_new(y) + th u_old(y),
// X = x - tau/6 (k1 + 2 k2 + 2 k3 + k4), T_hat = T(X).  A physical point is located by inverse blending
// (directions are kept: x = |y| / (c n.y^) y^), the macro's barycentric coordinates (own macro of the
// previous stage first, then all macros), the lattice cube and the one of its 6 tets (valid for the
// cube's anchor sum) with the largest minimum barycentric coordinate; points outside the shell are
// moved radially onto it (R28).
namespace {
__constant__ double kTinv[6][9];  // per tet type: inverse of [V1-V0 | V2-V0 | V3-V0] (unit-cube offsets)

struct Loc {
  int mac, t, ci, cj, ck;
  double mu[4];
};

__device__ bool locate(const MacroGeo* __restrict__ mg, int nm, int n1, bool blend, const double (&y)[3], int hint,
                       double tol, Loc& L) {
  const double ry = sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2]);
  const double d[3] = {y[0] / ry, y[1] / ry, y[2] / ry};
  for (int a = 0; a <= nm; ++a) {
    const int m = a == 0 ? hint : (a - 1 < hint ? a - 1 : a);
    if (m >= nm) break;
    const MacroGeo& g = mg[m];
    double x[3];
    if (blend) {
      const double den = g.cK * (g.nhat[0] * d[0] + g.nhat[1] * d[1] + g.nhat[2] * d[2]);
      if (!(den > 0.0)) continue;
      for (int r = 0; r < 3; ++r) x[r] = ry / den * d[r];
    } else {
      for (int r = 0; r < 3; ++r) x[r] = y[r];
    }
    double lam[3];
    for (int r = 0; r < 3; ++r)
      lam[r] = g.Jminv[3 * r] * (x[0] - g.X0[0]) + g.Jminv[3 * r + 1] * (x[1] - g.X0[1]) + g.Jminv[3 * r + 2] * (x[2] - g.X0[2]);
    if (fmin(fmin(lam[0], lam[1]), lam[2]) < -tol || lam[0] + lam[1] + lam[2] > 1.0 + tol) continue;
    double xi[3];
    int c[3];
    for (int r = 0; r < 3; ++r) {
      xi[r] = n1 * lam[r];
      c[r] = min(max((int)floor(xi[r]), 0), n1 - 1);
    }
    while (c[0] + c[1] + c[2] > n1 - 1) {  // far-face points: step back along a coordinate with f ~ 0
      int r = 0;
      double best = 2.0;
      for (int q = 0; q < 3; ++q)
        if (c[q] > 0 && xi[q] - c[q] < best) best = xi[q] - c[q], r = q;
      --c[r];
    }
    const int sc = c[0] + c[1] + c[2];
    const double f[3] = {xi[0] - c[0], xi[1] - c[1], xi[2] - c[2]};
    double bestmin = -1e300;
    for (int t = 0; t < 6; ++t) {
      if ((t >= 1 && t <= 4 && sc > n1 - 2) || (t == 5 && sc > n1 - 3)) continue;
      double o[3];
      for (int r = 0; r < 3; ++r) o[r] = f[r] - kTV[t][0][r];
      double mu[4];
      for (int r = 0; r < 3; ++r) mu[r + 1] = kTinv[t][3 * r] * o[0] + kTinv[t][3 * r + 1] * o[1] + kTinv[t][3 * r + 2] * o[2];
      mu[0] = 1.0 - mu[1] - mu[2] - mu[3];
      const double mn = fmin(fmin(mu[0], mu[1]), fmin(mu[2], mu[3]));
      if (mn > bestmin) {
        bestmin = mn;
        L.t = t;
        for (int v = 0; v < 4; ++v) L.mu[v] = mu[v];
      }
    }
    L.mac = m;
    L.ci = c[0];
    L.cj = c[1];
    L.ck = c[2];
    return true;
  }
  return false;
}

// P2 basis of the located tet and the stored indices of its 10 nodes
__device__ void p2_eval_setup(const Loc& L, int n1, double (&ph)[10], int (&idx)[10]) {
  const int n2 = 2 * n1;
  for (int v = 0; v < 4; ++v) {
    ph[v] = L.mu[v] * (2.0 * L.mu[v] - 1.0);
    idx[v] = rs32(n2, 2 * (L.cj + kTV[L.t][v][1]), 2 * (L.ck + kTV[L.t][v][2])) + 2 * (L.ci + kTV[L.t][v][0]);
  }
  for (int e = 0; e < 6; ++e) {
    const int a = kEP[e][0], b = kEP[e][1];
    ph[4 + e] = 4.0 * L.mu[a] * L.mu[b];
    idx[4 + e] = rs32(n2, 2 * L.cj + kTV[L.t][a][1] + kTV[L.t][b][1], 2 * L.ck + kTV[L.t][a][2] + kTV[L.t][b][2]) +
                 2 * L.ci + kTV[L.t][a][0] + kTV[L.t][b][0];
  }
}

__device__ __forceinline__ void clamp_r(double (&y)[3], bool blend, double rmin, double rmax) {
  if (!blend) return;
  const double r = sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2]);
  const double s = r > rmax ? rmax / r : (r < rmin ? rmin / r : 1.0);
  for (int q = 0; q < 3; ++q) y[q] *= s;
}

__global__ void k_mmoc(const MacroGeo* __restrict__ mg, int nm, const int32_t* __restrict__ rows, int64_t nrows, int n1,
                       int64_t npts2, const uint8_t* __restrict__ own, bool blend, double rmin, double rmax, double tau,
                       const double* __restrict__ T, const double* __restrict__ un, const double* __restrict__ uo,
                       double* __restrict__ out, int* __restrict__ fail_flag) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const int n2 = 2 * n1;
  const int j = rows[row] & 0xffff, k = rows[row] >> 16, len = n2 - j - k + 1;
  const int mac = blockIdx.y;
  const int64_t cs = (int64_t)nm * npts2;
  const MacroGeo& g = mg[mac];
  for (int i = threadIdx.x & 31; i < len; i += 32) {
    const int64_t node = (int64_t)mac * npts2 + rs32(n2, j, k) + i;
    if (!own[node]) continue;
    double x[3];
    const double a = (double)i / n2, b = (double)j / n2, c = (double)k / n2;
    for (int r = 0; r < 3; ++r) x[r] = g.X0[r] + g.Jm[3 * r] * a + g.Jm[3 * r + 1] * b + g.Jm[3 * r + 2] * c;
    if (blend) {
      const double rr = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
      const double fct = g.cK * (g.nhat[0] * x[0] + g.nhat[1] * x[1] + g.nhat[2] * x[2]) / rr;
      for (int r = 0; r < 3; ++r) x[r] *= fct;
    }
    int hint = mac;
    bool ok = true;
    auto vel = [&](const double (&p)[3], double th, double (&v)[3]) {
      double y[3] = {p[0], p[1], p[2]};
      clamp_r(y, blend, rmin, rmax);
      Loc L;
      if (!locate(mg, nm, n1, blend, y, hint, 1e-12, L) && !locate(mg, nm, n1, blend, y, hint, 1e-9, L)) {
        ok = false;
        v[0] = v[1] = v[2] = 0.0;
        return;
      }
      hint = L.mac;
      double ph[10];
      int id[10];
      p2_eval_setup(L, n1, ph, id);
      const int64_t mb = (int64_t)L.mac * npts2;
      for (int q = 0; q < 3; ++q) {
        double sn = 0.0, so = 0.0;
        for (int e = 0; e < 10; ++e) {
          sn += ph[e] * un[q * cs + mb + id[e]];
          so += ph[e] * uo[q * cs + mb + id[e]];
        }
        v[q] = (1.0 - th) * sn + th * so;
      }
    };
    double k1[3], k2[3], k3[3], k4[3], p[3];
    vel(x, 0.0, k1);
    for (int q = 0; q < 3; ++q) p[q] = x[q] - 0.5 * tau * k1[q];
    vel(p, 0.5, k2);
    for (int q = 0; q < 3; ++q) p[q] = x[q] - 0.5 * tau * k2[q];
    vel(p, 0.5, k3);
    for (int q = 0; q < 3; ++q) p[q] = x[q] - tau * k3[q];
    vel(p, 1.0, k4);
    for (int q = 0; q < 3; ++q) p[q] = x[q] - tau / 6.0 * (k1[q] + 2.0 * k2[q] + 2.0 * k3[q] + k4[q]);
    clamp_r(p, blend, rmin, rmax);
    Loc L;
    double val = 0.0;
    if (locate(mg, nm, n1, blend, p, hint, 1e-12, L) || locate(mg, nm, n1, blend, p, hint, 1e-9, L)) {
      double ph[10];
      int id[10];
      p2_eval_setup(L, n1, ph, id);
      const int64_t mb = (int64_t)L.mac * npts2;
      for (int e = 0; e < 10; ++e) val += ph[e] * T[mb + id[e]];
    } else {
      ok = false;
    }
    out[node] = val;
    if (!ok) atomicOr(fail_flag, 1);
  }
}
}  // namespace

int launch_mmoc(const Mesh* m, const Level& L, double rmin, double rmax, double tau, const double* T, const double* un,
                const double* uo, double* out, int* fail_flag, cudaStream_t s) {
  static bool tinv_ready = false;
  if (!tinv_ready) {
    const int TV[6][4][3] = {
        {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, {{0, 1, 0}, {1, 0, 0}, {1, 0, 1}, {1, 1, 0}},
        {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {1, 0, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
        {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 1}}, {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}}};
    double inv[6][9];
    for (int t = 0; t < 6; ++t) {
      double E[3][3];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) E[r][c] = TV[t][c + 1][r] - TV[t][0][r];
      const double det = E[0][0] * (E[1][1] * E[2][2] - E[1][2] * E[2][1]) - E[0][1] * (E[1][0] * E[2][2] - E[1][2] * E[2][0]) +
                         E[0][2] * (E[1][0] * E[2][1] - E[1][1] * E[2][0]);
      inv[t][0] = (E[1][1] * E[2][2] - E[1][2] * E[2][1]) / det;
      inv[t][1] = (E[0][2] * E[2][1] - E[0][1] * E[2][2]) / det;
      inv[t][2] = (E[0][1] * E[1][2] - E[0][2] * E[1][1]) / det;
      inv[t][3] = (E[1][2] * E[2][0] - E[1][0] * E[2][2]) / det;
      inv[t][4] = (E[0][0] * E[2][2] - E[0][2] * E[2][0]) / det;
      inv[t][5] = (E[0][2] * E[1][0] - E[0][0] * E[1][2]) / det;
      inv[t][6] = (E[1][0] * E[2][1] - E[1][1] * E[2][0]) / det;
      inv[t][7] = (E[0][1] * E[2][0] - E[0][0] * E[2][1]) / det;
      inv[t][8] = (E[0][0] * E[1][1] - E[0][1] * E[1][0]) / det;
    }
    HHG_CUDA(cudaMemcpyToSymbol(kTinv, inv, sizeof(inv)));
    tinv_ready = true;
  }
  HHG_TRY(ensure_device_geo(const_cast<Mesh*>(m)));
  const int64_t nm = macro_count(m);
  if (nm == 0) return HHG_OK;
  dim3 grid((unsigned)((L.nrows2 + 7) / 8), (unsigned)nm);
  k_mmoc<<<grid, 256, 0, s>>>(m->dgeo, (int)nm, L.rows2, L.nrows2, L.n1, L.npts2, L.own2, m->blend == HHG_BLEND_SHELL,
                              rmin, rmax, tau, T, un, uo, out, fail_flag);
  count_launch();
  HHG_CUDA(cudaGetLastError());
  return HHG_OK;
}

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
