// Per-voxel constitutive update (K1), commit (K10) and staggered-error reductions.
//
// J2-Lemaitre with linear hardening (backward Euler App. A P:1131-1160 with the
// main-text sqrt(2/3) convention, A-14, and the total-form stress sigma = (1-D) sigma~, A-15):
//   s_tr = 2 mu (dev eps - eps^p_n), q = |s_tr|, f = q - sqrt(2/3)(sigma_y + H eps_p,n)
//   f > 0: dlam = f/(2mu + 2H/3), n = s_tr/q, eps^p = eps^p_n + dlam n, eps_p = eps_p,n + sqrt(2/3) dlam
//   sigma = (1-D)[K tr(eps) I + 2mu(dev eps - eps^p)]
//   C = (1-D)[K 1x1 + 2 mu theta I_dev - 2 mu thetabar n x n]  (theta = 1 - 2mu dlam/q,
//       thetabar = 1/(1 + H/(3mu)) - (1 - theta))
// with D frozen from the non-local field, D = max(D_n, D(abar)) (A-16),
// capped at d_max.  Elastic phase: C_e.  Elastic-brittle particle (A-18):
// eps_eq = sqrt(eps:C_p:eps/E), kappa = max(kappa_n, abar_p), d = clamp((kappa-k0)/(kf-k0), 0, d_max).
// Sources of the Helmholtz equations: alpha_j = eps_p (J2 phase) or eps_eq
// (brittle phase) on the source phase of field j, 0 elsewhere.
// One thread per voxel; all loads/stores are component-planar and coalesced along x.
#include "reduce.cuh"

namespace fgd {

struct MatTable {
  Material m[kMaxPhases];
  int field_of[kMaxPhases];
  int nfields;
};

__device__ __forceinline__ double clamp01cap(double v, double cap) {
  v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  return v < cap ? v : cap;
}

// The consistent tangent of every model here has the structure
//   C = ca 1(x)1 + cb I - cc n(x)n        (1 = (1,1,1,0,0,0) in Mandel form)
// so it is stored compactly as 9 doubles per voxel [n0..n5, ca, cb, cc] (72 B instead of the
// 168 B of the packed 6x6; the CG reads it every iteration).
struct PointOut {
  double sig[6];
  double n[6];
  double ca, cb, cc;
  double epsp[6];
  double ep;
  double alpha;
  double alpha2;    // GTN: source of the phase's second field (tr eps^p)
  int fail;         // GTN: return mapping did not converge
};

__device__ __forceinline__ void elastic_C(double K, double mu, double f, PointOut& o) {
  // f (K 1x1 + 2 mu I_dev) = f (K - 2mu/3) 1x1 + f 2mu I
  o.ca = f * (K - 2.0 * mu / 3.0);
  o.cb = f * 2.0 * mu;
  o.cc = 0.0;
  for (int i = 0; i < 6; ++i) o.n[i] = 0.0;
}


// ---------------------------------------------------------------------------------------------
// Non-local GTN (model 3): Sec. 2.1.1, Sec. 2.2.2, App. A P:1100-1129.
// Mandel vectors; q = Mises stress (the paper's s), p = -tr(sigma)/3, sigma_0 = sigma_y x.
// Frozen porosity (App. A P:1119 with the non-local fields of the staggered iterate, A-30):
//   f = max(f_n, (f_n + A_N(ebar0) (ebar0 - ebar0_n) + (trbar - trbar_n)) / (1 + trbar - trbar_n)), <= 1
// Return mapping in u = (a, b, x): d eps^p = (a/3) 1 + b n, n = 1.5 s_tr/q_tr, p = p_tr + K a,
// q = q_tr - 3 mu b, residuals (scaled)
//   R1 = a Q + b c sinh(xi)                         (normality with dlam eliminated)
//   R2 = Q^2 + 2 f* q1 cosh(xi) - 1 - q3 f*^2       (yield)
//   R3 = (1 - f)(e(x) - e_n) + P a - Q b            (plastic work P:125-131 over sigma_0)
// P = p/sigma_0, Q = q/sigma_0, xi = 1.5 q2 P, c = 1.5 f* q1 q2, e(x) = sigma_y (x^(1/N) - x)/(3 mu)
// (Aravas P:826-829 solved for eps0p).  Newton from (0, 0, x_n) with step halving on |R|^2 and
// x >= 1; converged when the Newton step is at round-off (relative 1e-13, plus an absolute
// 1e-14 sigma_y/(3 mu) on a, b: the rounding floor of e(x) near x = 1); 50 iterations max.
// Tangent: du = -J^-1 dR/d(p_tr, q_tr) (dp_tr, dq_tr), dp_tr = -K 1:de, dq_tr = 2 mu n:de, giving
//   C = 2 mu theta I_dev + K a_pp 1x1 - 2 mu a_pq 1xn - (2/3) K a_qp nx1 + (4/3) mu (a_qq - theta) nxn,
// used symmetrised (A-32): ca 1x1 + cb I - cc nxn + cd (1xn + nx1) with cb = 2 mu theta,
// ca = K a_pp - cb/3, cc = (4/3) mu (theta - a_qq), cd = -mu a_pq - K a_qp/3 (cd := 0 where
// |cc| < 1e-6 cb, A-33), and folded into the compact form with m = n - (cd/cc) 1:
//   ca 1x1 - cc nxn + cd (1xn + nx1) = (ca + cd^2/cc) 1x1 - cc m x m.
__device__ __forceinline__ double gtn_fstar(double f, const Material& m) {
  const double fv = (m.q1 + sqrt(m.q1 * m.q1 - m.q3)) / m.q3;
  double fs = f < m.f_c ? f : (f < m.f_f ? m.f_c + (fv - m.f_c) / (m.f_f - m.f_c) * (f - m.f_c) : fv);
  return fs < m.fstar_max ? fs : m.fstar_max;
}

__device__ __forceinline__ double gtn_porosity(double fn, double e0, double e0n, double t, double tn,
                                               const Material& m) {
  const double z = (e0 - m.eps_n) / m.s_n;
  const double AN = m.f_n / (m.s_n * 2.50662827463100050242) * exp(-0.5 * z * z);   // sqrt(2 pi)
  const double dt = t - tn;
  double f = (fn + AN * (e0 - e0n) + dt) / (1.0 + dt);
  f = f > fn ? f : fn;   // irreversible (A-30): no net void closure
  return f > 1.0 ? 1.0 : f;
}

// x = sigma_0/sigma_y at eps0p = e: Newton on x^(1/N) - x - 3 mu e/sigma_y from x = 1
__device__ double gtn_aravas_x(double e, const Material& m, double mu) {
  const double c = 3.0 * mu * e / m.sigma_y;
  if (!(c > 0.0)) return 1.0;
  const double iN = 1.0 / m.n_hard;
  double x = 1.0;
  for (int it = 0; it < 100; ++it) {
    const double xp = exp((iN - 1.0) * log(x));
    const double dx = (xp * x - x - c) / (iN * xp - 1.0);
    x -= dx;
    if (fabs(dx) <= 1e-15 * x) break;
  }
  return x;
}

struct GtnCtx {
  double ptr, qtr, e0n, f, fs, K, mu;
};

__device__ void gtn_eval(const Material& m, const GtnCtx& g, const double u[3], double R[3], double J[3][3],
                         double B[3][2]) {
  const double a = u[0], b = u[1], x = u[2];
  const double s0 = m.sigma_y * x, is0 = 1.0 / s0;
  const double P = (g.ptr + g.K * a) * is0, Q = (g.qtr - 3.0 * g.mu * b) * is0;
  const double k = 1.5 * m.q2, xi = k * P;
  const double c = 1.5 * g.fs * m.q1 * m.q2;
  const double ex = exp(xi), iex = 1.0 / ex;   // cosh and sinh from one exponential
  const double ch = 0.5 * (ex + iex), sh = 0.5 * (ex - iex);
  const double iN = 1.0 / m.n_hard;
  const double xp = exp((iN - 1.0) * log(x));   // x^(1/N - 1), x >= 1 (cheaper than the IEEE pow)
  const double e0 = m.sigma_y * (xp * x - x) / (3.0 * g.mu);
  R[0] = a * Q + b * c * sh;
  R[1] = Q * Q + 2.0 * g.fs * m.q1 * ch - 1.0 - m.q3 * g.fs * g.fs;
  R[2] = (1.0 - g.f) * (e0 - g.e0n) + P * a - Q * b;
  if (J) {
    const double dPa = g.K * is0, dPx = -P / x, dQb = -3.0 * g.mu * is0, dQx = -Q / x;
    const double dex = m.sigma_y * (iN * xp - 1.0) / (3.0 * g.mu);
    const double tq = 2.0 * g.fs * m.q1 * sh * k;   // d(2 f* q1 cosh xi)/dP
    J[0][0] = Q + b * c * ch * k * dPa;
    J[0][1] = a * dQb + c * sh;
    J[0][2] = a * dQx + b * c * ch * k * dPx;
    J[1][0] = tq * dPa;
    J[1][1] = 2.0 * Q * dQb;
    J[1][2] = 2.0 * Q * dQx + tq * dPx;
    J[2][0] = P + a * dPa;
    J[2][1] = -Q - b * dQb;
    J[2][2] = (1.0 - g.f) * dex + a * dPx - b * dQx;
    B[0][0] = b * c * ch * k * is0;
    B[0][1] = a * is0;
    B[1][0] = tq * is0;
    B[1][1] = 2.0 * Q * is0;
    B[2][0] = a * is0;
    B[2][1] = -b * is0;
  }
}

// x = A^-1 r (Cramer)
__device__ __forceinline__ void solve3(const double A[3][3], const double r[3], double x[3]) {
  const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1];
  const double c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2];
  const double c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
  const double id = 1.0 / (A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02);
  const double c10 = A[0][2] * A[2][1] - A[0][1] * A[2][2];
  const double c11 = A[0][0] * A[2][2] - A[0][2] * A[2][0];
  const double c12 = A[0][1] * A[2][0] - A[0][0] * A[2][1];
  const double c20 = A[0][1] * A[1][2] - A[0][2] * A[1][1];
  const double c21 = A[0][2] * A[1][0] - A[0][0] * A[1][2];
  const double c22 = A[0][0] * A[1][1] - A[0][1] * A[1][0];
  x[0] = (c00 * r[0] + c10 * r[1] + c20 * r[2]) * id;
  x[1] = (c01 * r[0] + c11 * r[1] + c21 * r[2]) * id;
  x[2] = (c02 * r[0] + c12 * r[1] + c22 * r[2]) * id;
}

// trial state; returns true if the trial violates the yield condition (plastic)
__device__ __forceinline__ bool gtn_setup(const Material& m, double K, double mu, const double* e,
                                          const double* epsp_n, double e0n, double f, GtnCtx& g, double* n,
                                          double& xn, bool& tiny, double* sig_el) {
  double ee[6];
  for (int i = 0; i < 6; ++i) ee[i] = e[i] - epsp_n[i];
  const double tr = ee[0] + ee[1] + ee[2];
  double s_tr[6], ss = 0.0;
  for (int i = 0; i < 6; ++i) {
    s_tr[i] = 2.0 * mu * (ee[i] - (i < 3 ? tr / 3.0 : 0.0));
    ss += s_tr[i] * s_tr[i];
  }
  g = GtnCtx{-K * tr, sqrt(1.5 * ss), e0n, f, gtn_fstar(f, m), K, mu};
  xn = gtn_aravas_x(e0n, m, mu);
  const double Ptr = g.ptr / (m.sigma_y * xn), Qtr = g.qtr / (m.sigma_y * xn);
  const double phi_tr = Qtr * Qtr + 2.0 * g.fs * m.q1 * cosh(1.5 * m.q2 * Ptr) - 1.0 - m.q3 * g.fs * g.fs;
  tiny = g.qtr <= 1e-12 * m.sigma_y;
  for (int i = 0; i < 6; ++i) {
    n[i] = tiny ? 0.0 : 1.5 * s_tr[i] / g.qtr;
    sig_el[i] = s_tr[i] + (i < 3 ? K * tr : 0.0);
  }
  return phi_tr > 0.0;
}

__device__ __forceinline__ void gtn_elastic_out(double K, double mu, const double* sig_el, const double* epsp_n,
                                                double e0n, PointOut& o) {
  for (int i = 0; i < 6; ++i) {
    o.sig[i] = sig_el[i];
    o.epsp[i] = epsp_n[i];
  }
  elastic_C(K, mu, 1.0, o);
  o.ep = e0n;
  o.alpha = e0n;
  o.alpha2 = epsp_n[0] + epsp_n[1] + epsp_n[2];
  o.fail = 0;
}

// One Newton step of the return mapping at u (R, J, B at u on entry, at the new u on exit).
// J, B always hold the Jacobians at u: the line-search candidates are evaluated with them
// (J at u is dead once du is known), so an accepted step needs no second evaluation.
// Returns true when the step was at round-off (u then holds the converged point).
__device__ __forceinline__ bool gtn_newton_step(const Material& m, const GtnCtx& g, double* u, double* R,
                                                double (&J)[3][3], double (&B)[3][2]) {
  double du[3];
  solve3(J, R, du);
  for (int i = 0; i < 3; ++i) du[i] = -du[i];
  if (fabs(du[0]) + fabs(du[1]) <= 1e-13 * (fabs(u[0]) + fabs(u[1])) + 1e-14 * m.sigma_y / (3.0 * g.mu) &&
      fabs(du[2]) <= 1e-13 * u[2]) {
    for (int i = 0; i < 3; ++i) u[i] += du[i];
    return true;
  }
  const double psi = R[0] * R[0] + R[1] * R[1] + R[2] * R[2];
  double t = 1.0, un[3];
  for (int ls = 0; ls < 30; ++ls) {
    for (int i = 0; i < 3; ++i) un[i] = u[i] + t * du[i];
    un[2] = un[2] > 1.0 ? un[2] : 1.0;
    gtn_eval(m, g, un, R, J, B);
    if (R[0] * R[0] + R[1] * R[1] + R[2] * R[2] < psi) break;
    t *= 0.5;
  }
  for (int i = 0; i < 3; ++i) u[i] = un[i];
  return false;
}

// stress, plastic state, sources and the compact consistent tangent at the returned point u
__device__ __forceinline__ void gtn_finish(const Material& m, const GtnCtx& g, const double* u, const double* n,
                                           bool tiny, const double* epsp_n, bool conv, PointOut& o) {
  const double K = g.K, mu = g.mu;
  o.fail = conv ? 0 : 1;
  const double a = u[0], b = u[1], x = u[2];
  const double p = g.ptr + K * a, q = g.qtr - 3.0 * mu * b;
  for (int i = 0; i < 6; ++i) {
    o.sig[i] = (2.0 / 3.0) * q * n[i] - (i < 3 ? p : 0.0);
    o.epsp[i] = epsp_n[i] + b * n[i] + (i < 3 ? a / 3.0 : 0.0);
  }
  o.ep = m.sigma_y * (pow(x, 1.0 / m.n_hard) - x) / (3.0 * mu);
  o.alpha = o.ep;
  o.alpha2 = o.epsp[0] + o.epsp[1] + o.epsp[2];
  double R[3], J[3][3], B[3][2];
  gtn_eval(m, g, u, R, J, B);
  double Mc[3][2];
  for (int col = 0; col < 2; ++col) {
    const double rhs[3] = {B[0][col], B[1][col], B[2][col]};
    double sol[3];
    solve3(J, rhs, sol);
    for (int i = 0; i < 3; ++i) Mc[i][col] = -sol[i];
  }
  const double a_pp = 1.0 + K * Mc[0][0], a_pq = K * Mc[0][1];
  const double a_qp = -3.0 * mu * Mc[1][0], a_qq = 1.0 - 3.0 * mu * Mc[1][1];
  const double theta = tiny ? 1.0 : q / g.qtr;
  const double cb = 2.0 * mu * theta;
  double ca = K * a_pp - cb / 3.0;
  const double cc = (4.0 / 3.0) * mu * (theta - a_qq);
  double cd = -mu * a_pq - K * a_qp / 3.0;
  if (fabs(cc) < 1e-6 * cb) cd = 0.0;
  const double gam = cd != 0.0 ? cd / cc : 0.0;
  ca += cd * gam;
  o.ca = ca;
  o.cb = cb;
  o.cc = cc;
  for (int i = 0; i < 6; ++i) o.n[i] = n[i] - (i < 3 ? gam : 0.0);
}

__device__ __forceinline__ void gtn_update(const Material& m, double K, double mu, const double* e, const double* epsp_n,
                                           double e0n, double f, PointOut& o) {
  GtnCtx g;
  double n[6], sig_el[6], xn;
  bool tiny;
  if (!gtn_setup(m, K, mu, e, epsp_n, e0n, f, g, n, xn, tiny, sig_el)) {
    gtn_elastic_out(K, mu, sig_el, epsp_n, e0n, o);
    return;
  }
  double u[3] = {0.0, 0.0, xn}, R[3], J[3][3], B[3][2];
  gtn_eval(m, g, u, R, J, B);
  bool conv = false;
  for (int it = 0; it < 50 && !conv; ++it) conv = gtn_newton_step(m, g, u, R, J, B);
  gtn_finish(m, g, u, n, tiny, epsp_n, conv, o);
}

// gf: the frozen porosity of a GTN phase (unused by the other models)
template <bool GTN>
__device__ void point_update(const Material& m, int has_field, const double* e, const double* epsp_n, double ep_n,
                             double hist, double abar, double D_override, double gf, PointOut& o) {
  const double K = m.E / (3.0 * (1.0 - 2.0 * m.nu));
  const double mu = m.E / (2.0 * (1.0 + m.nu));
  const double tr = e[0] + e[1] + e[2];
  const double de[6] = {e[0] - tr / 3.0, e[1] - tr / 3.0, e[2] - tr / 3.0, e[3], e[4], e[5]};
  o.alpha = 0.0;
  o.alpha2 = 0.0;
  o.fail = 0;
  o.ep = ep_n;
  for (int i = 0; i < 6; ++i) o.epsp[i] = epsp_n[i];
  if constexpr (GTN) {
    if (m.model == 3) {
      gtn_update(m, K, mu, e, epsp_n, ep_n, gf, o);
      return;
    }
  }
  if (m.model == 0) {
    elastic_C(K, mu, 1.0, o);
    for (int i = 0; i < 6; ++i) o.sig[i] = 2.0 * mu * de[i] + (i < 3 ? K * tr : 0.0);
  } else if (m.model == 1) {
    double D = 0.0;
    if (has_field) {
      const double ab = abar > 0.0 ? abar : 0.0;
      D = clamp01cap((ab - m.eps_c) / (m.eps_r - m.eps_c), m.d_max);
      D = D > hist ? D : hist;
    }
    if (D_override >= 0.0) D = D_override;
    double s_tr[6], q2 = 0.0;
    for (int i = 0; i < 6; ++i) {
      s_tr[i] = 2.0 * mu * (de[i] - epsp_n[i]);
      q2 += s_tr[i] * s_tr[i];
    }
    const double q = sqrt(q2);
    const double sq23 = 0.81649658092772603273;
    const double f = q - sq23 * (m.sigma_y + m.H * ep_n);
    const double w = 1.0 - D;
    if (f > 0.0) {
      const double dlam = f / (2.0 * mu + 2.0 * m.H / 3.0);
      double n[6];
      for (int i = 0; i < 6; ++i) {
        n[i] = s_tr[i] / q;
        o.epsp[i] = epsp_n[i] + dlam * n[i];
      }
      o.ep = ep_n + sq23 * dlam;
      const double theta = 1.0 - 2.0 * mu * dlam / q;
      const double thetab = 1.0 / (1.0 + m.H / (3.0 * mu)) - (1.0 - theta);
      // C = w [K 1x1 + 2 mu theta (I - 1x1/3) - 2 mu thetab n x n]
      o.ca = w * (K - 2.0 * mu * theta / 3.0);
      o.cb = w * 2.0 * mu * theta;
      o.cc = w * 2.0 * mu * thetab;
      for (int i = 0; i < 6; ++i) o.n[i] = n[i];
    } else {
      elastic_C(K, mu, w, o);
    }
    for (int i = 0; i < 6; ++i) o.sig[i] = w * (2.0 * mu * (de[i] - o.epsp[i]) + (i < 3 ? K * tr : 0.0));
    o.alpha = o.ep;
  } else {
    double kap = hist;
    if (has_field) kap = abar > kap ? abar : kap;
    double d = clamp01cap((kap - m.kappa0) / (m.kappa_f - m.kappa0), m.d_max);
    if (D_override >= 0.0) d = D_override;
    double ce[6], ee = 0.0;
    for (int i = 0; i < 6; ++i) {
      ce[i] = 2.0 * mu * de[i] + (i < 3 ? K * tr : 0.0);
      ee += e[i] * ce[i];
    }
    o.alpha = sqrt((ee > 0.0 ? ee : 0.0) / m.E);
    const double w = 1.0 - d;
    for (int i = 0; i < 6; ++i) o.sig[i] = w * ce[i];
    elastic_C(K, mu, w, o);
  }
}

struct KArgs {
  size_t nvox;
  const double* eps;
  const double* epsp_n;
  const double* ep_n;
  const double* hist;
  const double* abar;   // J * nvox: non-local fields the mechanics is frozen at
  const double* abar_n; // J * nvox: committed non-local fields (GTN porosity increments)
  const uint8_t* phase;
  double* sig;
  double* C;
  double* alpha;        // J * nvox
  DevScalars* sc;
  double* partials;
};

// frozen porosity of GTN voxel g from the fields (j: ebar0, j + 1: trbar) at ab against the committed ones
__device__ __forceinline__ double gtn_frozen_f(const Material& m, const double* ab, const double* abn, double fn,
                                               int j, size_t n, size_t g) {
  return gtn_porosity(fn, ab[(size_t)j * n + g], abn[(size_t)j * n + g], ab[(size_t)(j + 1) * n + g],
                      abn[(size_t)(j + 1) * n + g], m);
}

template <bool GTN>
__global__ void __launch_bounds__(256, GTN ? 2 : 1) k_constitutive(KArgs a, MatTable mt) {
  constexpr int NR = GTN ? 7 : 6;   // <sigma> sums (+ GTN return-mapping failures)
  double red[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) red[i] = 0.0;
  const size_t n = a.nvox;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n; g += (size_t)gridDim.x * blockDim.x) {
    const int q = a.phase[g];
    const Material& m = mt.m[q];
    const int j = mt.field_of[q];
    double e[6], ep6[6];
    for (int i = 0; i < 6; ++i) {
      e[i] = a.eps[i * n + g];
      ep6[i] = a.epsp_n[i * n + g];
    }
    const double abar = (j >= 0) ? a.abar[(size_t)j * n + g] : 0.0;
    double gf = 0.0;
    const bool gtn = GTN && m.model == 3;
    if (gtn) gf = gtn_frozen_f(m, a.abar, a.abar_n, a.hist[g], j, n, g);
    PointOut o;
    point_update<GTN>(m, j >= 0, e, ep6, a.ep_n[g], a.hist[g], abar, -1.0, gf, o);
    if constexpr (GTN) red[NR - 1] += (double)o.fail;
    for (int i = 0; i < 6; ++i) {
      a.sig[i * n + g] = o.sig[i];
      red[i] += o.sig[i];
    }
    for (int i = 0; i < 6; ++i) a.C[(size_t)i * n + g] = o.n[i];
    a.C[6 * n + g] = o.ca;
    a.C[7 * n + g] = o.cb;
    a.C[8 * n + g] = o.cc;
    for (int f = 0; f < mt.nfields; ++f)
      a.alpha[(size_t)f * n + g] = (f == j) ? o.alpha : ((gtn && f == j + 1) ? o.alpha2 : 0.0);
  }
  reduce_finalize<NR>(red, a.partials, a.sc, RED_STORE, 0);
}


// commit: recompute eps^p, eps_p at the converged strain with the non-local fields the last
// mechanics was frozen at (a.abar); history from the accepted new fields abar_new:
// D_n <- max(D_n, D(abar_new)), kappa_n <- max(kappa_n, abar_new), GTN f_n <- f(abar_new) (A-30)
template <bool GTN>
__global__ void __launch_bounds__(256) k_commit(KArgs a, MatTable mt, const double* abar_new, double* epsp_out,
                                                double* ep_out, double* hist_out) {
  const size_t n = a.nvox;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n; g += (size_t)gridDim.x * blockDim.x) {
    const int q = a.phase[g];
    const Material& m = mt.m[q];
    const int j = mt.field_of[q];
    double e[6], ep6[6];
    for (int i = 0; i < 6; ++i) {
      e[i] = a.eps[i * n + g];
      ep6[i] = a.epsp_n[i * n + g];
    }
    const double abar = (j >= 0) ? a.abar[(size_t)j * n + g] : 0.0;
    const bool gtn = GTN && m.model == 3;
    const double gf = gtn ? gtn_frozen_f(m, a.abar, a.abar_n, a.hist[g], j, n, g) : 0.0;
    PointOut o;
    point_update<GTN>(m, j >= 0, e, ep6, a.ep_n[g], a.hist[g], abar, 0.0, gf, o);
    for (int i = 0; i < 6; ++i) epsp_out[i * n + g] = o.epsp[i];
    ep_out[g] = o.ep;
    double h = a.hist[g];
    if (j >= 0) {
      const double an = abar_new[(size_t)j * n + g];
      if (m.model == 1) {
        const double ab = an > 0.0 ? an : 0.0;
        const double D = clamp01cap((ab - m.eps_c) / (m.eps_r - m.eps_c), m.d_max);
        h = D > h ? D : h;
      } else if (m.model == 2) {
        h = an > h ? an : h;
      } else if (gtn) {
        h = gtn_frozen_f(m, abar_new, a.abar_n, a.hist[g], j, n, g);
      }
    }
    hist_out[g] = h;
  }
}

// staggered ERR ingredients (A-02): max_{x,ij} |eps - eps_prev| (tensor components) via
// an order-independent atomicMax on the bit pattern, sums of eps (6), and per field
// sum (abar_new - abar_old)^2, sum abar_new^2.
__global__ void __launch_bounds__(256) k_err(size_t n, const double* eps, const double* eps_prev, int J,
                                             const double* abar_new, const double* abar_old,
                                             unsigned long long* maxbits, DevScalars* sc, double* partials) {
  double red[14];
  for (int i = 0; i < 14; ++i) red[i] = 0.0;
  double mx = 0.0;
  const double w[6] = {1.0, 1.0, 1.0, 0.70710678118654752440, 0.70710678118654752440, 0.70710678118654752440};
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n; g += (size_t)gridDim.x * blockDim.x) {
    for (int i = 0; i < 6; ++i) {
      const double e = eps[i * n + g];
      red[i] += e;
      const double d = fabs(e - eps_prev[i * n + g]) * w[i];
      mx = d > mx ? d : mx;
    }
    for (int f = 0; f < J; ++f) {
      const double an = abar_new[(size_t)f * n + g], ao = abar_old[(size_t)f * n + g];
      red[6 + 2 * f] += (an - ao) * (an - ao);
      red[7 + 2 * f] += an * an;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(mx));
  reduce_finalize<14>(red, partials, sc, RED_STORE, 16);
}

// compact [n0..n5, ca, cb, cc] -> packed upper triangle (21) of ca 1x1 + cb I - cc n x n
__global__ void k_expand_tangent(size_t n, const double* __restrict__ Cc, double* __restrict__ Cp) {
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n; g += (size_t)gridDim.x * blockDim.x) {
    double v[6];
    for (int i = 0; i < 6; ++i) v[i] = Cc[i * n + g];
    const double ca = Cc[6 * n + g], cb = Cc[7 * n + g], cc = Cc[8 * n + g];
    int t = 0;
    for (int i = 0; i < 6; ++i)
      for (int j = i; j < 6; ++j, ++t)
        Cp[(size_t)t * n + g] = (i < 3 && j < 3 ? ca : 0.0) + (i == j ? cb : 0.0) - cc * v[i] * v[j];
  }
}

__global__ void k_dot(size_t n, const double* a, const double* b, DevScalars* sc, double* partials, int op, int slot) {
  double red[1] = {0.0};
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n; g += (size_t)gridDim.x * blockDim.x)
    red[0] = fma(a[g], b[g], red[0]);
  reduce_finalize<1>(red, partials, sc, op, slot);
}

__global__ void k_axpy(size_t n, double* y, const double* x, double s) {
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n; g += (size_t)gridDim.x * blockDim.x)
    y[g] = fma(s, x[g], y[g]);
}

__global__ void k_guard_init(DevScalars* sc, double tol2) {
  sc->tol2 = tol2;
  sc->done = 0;
  sc->iters = 0;
}

// y += alpha x with alpha the device-resident Krylov step (final deferred CG solution update)
__global__ void k_axpy_alpha(size_t n, double* y, const double* x, const DevScalars* sc) {
  const double s = sc->alpha;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n; g += (size_t)gridDim.x * blockDim.x)
    y[g] = fma(s, x[g], y[g]);
}

// eps = eps_n + dE (uniform on strain-controlled components)
__global__ void k_init_iterate(size_t n, const double* eps_n, double* eps, const double* dE6) {
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < 6 * n; g += (size_t)gridDim.x * blockDim.x)
    eps[g] = eps_n[g] + dE6[g / n];
}

__global__ void k_phase_count(size_t n, const uint8_t* ph, unsigned long long* cnt, int nph, int* bad) {
  __shared__ unsigned long long s[kMaxPhases];
  if (threadIdx.x < kMaxPhases) s[threadIdx.x] = 0;
  __syncthreads();
  // warp-aggregated: one shared atomic per distinct phase id per warp and element round
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t g0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nround = (n + stride - 1) / stride;
  for (size_t k = 0; k < nround; ++k) {
    const size_t g = g0 + k * stride;
    const int q = g < n ? (int)ph[g] : -1;
    if (q >= nph) atomicExch(bad, 1);
    const unsigned same = __match_any_sync(0xffffffffu, q);
    if (q >= 0 && q < nph && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&s[q], (unsigned long long)__popc(same));
  }
  __syncthreads();
  if (threadIdx.x < nph) atomicAdd(&cnt[threadIdx.x], s[threadIdx.x]);
}

}  // namespace fgd

// ---------------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------------
namespace fgd {

static int ew_blocks(const fgd_ctx* c, size_t n) {
  size_t b = (n + 255) / 256;
  const size_t cap = 148 * 8;
  return (int)std::max<size_t>(1, std::min(b, cap));
}

static MatTable make_table(const fgd_ctx* c) {
  MatTable t{};
  for (int q = 0; q < kMaxPhases; ++q) {
    t.m[q] = c->mat[q];
    t.field_of[q] = -1;
  }
  for (int j = c->nfields - 1; j >= 0; --j) t.field_of[c->source_phase[j]] = j;   // first field of the phase
  t.nfields = c->nfields;
  return t;
}

#define FGD_CHECK_LAUNCH(ctx, name)                                                                      \
  do {                                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                                 \
    if (e_ != cudaSuccess) return set_err(ctx, FGD_ECUDA, std::string(name) + ": " + cudaGetErrorString(e_)); \
  } while (0)

bool has_gtn(const fgd_ctx* c) {
  for (int q = 0; q < c->nphases; ++q)
    if (c->mat[q].model == 3) return true;
  return false;
}

// every GTN phase needs two consecutive fields (eps0p, tr eps^p) sourced by it
static fgd_status check_gtn_fields(fgd_ctx* c, const MatTable& t) {
  for (int q = 0; q < c->nphases; ++q) {
    if (c->mat[q].model != 3) continue;
    const int j = t.field_of[q];
    if (j < 0 || j + 1 >= c->nfields || c->source_phase[j + 1] != q)
      return set_err(c, FGD_ESTATE, "GTN phase " + std::to_string(q) +
                                        " needs two consecutive non-local fields with source_phase = " +
                                        std::to_string(q) + " (eps0p, tr eps^p)");
  }
  return FGD_OK;
}

fgd_status launch_constitutive(fgd_ctx* c, const double* eps) {
  const int nb = ew_blocks(c, c->nvox);
  fgd_status s = ensure_partials(c, nb);
  if (s != FGD_OK) return s;
  const MatTable t = make_table(c);
  const bool gtn = has_gtn(c);
  if (gtn && (s = check_gtn_fields(c, t)) != FGD_OK) return s;
  KArgs a{c->nvox, eps, c->st_epsp, c->st_ep, c->st_hist, c->w_abar, c->st_abar, c->phase, c->w_sig, c->Cc,
          c->w_alpha, c->sc, c->partials};
  c->launches++;
  KTimer kt(c, KC_CONST);
  if (gtn) {
    k_constitutive<true><<<nb, 256, 0, c->stream>>>(a, t);
  } else {
    k_constitutive<false><<<nb, 256, 0, c->stream>>>(a, t);
  }
  FGD_CHECK_LAUNCH(c, "k_constitutive");
  return FGD_OK;
}

fgd_status launch_commit(fgd_ctx* c, const double* eps, const double* abar_new, double* epsp_out, double* ep_out,
                         double* hist_out) {
  const int nb = ew_blocks(c, c->nvox);
  KArgs a{c->nvox, eps, c->st_epsp, c->st_ep, c->st_hist, c->w_abar, c->st_abar, c->phase, nullptr, nullptr, nullptr,
          c->sc, nullptr};
  c->launches++;
  KTimer kt(c, KC_OTHER);
  if (has_gtn(c))
    k_commit<true><<<nb, 256, 0, c->stream>>>(a, make_table(c), abar_new, epsp_out, ep_out, hist_out);
  else
    k_commit<false><<<nb, 256, 0, c->stream>>>(a, make_table(c), abar_new, epsp_out, ep_out, hist_out);
  FGD_CHECK_LAUNCH(c, "k_commit");
  return FGD_OK;
}

fgd_status launch_err(fgd_ctx* c, const double* eps, const double* eps_prev, const double* abar_new,
                      const double* abar_old, unsigned long long* maxbits) {
  const int nb = ew_blocks(c, c->nvox);
  fgd_status s = ensure_partials(c, (size_t)nb * 14);
  if (s != FGD_OK) return s;
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_err<<<nb, 256, 0, c->stream>>>(c->nvox, eps, eps_prev, c->nfields, abar_new, abar_old, maxbits, c->sc,
                                   c->partials);
  FGD_CHECK_LAUNCH(c, "k_err");
  return FGD_OK;
}

fgd_status launch_dot(fgd_ctx* c, size_t n, const double* a, const double* b, int op, int slot) {
  const int nb = ew_blocks(c, n);
  fgd_status s = ensure_partials(c, nb);
  if (s != FGD_OK) return s;
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_dot<<<nb, 256, 0, c->stream>>>(n, a, b, c->sc, c->partials, op, slot);
  FGD_CHECK_LAUNCH(c, "k_dot");
  return FGD_OK;
}

fgd_status launch_axpy(fgd_ctx* c, size_t n, double* y, const double* x, double s) {
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_axpy<<<ew_blocks(c, n), 256, 0, c->stream>>>(n, y, x, s);
  FGD_CHECK_LAUNCH(c, "k_axpy");
  return FGD_OK;
}

fgd_status launch_guard_init(fgd_ctx* c, double tol2) {
  c->launches++;
  k_guard_init<<<1, 1, 0, c->stream>>>(c->sc, tol2);
  FGD_CHECK_LAUNCH(c, "k_guard_init");
  return FGD_OK;
}

fgd_status launch_axpy_alpha(fgd_ctx* c, size_t n, double* y, const double* x) {
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_axpy_alpha<<<ew_blocks(c, n), 256, 0, c->stream>>>(n, y, x, c->sc);
  FGD_CHECK_LAUNCH(c, "k_axpy_alpha");
  return FGD_OK;
}

fgd_status launch_init_iterate(fgd_ctx* c, const double* eps_n, double* eps, const double* dE6_dev) {
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_init_iterate<<<ew_blocks(c, 6 * c->nvox), 256, 0, c->stream>>>(c->nvox, eps_n, eps, dE6_dev);
  FGD_CHECK_LAUNCH(c, "k_init_iterate");
  return FGD_OK;
}

fgd_status launch_expand_tangent(fgd_ctx* c, const double* Cc, double* Cp) {
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_expand_tangent<<<ew_blocks(c, c->nvox), 256, 0, c->stream>>>(c->nvox, Cc, Cp);
  FGD_CHECK_LAUNCH(c, "k_expand_tangent");
  return FGD_OK;
}

fgd_status launch_phase_count(fgd_ctx* c, const uint8_t* ph, unsigned long long* cnt, int nph, int* bad) {
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_phase_count<<<ew_blocks(c, c->nvox), 256, 0, c->stream>>>(c->nvox, ph, cnt, nph, bad);
  FGD_CHECK_LAUNCH(c, "k_phase_count");
  return FGD_OK;
}

}  // namespace fgd
