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
};

__device__ __forceinline__ void elastic_C(double K, double mu, double f, PointOut& o) {
  // f (K 1x1 + 2 mu I_dev) = f (K - 2mu/3) 1x1 + f 2mu I
  o.ca = f * (K - 2.0 * mu / 3.0);
  o.cb = f * 2.0 * mu;
  o.cc = 0.0;
  for (int i = 0; i < 6; ++i) o.n[i] = 0.0;
}

__device__ void point_update(const Material& m, int has_field, const double* e, const double* epsp_n, double ep_n,
                             double hist, double abar, double D_override, PointOut& o) {
  const double K = m.E / (3.0 * (1.0 - 2.0 * m.nu));
  const double mu = m.E / (2.0 * (1.0 + m.nu));
  const double tr = e[0] + e[1] + e[2];
  const double de[6] = {e[0] - tr / 3.0, e[1] - tr / 3.0, e[2] - tr / 3.0, e[3], e[4], e[5]};
  o.alpha = 0.0;
  o.ep = ep_n;
  for (int i = 0; i < 6; ++i) o.epsp[i] = epsp_n[i];
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
  const double* abar;   // J * nvox
  const uint8_t* phase;
  double* sig;
  double* C;
  double* alpha;        // J * nvox
  DevScalars* sc;
  double* partials;
};

__global__ void __launch_bounds__(256) k_constitutive(KArgs a, MatTable mt) {
  double red[6] = {0, 0, 0, 0, 0, 0};
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
    PointOut o;
    point_update(m, j >= 0, e, ep6, a.ep_n[g], a.hist[g], abar, -1.0, o);
    for (int i = 0; i < 6; ++i) {
      a.sig[i * n + g] = o.sig[i];
      red[i] += o.sig[i];
    }
    for (int i = 0; i < 6; ++i) a.C[(size_t)i * n + g] = o.n[i];
    a.C[6 * n + g] = o.ca;
    a.C[7 * n + g] = o.cb;
    a.C[8 * n + g] = o.cc;
    for (int f = 0; f < mt.nfields; ++f) a.alpha[(size_t)f * n + g] = (f == j) ? o.alpha : 0.0;
  }
  reduce_finalize<6>(red, a.partials, a.sc, RED_STORE, 0);
}

// commit: recompute eps^p, eps_p at the converged strain; D_n <- max(D_n, D(abar)), kappa_n <- max
__global__ void __launch_bounds__(256) k_commit(KArgs a, MatTable mt, double* epsp_out, double* ep_out,
                                                double* hist_out) {
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
    PointOut o;
    point_update(m, j >= 0, e, ep6, a.ep_n[g], a.hist[g], abar, 0.0, o);
    for (int i = 0; i < 6; ++i) epsp_out[i * n + g] = o.epsp[i];
    ep_out[g] = o.ep;
    double h = a.hist[g];
    if (j >= 0) {
      if (m.model == 1) {
        const double ab = abar > 0.0 ? abar : 0.0;
        const double D = clamp01cap((ab - m.eps_c) / (m.eps_r - m.eps_c), m.d_max);
        h = D > h ? D : h;
      } else if (m.model == 2) {
        h = abar > h ? abar : h;
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
  for (int j = 0; j < c->nfields; ++j) t.field_of[c->source_phase[j]] = j;
  t.nfields = c->nfields;
  return t;
}

#define FGD_CHECK_LAUNCH(ctx, name)                                                                      \
  do {                                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                                 \
    if (e_ != cudaSuccess) return set_err(ctx, FGD_ECUDA, std::string(name) + ": " + cudaGetErrorString(e_)); \
  } while (0)

fgd_status launch_constitutive(fgd_ctx* c, const double* eps) {
  const int nb = ew_blocks(c, c->nvox);
  fgd_status s = ensure_partials(c, nb);
  if (s != FGD_OK) return s;
  KArgs a{c->nvox, eps, c->st_epsp, c->st_ep, c->st_hist, c->w_abar, c->phase, c->w_sig, c->Cc, c->w_alpha, c->sc,
          c->partials};
  c->launches++;
  KTimer kt(c, KC_CONST);
  k_constitutive<<<nb, 256, 0, c->stream>>>(a, make_table(c));
  FGD_CHECK_LAUNCH(c, "k_constitutive");
  return FGD_OK;
}

fgd_status launch_commit(fgd_ctx* c, const double* eps, double* epsp_out, double* ep_out, double* hist_out) {
  const int nb = ew_blocks(c, c->nvox);
  KArgs a{c->nvox, eps, c->st_epsp, c->st_ep, c->st_hist, c->w_abar, c->phase, nullptr, nullptr, nullptr, c->sc,
          nullptr};
  c->launches++;
  KTimer kt(c, KC_OTHER);
  k_commit<<<nb, 256, 0, c->stream>>>(a, make_table(c), epsp_out, ep_out, hist_out);
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
