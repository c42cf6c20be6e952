// The five HBM passes of a 3D real FFT round trip with the method's pointwise work fused in.
//
//   real  R[c][z][y][x]  --x-fwd (R2C, fused producer)-->  A[c][z][kx][y]
//                        --y-fwd (C2C)----------------->  B[c][kx][ky][z]
//                        --z (fwd C2C, spectral multiply, inv C2C) in place on B
//                        --y-inv (C2C)----------------->  A[c][z][kx][y]
//                        --x-inv (C2R, fused epilogue)->  R'[c][z][y][x]
//
// Every pass reads and writes whole lines that are contiguous in global memory on one side
// and TY/TZ-element contiguous chunks on the transposed side.  The spectral multiply of the
// z pass is either the Galerkin projection G^*(xi) (A-04/A-07/A-08) on 6 Mandel
// components or the Helmholtz preconditioner 1/(1 + <l^2>|k|^2) on 1 component;
// the 1/N of F^-1 is folded into it.  x-fwd producers: plain load, tangent contraction
// tau = C:p, the CG direction update p = r + beta p with p.Cp, or the PCG
// x/r update.  x-inv epilogues: store, or the CG update x += alpha p, r -= alpha q with r.r.
#include "reduce.cuh"

namespace fgd {

constexpr int kMaxThr = 384;

struct XArgs {
  int Ny, Nz, TY, Hx;
  size_t nvox;
  const double* in0;
  const double* in1;
  double* out0;
  double* io1;
  double* io2;
  const double* Cp;
  double2* spec;
  DevScalars* sc;
  double* partials;
  int red_op, red_slot;
};

// packed upper-triangle offsets of row i
__device__ __forceinline__ void tangent_apply(const double* __restrict__ Cp, size_t g, size_t n, const double* p,
                                              double* tau) {
  double c[21];
#pragma unroll
  for (int t = 0; t < 21; ++t) c[t] = __ldcs(Cp + (size_t)t * n + g);
  // rows: 0:{0..5}=c0..c5, 1:{1..5}=c6..c10, 2:{2..5}=c11..c14, 3:{3..5}=c15..c17, 4:{4,5}=c18,c19, 5:c20
  tau[0] = c[0] * p[0] + c[1] * p[1] + c[2] * p[2] + c[3] * p[3] + c[4] * p[4] + c[5] * p[5];
  tau[1] = c[1] * p[0] + c[6] * p[1] + c[7] * p[2] + c[8] * p[3] + c[9] * p[4] + c[10] * p[5];
  tau[2] = c[2] * p[0] + c[7] * p[1] + c[11] * p[2] + c[12] * p[3] + c[13] * p[4] + c[14] * p[5];
  tau[3] = c[3] * p[0] + c[8] * p[1] + c[12] * p[2] + c[15] * p[3] + c[16] * p[4] + c[17] * p[5];
  tau[4] = c[4] * p[0] + c[9] * p[1] + c[13] * p[2] + c[16] * p[3] + c[18] * p[4] + c[19] * p[5];
  tau[5] = c[5] * p[0] + c[10] * p[1] + c[14] * p[2] + c[17] * p[3] + c[19] * p[4] + c[20] * p[5];
}

template <int N, int NC, int MODE>
__global__ void __launch_bounds__(kMaxThr) k_xfwd(XArgs a, const double2* __restrict__ tw) {
  extern __shared__ double2 sm[];
  constexpr int LP = pad_len(N);
  const int TY = a.TY;
  const int y0 = blockIdx.x * TY;
  const int z = blockIdx.y;
  const size_t n = a.nvox;
  double* smd = reinterpret_cast<double*>(sm);
  double red[1] = {0.0};
  double beta = 0.0, alpha = 0.0;
  if (MODE == XF_TANGENT_CG) beta = a.sc->beta;
  if (MODE == XF_HELM_UPDATE) alpha = a.sc->alpha;
  for (int idx = threadIdx.x; idx < TY * N; idx += blockDim.x) {
    const int yy = idx / N, x = idx % N;
    const size_t g = ((size_t)z * a.Ny + y0 + yy) * N + x;
    double tau[NC];
    if (MODE == XF_PLAIN) {
#pragma unroll
      for (int c = 0; c < NC; ++c) tau[c] = a.in0[c * n + g];
    } else if (MODE == XF_TANGENT) {
      double p[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) p[c] = a.in0[c * n + g];
      tangent_apply(a.Cp, g, n, p, tau);
    } else if (MODE == XF_TANGENT_CG) {
      double p[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        p[c] = fma(beta, a.out0[c * n + g], a.in0[c * n + g]);
        a.out0[c * n + g] = p[c];
      }
      tangent_apply(a.Cp, g, n, p, tau);
#pragma unroll
      for (int c = 0; c < 6; ++c) red[0] = fma(p[c], tau[c], red[0]);
    } else if (MODE == XF_HELM_UPDATE) {
      const double pv = a.in0[g];
      a.out0[g] = fma(alpha, pv, a.out0[g]);
      const double r = fma(-alpha, a.in1[g], a.io1[g]);
      a.io1[g] = r;
      tau[0] = r;
      red[0] = fma(r, r, red[0]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int l = c * TY + yy;
      smd[(size_t)((l >> 1) * LP + PAD(x)) * 2 + (l & 1)] = tau[c];
    }
  }
  __syncthreads();
  const int nl = NC * TY / 2;
  fft_lines<N, false>(sm, nl, LP, tw);
  __syncthreads();
  const int Hx = N / 2 + 1;
  for (int idx = threadIdx.x; idx < NC * Hx * TY; idx += blockDim.x) {
    const int yy = idx % TY;
    const int rest = idx / TY;
    const int kx = rest % Hx, c = rest / Hx;
    const int l = c * TY + yy;
    const double2* line = sm + (size_t)(l >> 1) * LP;
    const double2 z1 = line[PAD(kx)];
    const double2 z2 = line[PAD((N - kx) & (N - 1))];
    double2 v;
    if ((l & 1) == 0)
      v = make_double2(0.5 * (z1.x + z2.x), 0.5 * (z1.y - z2.y));
    else
      v = make_double2(0.5 * (z1.y + z2.y), -0.5 * (z1.x - z2.x));
    a.spec[((size_t)(c * a.Nz + z) * Hx + kx) * a.Ny + y0 + yy] = v;
  }
  if (MODE == XF_TANGENT_CG || MODE == XF_HELM_UPDATE) reduce_finalize<1>(red, a.partials, a.sc, a.red_op, a.red_slot);
}

template <int N, int NC, int MODE>
__global__ void __launch_bounds__(kMaxThr) k_xinv(XArgs a, const double2* __restrict__ tw) {
  extern __shared__ double2 sm[];
  constexpr int LP = pad_len(N);
  const int TY = a.TY;
  const int y0 = blockIdx.x * TY;
  const int z = blockIdx.y;
  const size_t n = a.nvox;
  const int Hx = N / 2 + 1;
  const int hp = TY / 2;
  for (int idx = threadIdx.x; idx < NC * Hx * hp; idx += blockDim.x) {
    const int pp = idx % hp;
    const int rest = idx / hp;
    const int kx = rest % Hx, c = rest / Hx;
    const int yy = 2 * pp;
    const int m = c * hp + pp;
    const size_t base = ((size_t)(c * a.Nz + z) * Hx + kx) * a.Ny + y0 + yy;
    double2 A1 = a.spec[base], A2 = a.spec[base + 1];
    if (kx == 0 || kx == N / 2) {
      A1.y = 0.0;
      A2.y = 0.0;
    }
    double2* line = sm + (size_t)m * LP;
    line[PAD(kx)] = make_double2(A1.x - A2.y, A1.y + A2.x);
    if (kx > 0 && kx < N / 2) line[PAD(N - kx)] = make_double2(A1.x + A2.y, A2.x - A1.y);
  }
  __syncthreads();
  fft_lines<N, true>(sm, NC * hp, LP, tw);
  __syncthreads();
  const double* smd = reinterpret_cast<const double*>(sm);
  double red[1] = {0.0};
  double alpha = 0.0;
  if (MODE == XI_MECH_CG) alpha = a.sc->alpha;
  for (int idx = threadIdx.x; idx < TY * N; idx += blockDim.x) {
    const int yy = idx / N, x = idx % N;
    const size_t g = ((size_t)z * a.Ny + y0 + yy) * N + x;
    double q[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int l = c * TY + yy;
      q[c] = smd[(size_t)((l >> 1) * LP + PAD(x)) * 2 + (l & 1)];
    }
    if (MODE == XI_STORE || MODE == XI_STORE_RR) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        a.out0[c * n + g] = q[c];
        if (MODE == XI_STORE_RR) red[0] = fma(q[c], q[c], red[0]);
      }
    } else if (MODE == XI_MECH_CG) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double p = a.in1[c * n + g];
        a.io1[c * n + g] = fma(alpha, p, a.io1[c * n + g]);
        const double r = fma(-alpha, q[c], a.io2[c * n + g]);
        a.io2[c * n + g] = r;
        red[0] = fma(r, r, red[0]);
      }
    } else if (MODE == XI_HELM_Z) {
      a.out0[g] = q[0];
      red[0] = fma(a.in1[g], q[0], red[0]);
    }
  }
  if (MODE != XI_STORE) reduce_finalize<1>(red, a.partials, a.sc, a.red_op, a.red_slot);
}

template <int N, bool INV>
__global__ void __launch_bounds__(kMaxThr) k_ypass(double2* __restrict__ A, double2* __restrict__ B, int Nz, int Hx, int TZ,
                                                const double2* __restrict__ tw) {
  extern __shared__ double2 sm[];
  constexpr int LP = pad_len(N);
  const int z0 = blockIdx.x * TZ;
  const int kx = blockIdx.y;
  const int c = blockIdx.z;
  if (!INV) {
    for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
      const int zz = idx / N, y = idx % N;
      sm[zz * LP + PAD(y)] = A[((size_t)(c * Nz + z0 + zz) * Hx + kx) * N + y];
    }
  } else {
    for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
      const int zz = idx % TZ, ky = idx / TZ;
      sm[zz * LP + PAD(ky)] = B[((size_t)(c * Hx + kx) * N + ky) * Nz + z0 + zz];
    }
  }
  __syncthreads();
  fft_lines<N, INV>(sm, TZ, LP, tw);
  __syncthreads();
  if (!INV) {
    for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
      const int zz = idx % TZ, ky = idx / TZ;
      B[((size_t)(c * Hx + kx) * N + ky) * Nz + z0 + zz] = sm[zz * LP + PAD(ky)];
    }
  } else {
    for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
      const int zz = idx / N, y = idx % N;
      A[((size_t)(c * Nz + z0 + zz) * Hx + kx) * N + y] = sm[zz * LP + PAD(y)];
    }
  }
}

struct ZArgs {
  int Nx, Ny, Hx, TL, scheme;
  double h[3], L[3];
  double scale;
  double shift[6];
  int mask[6];
  double mean_ell2;
};

// e^{i theta} for frequency index m of an axis of length N (exact at quarter turns)
__device__ __forceinline__ double2 eith(const double2* __restrict__ tw, int m) {
  const double2 w = __ldg(&tw[m]);
  return make_double2(w.x, -w.y);
}

__device__ __forceinline__ void symbol(const ZArgs& a, int Nz, const double2* twx, const double2* twy,
                                       const double2* twz, int kx, int ky, int kz, double2* k) {
  if (a.scheme == 1) {
    const double2 ex = eith(twx, kx), ey = eith(twy, ky), ez = eith(twz, kz);
    const double2 dx = make_double2(ex.x - 1.0, ex.y), dy = make_double2(ey.x - 1.0, ey.y),
                  dz = make_double2(ez.x - 1.0, ez.y);
    const double2 cx = make_double2(ex.x + 1.0, ex.y), cy = make_double2(ey.x + 1.0, ey.y),
                  cz = make_double2(ez.x + 1.0, ez.y);
    k[0] = cscale(cmul(dx, cmul(cy, cz)), 0.25 / a.h[0]);
    k[1] = cscale(cmul(cx, cmul(dy, cz)), 0.25 / a.h[1]);
    k[2] = cscale(cmul(cx, cmul(cy, dz)), 0.25 / a.h[2]);
  } else {
    const int Ns[3] = {a.Nx, a.Ny, Nz};
    const int ms[3] = {kx, ky, kz};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      int m = ms[j];
      const int Nj = Ns[j];
      if ((Nj % 2 == 0) && m == Nj / 2) {
        k[j] = make_double2(0.0, 0.0);
      } else {
        if (m > Nj / 2) m -= Nj;
        k[j] = make_double2(0.0, 2.0 * 3.14159265358979323846 * m / a.L[j]);
      }
    }
  }
}

constexpr double kS2 = 1.41421356237309504880;
constexpr double kIS2 = 0.70710678118654752440;

template <int N, int NC, int MODE>
__global__ void __launch_bounds__(kMaxThr) k_zpass(double2* __restrict__ B, ZArgs a, const double2* __restrict__ twx,
                                                const double2* __restrict__ twy, const double2* __restrict__ tw) {
  extern __shared__ double2 sm[];
  constexpr int LP = pad_len(N);
  const int TL = a.TL;
  const int ky0 = blockIdx.x * TL;
  const int kx = blockIdx.y;
  const int Ny = a.Ny, Hx = a.Hx;
  for (int idx = threadIdx.x; idx < NC * TL * N; idx += blockDim.x) {
    const int kz = idx % N;
    const int rest = idx / N;
    const int ll = rest % TL, c = rest / TL;
    sm[(c * TL + ll) * LP + PAD(kz)] = B[((size_t)(c * Hx + kx) * Ny + ky0 + ll) * N + kz];
  }
  __syncthreads();
  fft_lines<N, false>(sm, NC * TL, LP, tw);
  __syncthreads();
  for (int idx = threadIdx.x; idx < TL * N; idx += blockDim.x) {
    const int kz = idx % N, ll = idx / N;
    const int ky = ky0 + ll;
    double2 k[3];
    symbol(a, N, twx, twy, tw, kx, ky, kz, k);
    const double k2 = k[0].x * k[0].x + k[0].y * k[0].y + k[1].x * k[1].x + k[1].y * k[1].y +
                      k[2].x * k[2].x + k[2].y * k[2].y;
    const bool dc = (kx == 0 && ky == 0 && kz == 0);
    if (MODE == Z_PRECOND) {
      double2* v = &sm[ll * LP + PAD(kz)];
      *v = cscale(*v, a.scale / (1.0 + a.mean_ell2 * k2));
    } else {
      double2 t6[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) t6[c] = sm[(c * TL + ll) * LP + PAD(kz)];
      double2 o[6];
      if (dc) {
#pragma unroll
        for (int c = 0; c < 6; ++c)
          o[c] = a.mask[c] ? cscale(make_double2(t6[c].x - a.shift[c], t6[c].y), a.scale) : make_double2(0.0, 0.0);
      } else if (k2 == 0.0) {
#pragma unroll
        for (int c = 0; c < 6; ++c) o[c] = make_double2(0.0, 0.0);
      } else {
        // T (symmetric) from Mandel
        const double2 T00 = t6[0], T11 = t6[1], T22 = t6[2];
        const double2 T12 = cscale(t6[3], kIS2), T02 = cscale(t6[4], kIS2), T01 = cscale(t6[5], kIS2);
        const double2 kc0 = conjg(k[0]), kc1 = conjg(k[1]), kc2 = conjg(k[2]);
        double2 t[3];
        t[0] = cadd(cadd(cmul(T00, kc0), cmul(T01, kc1)), cmul(T02, kc2));
        t[1] = cadd(cadd(cmul(T01, kc0), cmul(T11, kc1)), cmul(T12, kc2));
        t[2] = cadd(cadd(cmul(T02, kc0), cmul(T12, kc1)), cmul(T22, kc2));
        const double2 s = cadd(cadd(cmul(kc0, t[0]), cmul(kc1, t[1])), cmul(kc2, t[2]));
        const double inv = 1.0 / k2;
        const double2 hs = cscale(s, 0.5 * inv);
        double2 u[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) u[i] = cscale(csub(t[i], cmul(k[i], hs)), 2.0 * inv);
        // P_ij = (u_i k_j + k_i u_j)/2 ; Mandel out scaled by a.scale
        const double sc = a.scale;
        o[0] = cscale(cmul(u[0], k[0]), sc);
        o[1] = cscale(cmul(u[1], k[1]), sc);
        o[2] = cscale(cmul(u[2], k[2]), sc);
        o[3] = cscale(cadd(cmul(u[1], k[2]), cmul(k[1], u[2])), 0.5 * kS2 * sc);
        o[4] = cscale(cadd(cmul(u[0], k[2]), cmul(k[0], u[2])), 0.5 * kS2 * sc);
        o[5] = cscale(cadd(cmul(u[0], k[1]), cmul(k[0], u[1])), 0.5 * kS2 * sc);
      }
#pragma unroll
      for (int c = 0; c < 6; ++c) sm[(c * TL + ll) * LP + PAD(kz)] = o[c];
    }
  }
  __syncthreads();
  fft_lines<N, true>(sm, NC * TL, LP, tw);
  __syncthreads();
  for (int idx = threadIdx.x; idx < NC * TL * N; idx += blockDim.x) {
    const int kz = idx % N;
    const int rest = idx / N;
    const int ll = rest % TL, c = rest / TL;
    B[((size_t)(c * Hx + kx) * Ny + ky0 + ll) * N + kz] = sm[(c * TL + ll) * LP + PAD(kz)];
  }
}

// ---------------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------------
static int pow2_floor(long v) {
  int p = 1;
  while ((long)p * 2 <= v) p *= 2;
  return p;
}
static const size_t kSmemBudget = 56 * 1024;

static int choose_TY(int N, int NC, int Ny) {
  const int TPL = fft_TPL(N);
  long by_smem = (long)(2 * kSmemBudget) / ((long)NC * pad_len(N) * 16);
  long by_thr = (long)2 * kMaxThr / ((long)NC * TPL);
  int TY = pow2_floor(std::min(by_smem, by_thr));
  TY = std::min(TY, Ny);
  return std::max(TY, 2);
}
static int round32(int v) { return ((v + 31) / 32) * 32; }

template <typename K>
static fgd_status launch(fgd_ctx* c, K kernel, dim3 grid, int threads, size_t smem, const char* name) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string(name) + " smem attr: " + cudaGetErrorString(e));
  }
  c->launches++;
  return FGD_OK;
}

#define FGD_LAUNCH(ctx, kern, grid, thr, smem, ...)                                       \
  do {                                                                                    \
    fgd_status st_ = launch(ctx, kern, grid, thr, smem, #kern);                           \
    if (st_ != FGD_OK) return st_;                                                        \
    kern<<<grid, thr, smem, (ctx)->stream>>>(__VA_ARGS__);                                \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess) return set_err(ctx, FGD_ECUDA, std::string(#kern) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define FGD_DISPATCH_N(Nval, MACRO) \
  switch (Nval) {                   \
    case 4: MACRO(4); break;        \
    case 8: MACRO(8); break;        \
    case 16: MACRO(16); break;      \
    case 32: MACRO(32); break;      \
    case 64: MACRO(64); break;      \
    case 128: MACRO(128); break;    \
    case 256: MACRO(256); break;    \
    case 512: MACRO(512); break;    \
    default: return set_err(c, FGD_EINVAL, "unsupported FFT length"); \
  }

fgd_status launch_xfwd(fgd_ctx* c, int ncomp, int mode, const double* in0, const double* in1, double* out0,
                       const double* Cp, int red_op, int red_slot) {
  return launch_xfwd_io(c, ncomp, mode, in0, in1, out0, nullptr, Cp, red_op, red_slot);
}

fgd_status launch_xfwd_io(fgd_ctx* c, int ncomp, int mode, const double* in0, const double* in1, double* out0,
                          double* io1, const double* Cp, int red_op, int red_slot) {
  const int Nx = c->n[0], Ny = c->n[1], Nz = c->n[2];
  const int TY = choose_TY(Nx, ncomp, Ny);
  const int nl = ncomp * TY / 2;
  const int thr = std::min(kMaxThr, round32(nl * fft_TPL(Nx)));
  const size_t smem = (size_t)nl * pad_len(Nx) * sizeof(double2);
  dim3 grid(Ny / TY, Nz);
  XArgs a{Ny, Nz, TY, c->Hx, c->nvox, in0, in1, out0, io1, nullptr, Cp, c->specA, c->sc, c->partials, red_op, red_slot};
  if (red_op != RED_NONE) {
    fgd_status s = ensure_partials(c, (size_t)grid.x * grid.y);
    if (s != FGD_OK) return s;
    a.partials = c->partials;
  }
  const double2* tw = c->tabs.tw[ilog2(Nx)];
  KTimer kt(c, ncomp == 6 ? KC_XFWD6 : KC_XFWD1);
#define XF(NN)                                                                                   \
  if (ncomp == 6 && mode == XF_PLAIN) FGD_LAUNCH(c, (k_xfwd<NN, 6, XF_PLAIN>), grid, thr, smem, a, tw);            \
  else if (ncomp == 6 && mode == XF_TANGENT) FGD_LAUNCH(c, (k_xfwd<NN, 6, XF_TANGENT>), grid, thr, smem, a, tw);   \
  else if (ncomp == 6 && mode == XF_TANGENT_CG) FGD_LAUNCH(c, (k_xfwd<NN, 6, XF_TANGENT_CG>), grid, thr, smem, a, tw); \
  else if (ncomp == 1 && mode == XF_PLAIN) FGD_LAUNCH(c, (k_xfwd<NN, 1, XF_PLAIN>), grid, thr, smem, a, tw);       \
  else if (ncomp == 1 && mode == XF_HELM_UPDATE) FGD_LAUNCH(c, (k_xfwd<NN, 1, XF_HELM_UPDATE>), grid, thr, smem, a, tw); \
  else return set_err(c, FGD_EINVAL, "xfwd mode");
  FGD_DISPATCH_N(Nx, XF)
#undef XF
  return FGD_OK;
}

fgd_status launch_xinv(fgd_ctx* c, int ncomp, int mode, double* out0, double* io1, double* io2, const double* in1,
                       int red_op, int red_slot) {
  const int Nx = c->n[0], Ny = c->n[1], Nz = c->n[2];
  const int TY = choose_TY(Nx, ncomp, Ny);
  const int nl = ncomp * TY / 2;
  const int thr = std::min(kMaxThr, round32(nl * fft_TPL(Nx)));
  const size_t smem = (size_t)nl * pad_len(Nx) * sizeof(double2);
  dim3 grid(Ny / TY, Nz);
  XArgs a{Ny, Nz, TY, c->Hx, c->nvox, nullptr, in1, out0, io1, io2, nullptr, c->specA, c->sc, nullptr, red_op, red_slot};
  if (mode != XI_STORE) {
    fgd_status s = ensure_partials(c, (size_t)grid.x * grid.y);
    if (s != FGD_OK) return s;
    a.partials = c->partials;
  }
  const double2* tw = c->tabs.tw[ilog2(Nx)];
  KTimer kt(c, ncomp == 6 ? KC_XINV6 : KC_XINV1);
#define XI(NN)                                                                                   \
  if (ncomp == 6 && mode == XI_STORE) FGD_LAUNCH(c, (k_xinv<NN, 6, XI_STORE>), grid, thr, smem, a, tw);            \
  else if (ncomp == 6 && mode == XI_STORE_RR) FGD_LAUNCH(c, (k_xinv<NN, 6, XI_STORE_RR>), grid, thr, smem, a, tw); \
  else if (ncomp == 6 && mode == XI_MECH_CG) FGD_LAUNCH(c, (k_xinv<NN, 6, XI_MECH_CG>), grid, thr, smem, a, tw);   \
  else if (ncomp == 1 && mode == XI_STORE) FGD_LAUNCH(c, (k_xinv<NN, 1, XI_STORE>), grid, thr, smem, a, tw);       \
  else if (ncomp == 1 && mode == XI_STORE_RR) FGD_LAUNCH(c, (k_xinv<NN, 1, XI_STORE_RR>), grid, thr, smem, a, tw); \
  else if (ncomp == 1 && mode == XI_HELM_Z) FGD_LAUNCH(c, (k_xinv<NN, 1, XI_HELM_Z>), grid, thr, smem, a, tw);     \
  else return set_err(c, FGD_EINVAL, "xinv mode");
  FGD_DISPATCH_N(Nx, XI)
#undef XI
  return FGD_OK;
}

static int choose_TZ(int N, int Nz) {
  const int TPL = fft_TPL(N);
  long by_smem = (long)(80 * 1024) / ((long)pad_len(N) * 16);
  long by_thr = kMaxThr / TPL;
  int TZ = pow2_floor(std::min(std::min(by_smem, by_thr), 64L));
  return std::max(1, std::min(TZ, Nz));
}

static fgd_status launch_y(fgd_ctx* c, int ncomp, bool inv) {
  const int Ny = c->n[1], Nz = c->n[2];
  const int TZ = choose_TZ(Ny, Nz);
  const int thr = std::min(kMaxThr, round32(TZ * fft_TPL(Ny)));
  const size_t smem = (size_t)TZ * pad_len(Ny) * sizeof(double2);
  dim3 grid(Nz / TZ, c->Hx, ncomp);
  const double2* tw = c->tabs.tw[ilog2(Ny)];
  KTimer kt(c, inv ? (ncomp == 6 ? KC_YINV6 : KC_YINV1) : (ncomp == 6 ? KC_YFWD6 : KC_YFWD1));
#define YP(NN)                                                                                               \
  if (inv) FGD_LAUNCH(c, (k_ypass<NN, true>), grid, thr, smem, c->specA, c->specB, Nz, c->Hx, TZ, tw);     \
  else FGD_LAUNCH(c, (k_ypass<NN, false>), grid, thr, smem, c->specA, c->specB, Nz, c->Hx, TZ, tw);
  FGD_DISPATCH_N(Ny, YP)
#undef YP
  return FGD_OK;
}
fgd_status launch_yfwd(fgd_ctx* c, int ncomp) { return launch_y(c, ncomp, false); }
fgd_status launch_yinv(fgd_ctx* c, int ncomp) { return launch_y(c, ncomp, true); }

fgd_status launch_z(fgd_ctx* c, int ncomp, int mode, double scale, const double* dc_shift, double mean_ell2) {
  const int Ny = c->n[1], Nz = c->n[2];
  const int TPL = fft_TPL(Nz);
  long by_smem = (long)kSmemBudget / ((long)ncomp * pad_len(Nz) * 16);
  long by_thr = kMaxThr / ((long)ncomp * TPL);
  int TL = pow2_floor(std::max(1L, std::min(by_smem, by_thr)));
  TL = std::min(TL, Ny);
  if (Nz == 1) TL = std::min(Ny, 64);
  const int thr = std::min(kMaxThr, std::max(round32(ncomp * TL * TPL), round32(std::min(TL * Nz, 256))));
  const size_t smem = (size_t)ncomp * TL * pad_len(Nz) * sizeof(double2);
  dim3 grid(Ny / TL, c->Hx);
  ZArgs a{};
  a.Nx = c->n[0];
  a.Ny = Ny;
  a.Hx = c->Hx;
  a.TL = TL;
  a.scheme = c->scheme;
  for (int i = 0; i < 3; ++i) {
    a.h[i] = c->h[i];
    a.L[i] = c->L[i];
  }
  a.scale = scale;
  for (int i = 0; i < 6; ++i) {
    a.shift[i] = dc_shift ? dc_shift[i] : 0.0;
    a.mask[i] = c->stress_mask[i];
  }
  a.mean_ell2 = mean_ell2;
  const double2* twx = c->tabs.tw[ilog2(c->n[0])];
  const double2* twy = c->tabs.tw[ilog2(Ny)];
  const double2* twz = c->tabs.tw[ilog2(Nz)];
  KTimer kt(c, ncomp == 6 ? KC_Z6 : KC_Z1);
#define ZP(NN)                                                                                             \
  if (ncomp == 6 && mode == Z_PROJECT) FGD_LAUNCH(c, (k_zpass<NN, 6, Z_PROJECT>), grid, thr, smem, c->specB, a, twx, twy, twz); \
  else if (ncomp == 1 && mode == Z_PRECOND) FGD_LAUNCH(c, (k_zpass<NN, 1, Z_PRECOND>), grid, thr, smem, c->specB, a, twx, twy, twz); \
  else return set_err(c, FGD_EINVAL, "z mode");
  switch (Nz) {
    case 1: ZP(1); break;
    case 2: ZP(2); break;
    case 4: ZP(4); break;
    case 8: ZP(8); break;
    case 16: ZP(16); break;
    case 32: ZP(32); break;
    case 64: ZP(64); break;
    case 128: ZP(128); break;
    case 256: ZP(256); break;
    case 512: ZP(512); break;
    default: return set_err(c, FGD_EINVAL, "unsupported Nz");
  }
#undef ZP
  return FGD_OK;
}

}  // namespace fgd
