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
  int compact;
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

// Real line of N doubles <-> half spectrum X[0..N/2] through ONE complex FFT of length M = N/2
// (z[n] = x[2n] + i x[2n+1]):  X[k] = E_k + W^k O_k,  E_k = (Z_k + conj Z_{M-k})/2,
// O_k = -i (Z_k - conj Z_{M-k})/2,  W = e^{-2 pi i/N};  X[M-k] = conj(E_k - W^k O_k);
// X[0] = Re Z_0 + Im Z_0, X[M] = Re Z_0 - Im Z_0.  Inverse: Z''_k = A + i W^{-k} B,
// Z''_{M-k} = conj(A - i W^{-k} B), A = X_k + conj X_{M-k}, B = X_k - conj X_{M-k}; the unnormalised
// inverse FFT of Z'' is then x[2n] + i x[2n+1] (the 1/N is folded into the spectral multiply).
// A line holds M complex points (SWZ layout, xline(M) slots) plus the Nyquist slot at SWZ(l, M).
template <int N>
__device__ __forceinline__ void r2c_post(double2* line, int l, int k, const double2* __restrict__ twN) {
  constexpr int M = N / 2;
  if (k == 0) {
    const double2 z = line[SWZ(l, 0)];
    line[SWZ(l, 0)] = make_double2(z.x + z.y, 0.0);
    line[SWZ(l, M)] = make_double2(z.x - z.y, 0.0);
    return;
  }
  const double2 zk = line[SWZ(l, k)], zm = line[SWZ(l, M - k)];
  const double2 E = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
  const double2 O = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
  const double2 WO = cmul(__ldg(&twN[k]), O);
  line[SWZ(l, k)] = cadd(E, WO);
  if (k != M - k) line[SWZ(l, M - k)] = conjg(csub(E, WO));
}

// compact tangent (constitutive.cu): tau = ca tr(p) 1 + cb p - cc (n.p) n
__device__ __forceinline__ void tangent_apply_c(const double* __restrict__ Cc, size_t g, size_t n, const double* p,
                                                double* tau) {
  double v[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) v[i] = __ldcs(Cc + (size_t)i * n + g);
  const double ca = __ldcs(Cc + 6 * n + g), cb = __ldcs(Cc + 7 * n + g), cc = __ldcs(Cc + 8 * n + g);
  const double tr = ca * (p[0] + p[1] + p[2]);
  double np = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) np = fma(v[i], p[i], np);
  np *= cc;
#pragma unroll
  for (int i = 0; i < 6; ++i) tau[i] = fma(cb, p[i], fma(-np, v[i], i < 3 ? tr : 0.0));
}

template <int N, int NC, int MODE>
__global__ void __launch_bounds__(kMaxThr, 2) k_xfwd(XArgs a, const double2* __restrict__ twM,
                                                      const double2* __restrict__ twN) {
  extern __shared__ double2 sm[];
  constexpr int M = N / 2;
  constexpr int LP = xline(M);
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
      for (int c = 0; c < NC; ++c) tau[c] = __ldcs(a.in0 + c * n + g);
    } else if (MODE == XF_TANGENT) {
      double p[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) p[c] = a.in0[c * n + g];
      if (a.compact) tangent_apply_c(a.Cp, g, n, p, tau);
      else tangent_apply(a.Cp, g, n, p, tau);
    } else if (MODE == XF_TANGENT_CG) {
      double p[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) p[c] = fma(beta, a.out0[c * n + g], a.in0[c * n + g]);
#pragma unroll
      for (int c = 0; c < 6; ++c) a.out0[c * n + g] = p[c];
      if (a.compact) tangent_apply_c(a.Cp, g, n, p, tau);
      else tangent_apply(a.Cp, g, n, p, tau);
#pragma unroll
      for (int c = 0; c < 6; ++c) red[0] = fma(p[c], tau[c], red[0]);
    } else if (MODE == XF_HELM_UPDATE) {
      const double pv = a.in0[g], qv = a.in1[g], xv = a.out0[g], rv = a.io1[g];
      a.out0[g] = fma(alpha, pv, xv);
      const double r = fma(-alpha, qv, rv);
      a.io1[g] = r;
      tau[0] = r;
      red[0] = fma(r, r, red[0]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) smd[(size_t)((c * TY + yy) * LP + SWZ(c * TY + yy, x >> 1)) * 2 + (x & 1)] = tau[c];
  }
  const int nl = NC * TY;
  double2* tws = sm + (size_t)nl * LP;
  build_pass_tables<M>(tws, twM);
  __syncthreads();
  fft_lines<M, false>(sm, nl, LP, tws);
  __syncthreads();
  for (int idx = threadIdx.x; idx < nl * (M / 2 + 1); idx += blockDim.x) {
    const int k = idx % (M / 2 + 1), l = idx / (M / 2 + 1);
    r2c_post<N>(sm + (size_t)l * LP, l, k, twN);
  }
  __syncthreads();
  const int Hx = M + 1;
#pragma unroll 4
  for (int idx = threadIdx.x; idx < NC * Hx * TY; idx += blockDim.x) {
    const int yy = idx % TY;
    const int rest = idx / TY;
    const int kx = rest % Hx, c = rest / Hx;
    a.spec[((size_t)(c * a.Nz + z) * Hx + kx) * a.Ny + y0 + yy] = sm[(c * TY + yy) * LP + SWZ(c * TY + yy, kx)];
  }
  if (MODE == XF_TANGENT_CG || MODE == XF_HELM_UPDATE) reduce_finalize<1>(red, a.partials, a.sc, a.red_op, a.red_slot);
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
  // NC*TY real lines per CTA, each an FFT of length N/2 plus the Nyquist slot
  const int M = N / 2;
  const int TPL = fft_TPL(M);
  long by_smem = (long)kSmemBudget / ((long)NC * xline(M) * 16);
  long by_thr = (long)kMaxThr / ((long)NC * TPL);
  int TY = pow2_floor(std::max(1L, std::min(by_smem, by_thr)));
  TY = std::min(TY, Ny);
  return std::max(TY, 1);
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
  if (mode == XF_PLAIN && ((uintptr_t)in0 & 15) == 0) return pipe_xfwd_plain(c, ncomp, in0);
  const int Nx = c->n[0], Ny = c->n[1], Nz = c->nz_l;
  const int TY = choose_TY(Nx, ncomp, Ny);
  const int nl = ncomp * TY;
  const int thr = std::min(kMaxThr, std::max(64, round32(nl * fft_TPL(Nx / 2))));
  const size_t smem = ((size_t)nl * xline(Nx / 2) + Nx / 2) * sizeof(double2);
  dim3 grid(Ny / TY, Nz);
  XArgs a{Ny, Nz, TY, c->Hx, c->nvox, in0, in1, out0, io1, nullptr, Cp, c->specA, c->sc, c->partials, red_op, red_slot,
          (Cp != nullptr && Cp == c->Cc) ? 1 : 0};
  if (red_op != RED_NONE) {
    fgd_status s = ensure_partials(c, (size_t)grid.x * grid.y);
    if (s != FGD_OK) return s;
    a.partials = c->partials;
  }
  const double2* tw = c->tabs.tw[ilog2(Nx / 2)];
  const double2* twN = c->tabs.tw[ilog2(Nx)];
  KTimer kt(c, ncomp == 6 ? KC_XFWD6 : KC_XFWD1);
#define XF(NN)                                                                                   \
  if (ncomp == 6 && mode == XF_PLAIN) FGD_LAUNCH(c, (k_xfwd<NN, 6, XF_PLAIN>), grid, thr, smem, a, tw, twN);            \
  else if (ncomp == 6 && mode == XF_TANGENT) FGD_LAUNCH(c, (k_xfwd<NN, 6, XF_TANGENT>), grid, thr, smem, a, tw, twN);   \
  else if (ncomp == 6 && mode == XF_TANGENT_CG) FGD_LAUNCH(c, (k_xfwd<NN, 6, XF_TANGENT_CG>), grid, thr, smem, a, tw, twN); \
  else if (ncomp == 1 && mode == XF_PLAIN) FGD_LAUNCH(c, (k_xfwd<NN, 1, XF_PLAIN>), grid, thr, smem, a, tw, twN);       \
  else if (ncomp == 1 && mode == XF_HELM_UPDATE) FGD_LAUNCH(c, (k_xfwd<NN, 1, XF_HELM_UPDATE>), grid, thr, smem, a, tw, twN); \
  else return set_err(c, FGD_EINVAL, "xfwd mode");
  FGD_DISPATCH_N(Nx, XF)
#undef XF
  return FGD_OK;
}

fgd_status launch_xinv(fgd_ctx* c, int ncomp, int mode, double* out0, double* io1, double* io2, const double* in1,
                       int red_op, int red_slot) {
  return pipe_xinv(c, ncomp, mode, out0, io1, io2, in1, red_op, red_slot);
}

fgd_status launch_yfwd(fgd_ctx* c, int ncomp) { return pipe_y(c, ncomp, false); }
fgd_status launch_yinv(fgd_ctx* c, int ncomp) { return pipe_y(c, ncomp, true); }

fgd_status launch_z(fgd_ctx* c, int ncomp, int mode, double scale, const double* dc_shift, double mean_ell2) {
  return pipe_z(c, ncomp, mode, scale, dc_shift, mean_ell2);
}

}  // namespace fgd
