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
#include <cstdlib>

#include "reduce.cuh"
#include "tma.cuh"

namespace fgd {

constexpr int kMaxThr = 384;

struct XArgs {
  const DevScalars* guard;
  int Ny, Nz, TY, HxA;   // HxA: kx stride of layout A
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
__device__ __forceinline__ void r2c_post(double2* line, int l, int k, const double2* twN) {
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
  const double2 WO = cmul(twN[k], O);   // twN: global or shared table
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
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
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
  if (MODE == XF_TANGENT_CG) {
    beta = a.sc->beta;
    alpha = a.sc->alpha;
  }
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
      // CG with the solution update one step late: x += alpha_{k-1} p_{k-1} here (p_{k-1} is read
      // anyway), so that the inverse pass only touches r.  cg_mech adds the last alpha p at the end.
      double p[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const double po = a.out0[c * n + g];
        a.io1[c * n + g] = fma(alpha, po, a.io1[c * n + g]);
        p[c] = fma(beta, po, a.in0[c * n + g]);
      }
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
  constexpr int NB = (Hx + kKB - 1) / kKB;
#pragma unroll 4
  for (int idx = threadIdx.x; idx < NC * NB * TY * kKB; idx += blockDim.x) {
    // order (kx % kKB, yy, kx / kKB, c): runs of TY * kKB contiguous elements of layout A
    const int kl = idx % kKB, yy = (idx / kKB) % TY, rest = idx / (kKB * TY);
    const int kx = (rest % NB) * kKB + kl, c = rest / NB;
    if (kx < Hx) a.spec[aidx(a.HxA, a.Ny, a.Nz, c, z, y0 + yy, kx)] = sm[(c * TY + yy) * LP + SWZ(c * TY + yy, kx)];
  }
  if (MODE == XF_TANGENT_CG || MODE == XF_HELM_UPDATE) reduce_finalize<1>(red, a.partials, a.sc, a.red_op, a.red_slot);
}

// ---------------------------------------------------------------------------------------------
// Tangent x-forward pass as a persistent bulk-copy (TMA) pipeline
// ---------------------------------------------------------------------------------------------
// A tile is a pair of rows (z, y = 2 yb + {0, 1}) -- the kXR rows of one block of layout A.  The
// producer operands of a row chunk (CW voxels: r, p, x and the tangent for the CG step; p and the
// tangent for the plain apply) arrive in a ring of S shared-memory stages by 1-D bulk copies, one
// per operand row, completing on the stage's mbarrier; S - 1 chunks are in flight while one is
// consumed.  The consumer updates x and p (CG), contracts tau = C p voxel by voxel into the FFT
// buffer (12 lines: 6 components x 2 rows), and after the last chunk of the pair runs the R2C
// line transforms and stores the half spectra as one contiguous block per component.
struct XTArgs {
  const DevScalars* guard;
  int Ny, Nz, HxA, CW, S, R;   // chunk width, stages, rows per tile
  int first;                   // CG step 1: p = r, x = 0 (p_old and x are neither read nor needed)
  size_t nvox;
  double* r;           // CG: residual (in)                      HELM: r (in/out)
  double* p;           // CG: direction (in/out); TANGENT: operand  HELM: p (in)
  double* x;           // CG: solution (in/out, one step late)    HELM: x (in/out)
  const double* C;     // tangent, 9 (compact) or 21 (packed) rows  HELM: q (in)
  double2* spec;
  DevScalars* sc;
  double* partials;
  int red_op, red_slot;
  const double2* twM;
  const double2* twN;
};

template <int MODE>
__host__ __device__ constexpr int xt_nc() { return MODE == XF_HELM_UPDATE ? 1 : 6; }
template <int MODE, bool CMP>
__host__ __device__ constexpr int xt_rows() {
  return MODE == XF_HELM_UPDATE ? 4 : (MODE == XF_TANGENT_CG ? 18 : 6) + (CMP ? 9 : 21);
}
// rows per tile: a pair for the 6-component passes (12 lines), 8 rows (4 if Ny = 4) for the
// 1-component PCG pass
template <int N>
__host__ __device__ constexpr size_t xt_fixed_bytes(int nlines) {
  return 64 + ((size_t)nlines * xline(N / 2) + N / 2 + N + 240) * sizeof(double2);
}

// tau = C p with the tangent rows in shared memory (stride cs between rows)
template <bool CMP>
__device__ __forceinline__ void tangent_smem(const double* C, int v, int cs, const double* p, double* tau) {
  if (CMP) {
    double nv[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) nv[i] = C[i * cs + v];
    const double ca = C[6 * cs + v], cb = C[7 * cs + v], cc = C[8 * cs + v];
    const double tr = ca * (p[0] + p[1] + p[2]);
    double np = 0.0;
#pragma unroll
    for (int i = 0; i < 6; ++i) np = fma(nv[i], p[i], np);
    np *= cc;
#pragma unroll
    for (int i = 0; i < 6; ++i) tau[i] = fma(cb, p[i], fma(-np, nv[i], i < 3 ? tr : 0.0));
  } else {
    double c[21];
#pragma unroll
    for (int t = 0; t < 21; ++t) c[t] = C[t * cs + v];
    tau[0] = c[0] * p[0] + c[1] * p[1] + c[2] * p[2] + c[3] * p[3] + c[4] * p[4] + c[5] * p[5];
    tau[1] = c[1] * p[0] + c[6] * p[1] + c[7] * p[2] + c[8] * p[3] + c[9] * p[4] + c[10] * p[5];
    tau[2] = c[2] * p[0] + c[7] * p[1] + c[11] * p[2] + c[12] * p[3] + c[13] * p[4] + c[14] * p[5];
    tau[3] = c[3] * p[0] + c[8] * p[1] + c[12] * p[2] + c[15] * p[3] + c[16] * p[4] + c[17] * p[5];
    tau[4] = c[4] * p[0] + c[9] * p[1] + c[13] * p[2] + c[16] * p[3] + c[18] * p[4] + c[19] * p[5];
    tau[5] = c[5] * p[0] + c[10] * p[1] + c[14] * p[2] + c[17] * p[3] + c[19] * p[4] + c[20] * p[5];
  }
}

template <int N, int MODE, bool CMP, int R>
__global__ void __launch_bounds__(256) k_xtan(XTArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  constexpr int M = N / 2, Hx = M + 1;
  constexpr int LP = xline(M);
  constexpr int NC = xt_nc<MODE>();
  constexpr int NOP = xt_rows<MODE, CMP>();
  constexpr int C0 = MODE == XF_TANGENT_CG ? 18 : 6;   // first tangent row
  // R: rows per tile; line l = c * R + row
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw);                  // [S], S <= 8
  double2* fb = reinterpret_cast<double2*>(smraw + 64);                // FFT buffer: NC * R lines of LP
  double2* twM = fb + (size_t)NC * R * LP;
  double2* twN = twM + M;
  double2* twR = twN + N;                                              // [240] register-FFT twiddles
  double* stg = reinterpret_cast<double*>(twR + 240);                  // [S][NOP][CW]
  const int CW = a.CW, S = a.S;
  const int nch = N / CW;
  const int ntiles = a.Nz * (a.Ny / R);
  const size_t n = a.nvox;
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  build_pass_tables<M>(twM, a.twM);
  load_table(twN, a.twN, N);
  if constexpr (fft_reg_ok<M>()) fft_reg_tables<M>(twR, a.twM);
  __syncthreads();
  pdl_wait();
  const int myrows = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // chunk q: tile t = blockIdx.x + (q / (R nch)) gridDim.x, row rr = (q / nch) % R, part h = q % nch
  const int nq = myrows * nch * R;
  auto issue = [&](int q) {      // warp 0
    const int t = blockIdx.x + (q / (R * nch)) * gridDim.x, rr = (q / nch) % R, h = q % nch;
    const size_t g0 = ((size_t)t * R + rr) * N + (size_t)h * CW;   // row z Ny + R yb + rr
    double* dst = stg + (size_t)(q % S) * NOP * CW;
    uint64_t* bar = &bars[q % S];
    const unsigned bytes = CW * 8;
    const bool skip_px = MODE == XF_TANGENT_CG && a.first;   // rows 6..17 (p_old, x) not needed
    if (threadIdx.x == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, bytes * (skip_px ? NOP - 12 : NOP));
    }
    __syncwarp();
    for (int i = threadIdx.x; i < NOP; i += 32) {
      if (skip_px && i >= 6 && i < 18) continue;
      const double* src;
      if (MODE == XF_TANGENT_CG)
        src = i < 6 ? a.r + i * n : i < 12 ? a.p + (i - 6) * n : i < 18 ? a.x + (i - 12) * n : a.C + (i - 18) * n;
      else if (MODE == XF_TANGENT)
        src = i < 6 ? a.p + i * n : a.C + (i - 6) * n;
      else   // HELM: p, q, x, r
        src = i == 0 ? a.p : i == 1 ? a.C : i == 2 ? a.x : a.r;
      bulk_g2s(dst + (size_t)i * CW, src + g0, bytes, bar);
    }
  };
  if (threadIdx.x < 32)
    for (int q = 0; q < S - 1 && q < nq; ++q) issue(q);
  double beta = 0.0, alpha = 0.0;
  if (MODE == XF_TANGENT_CG) beta = a.sc->beta;
  if (MODE == XF_TANGENT_CG || MODE == XF_HELM_UPDATE) alpha = a.sc->alpha;
  double red = 0.0;
  double* fbd = reinterpret_cast<double*>(fb);
  // chunk coordinates (tile t, row rr, part h), stage and mbarrier phase advance incrementally: a thread
  // consumes one voxel per chunk when CW = blockDim.x, so per-chunk divisions are per-voxel work
  int t = blockIdx.x, rr = 0, h = 0, sq = 0;
  unsigned ph = 0;
  for (int q = 0; q < nq; ++q) {
    // refill the stage consumed at q - 1 (released by the barriers at the end of that iteration)
    if (threadIdx.x < 32 && q + S - 1 < nq) issue(q + S - 1);
    mbar_wait(&bars[sq], ph);
    const double* st = stg + (size_t)sq * NOP * CW;
    for (int v = threadIdx.x; v < CW; v += blockDim.x) {
      const int xg = h * CW + v;
      const size_t g = ((size_t)t * R + rr) * N + xg;
      double tau[NC];
      if (MODE == XF_HELM_UPDATE) {
        // PCG update (real space, A-10 / R-PCG): x += alpha p, r -= alpha q; tau = r; r.r
        a.x[g] = fma(alpha, st[v], st[2 * CW + v]);
        const double rn = fma(-alpha, st[CW + v], st[3 * CW + v]);
        a.r[g] = rn;
        tau[0] = rn;
        red = fma(rn, rn, red);
      } else {
        double p[6], tv[6];
        if (MODE == XF_TANGENT_CG) {
          // CG with the solution update one step late (x += alpha_{k-1} p_{k-1}); see cg_mech
          if (a.first) {
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              a.x[c * n + g] = 0.0;
              p[c] = st[c * CW + v];
              a.p[c * n + g] = p[c];
            }
          } else {
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              const double po = st[(6 + c) * CW + v];
              a.x[c * n + g] = fma(alpha, po, st[(12 + c) * CW + v]);
              p[c] = fma(beta, po, st[c * CW + v]);
              a.p[c * n + g] = p[c];
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 6; ++c) p[c] = st[c * CW + v];
        }
        tangent_smem<CMP>(st + C0 * CW, v, CW, p, tv);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          tau[c] = tv[c];
          if (MODE == XF_TANGENT_CG) red = fma(p[c], tv[c], red);
        }
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int l = c * R + rr;
        fbd[(size_t)(l * LP + SWZ(l, xg >> 1)) * 2 + (xg & 1)] = tau[c];
      }
    }
    __syncthreads();
    if (rr == R - 1 && h == nch - 1) {
      if constexpr (fft_reg_ok<M>()) {
        constexpr int TPT = fft_reg_tpl<M>();
        // fft_reg_inplace synchronises with full-warp __syncwarp(): whole warps must take part
        static_assert((NC * R * TPT) % 32 == 0, "register x FFT needs whole warps of lines");
        for (int base = 0; base < NC * R * TPT; base += blockDim.x) {
          const int id = base + threadIdx.x;
          if (id < NC * R * TPT) fft_reg_inplace<M, false>(fb + (size_t)(id / TPT) * LP, id / TPT, id % TPT, twR);
        }
      } else {
        fft_lines<M, false>(fb, NC * R, LP, twM);
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < NC * R * (M / 2 + 1); idx += blockDim.x) {
        const int k = idx % (M / 2 + 1), l = idx / (M / 2 + 1);
        r2c_post<N>(fb + (size_t)l * LP, l, k, twN);
      }
      __syncthreads();
      const int z = t / (a.Ny / R), y0 = (t % (a.Ny / R)) * R;
      constexpr int NB = (Hx + kKB - 1) / kKB;   // kx blocks holding data
      if constexpr (R == kXR && kKB == 2 && kXR == 2) {
        // order (kx % 2, row, kx / 2, c): runs of 4 contiguous elements (64 B) of layout A.  Thread tid
        // owns (kl, r2) = (tid & 1, (tid >> 1) & 1) and the kx blocks tid / 4 + j blockDim / 4: the
        // address is one base per tile plus constant steps (no per-element index arithmetic)
        constexpr int THR = N >= 512 ? 256 : 128, KS = THR / 4, NJ = (NB + KS - 1) / KS;   // blockDim.x == THR
        const int kl = threadIdx.x & 1, r2 = (threadIdx.x >> 1) & 1, kb0 = threadIdx.x >> 2;
        const size_t cstep = (size_t)a.Nz * (a.HxA / kKB) * a.Ny * kKB, kstep = (size_t)KS * a.Ny * kKB;
        double2* g0 = a.spec + (((size_t)z * (a.HxA / kKB) + kb0) * a.Ny + y0 + r2) * kKB + kl;
        // all loads of a thread first, then its stores (only the last kx block column can fall past Hx)
        const bool last = (kb0 + (NJ - 1) * KS) * kKB + kl < Hx;
        double2 val[NC][NJ];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int l = c * R + r2;
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (j < NJ - 1 || last) val[c][j] = fb[l * LP + SWZ(l, (kb0 + j * KS) * kKB + kl)];
        }
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (j < NJ - 1 || last) g0[c * cstep + j * kstep] = val[c][j];
      } else {
        for (int idx = threadIdx.x; idx < NC * NB * R * kKB; idx += blockDim.x) {
          // order (kx % kKB, row, kx / kKB, c): runs of R * kKB contiguous elements
          const int kl = idx % kKB, r2 = (idx / kKB) % R, kb = (idx / (kKB * R)) % NB, c = idx / (kKB * R * NB);
          const int kx = kb * kKB + kl, l = c * R + r2;
          if (kx < Hx) a.spec[aidx(a.HxA, a.Ny, a.Nz, c, z, y0 + r2, kx)] = fb[l * LP + SWZ(l, kx)];
        }
      }
      __syncthreads();
    }
    if (++h == nch) {
      h = 0;
      if (++rr == R) {
        rr = 0;
        t += gridDim.x;
      }
    }
    if (++sq == S) {
      sq = 0;
      ph ^= 1u;
    }
  }
  if (MODE == XF_TANGENT_CG || MODE == XF_HELM_UPDATE) {
    double rr2[1] = {red};
    reduce_finalize<1>(rr2, a.partials, a.sc, a.red_op, a.red_slot);
  }
}

// ---------------------------------------------------------------------------------------------
// Ping-pong variant of k_xtan for N = 512 (6-component tangent passes): one 512-thread CTA per SM
// made of two groups of 256 threads that take alternate tiles, each with its own FFT buffer, and
// share the ring of two 256-voxel stages.  k_xtan runs its phases one after the other (consume the
// four chunks of a row pair -> register FFTs -> R2C post-processing -> spectrum stores), so the copy
// pipeline idles through the FFT/store phase; here one group's FFT/store phase overlaps the other
// group's consumption.  Chunk q = 4 i + j belongs to local tile i (group i & 1), lives in stage
// j & 1 and completes on the owner group's mbarrier full[i & 1][j & 1] (a group only ever waits on
// its own barriers, so their phase parity stays in step with the group); the group that has
// consumed chunk q refills the stage with chunk q + 2 after its group barrier.  Group-local
// synchronisation uses named barriers 1 + group; the FFT twiddles of the R2C post-processing come
// from the global table (L1) instead of shared memory, which is what lets two FFT buffers fit.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void group_bar(int grp) { asm volatile("bar.sync %0, 256;" ::"r"(1 + grp) : "memory"); }

template <int N, int MODE, bool CMP>
constexpr size_t xtpp_smem() {
  return 64 + ((size_t)2 * 6 * kXR * xline(N / 2) + 240) * sizeof(double2) + (size_t)2 * xt_rows<MODE, CMP>() * 256 * 8;
}

template <int N, int MODE, bool CMP>
__global__ void __launch_bounds__(512, 1) k_xtan_pp(XTArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  static_assert(MODE == XF_TANGENT_CG || MODE == XF_TANGENT, "6-component tangent passes only");
  constexpr int M = N / 2, Hx = M + 1, LP = xline(M), NC = 6, R = kXR, GT = 256, CW = 256, S = 2;
  constexpr int NOP = xt_rows<MODE, CMP>();
  constexpr int C0 = MODE == XF_TANGENT_CG ? 18 : 6;   // first tangent row
  constexpr int nch = N / CW, CPT = nch * R;           // chunks per tile
  static_assert(fft_reg_ok<M>() && CPT % S == 0, "register x FFT, stage parity fixed per chunk slot");
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw);                  // full[group][stage]
  double2* fb0 = reinterpret_cast<double2*>(smraw + 64);               // FFT buffers: 2 x NC * R lines of LP
  double2* twR = fb0 + (size_t)2 * NC * R * LP;                        // [240] register-FFT twiddles
  double* stg = reinterpret_cast<double*>(twR + 240);                  // [S][NOP][CW]
  const int grp = threadIdx.x >> 8, gt = threadIdx.x & (GT - 1);
  double2* fb = fb0 + (size_t)grp * NC * R * LP;
  double* fbd = reinterpret_cast<double*>(fb);
  const int ntiles = a.Nz * (a.Ny / R);
  const size_t n = a.nvox;
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2 * S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  fft_reg_tables<M>(twR, a.twM);
  __syncthreads();
  pdl_wait();
  const int myrows = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nq = myrows * CPT;
  const bool skip_px = MODE == XF_TANGENT_CG && a.first;   // rows 6..17 (p_old, x) not needed
  auto issue = [&](int q) {      // one warp (lane = gt)
    const int i = q / CPT, j = q % CPT;
    const int t = blockIdx.x + i * gridDim.x, rr = j / nch, h = j % nch;
    const size_t g0 = ((size_t)t * R + rr) * N + (size_t)h * CW;
    double* dst = stg + (size_t)(j & 1) * NOP * CW;
    uint64_t* bar = &bars[(i & 1) * S + (j & 1)];
    const unsigned bytes = CW * 8;
    if (gt == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, bytes * (skip_px ? NOP - 12 : NOP));
    }
    __syncwarp();
    for (int r = gt; r < NOP; r += 32) {
      if (skip_px && r >= 6 && r < 18) continue;
      const double* src;
      if (MODE == XF_TANGENT_CG)
        src = r < 6 ? a.r + r * n : r < 12 ? a.p + (r - 6) * n : r < 18 ? a.x + (r - 12) * n : a.C + (r - 18) * n;
      else
        src = r < 6 ? a.p + r * n : a.C + (r - 6) * n;
      bulk_g2s(dst + (size_t)r * CW, src + g0, bytes, bar);
    }
  };
  if (threadIdx.x < 32)
    for (int q = 0; q < S && q < nq; ++q) issue(q);
  double beta = 0.0, alpha = 0.0;
  if (MODE == XF_TANGENT_CG) {
    beta = a.sc->beta;
    alpha = a.sc->alpha;
  }
  double red = 0.0;
  for (int i = grp, u = 0; i < myrows; i += 2, ++u) {   // u: tiles this group has done before
    const int t = blockIdx.x + i * gridDim.x;
#pragma unroll 1
    for (int j = 0; j < CPT; ++j) {
      const int q = i * CPT + j, rr = j / nch, h = j % nch;
      // use number of this group's barrier [j & 1]: u * CPT / S + j / S
      mbar_wait(&bars[grp * S + (j & 1)], (unsigned)((u * (CPT / S) + j / S) & 1));
      const double* st = stg + (size_t)(j & 1) * NOP * CW;
      {
        const int v = gt, xg = h * CW + v;
        const size_t g = ((size_t)t * R + rr) * N + xg;
        double p[6], tv[6];
        if (MODE == XF_TANGENT_CG) {
          // CG with the solution update one step late (x += alpha_{k-1} p_{k-1}); see cg_mech
          if (a.first) {
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              a.x[c * n + g] = 0.0;
              p[c] = st[c * CW + v];
              a.p[c * n + g] = p[c];
            }
          } else {
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              const double po = st[(6 + c) * CW + v];
              a.x[c * n + g] = fma(alpha, po, st[(12 + c) * CW + v]);
              p[c] = fma(beta, po, st[c * CW + v]);
              a.p[c * n + g] = p[c];
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 6; ++c) p[c] = st[c * CW + v];
        }
        tangent_smem<CMP>(st + C0 * CW, v, CW, p, tv);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (MODE == XF_TANGENT_CG) red = fma(p[c], tv[c], red);
          const int l = c * R + rr;
          fbd[(size_t)(l * LP + SWZ(l, xg >> 1)) * 2 + (xg & 1)] = tv[c];
        }
      }
      group_bar(grp);                              // the stage has been read by the whole group
      if (gt < 32 && q + S < nq) issue(q + S);
    }
    // ---- this group's FFT / post-processing / stores (the other group consumes meanwhile) ----
    {
      constexpr int TPT = fft_reg_tpl<M>();
      static_assert(NC * R * TPT <= GT && (NC * R * TPT) % 32 == 0, "whole warps of lines within one group");
      if (gt < NC * R * TPT) fft_reg_inplace<M, false>(fb + (size_t)(gt / TPT) * LP, gt / TPT, gt % TPT, twR);
    }
    group_bar(grp);
    for (int idx = gt; idx < NC * R * (M / 2 + 1); idx += GT) {
      const int k = idx % (M / 2 + 1), l = idx / (M / 2 + 1);
      r2c_post<N>(fb + (size_t)l * LP, l, k, a.twN);
    }
    group_bar(grp);
    {
      const int z = t / (a.Ny / R), y0 = (t % (a.Ny / R)) * R;
      constexpr int NB = (Hx + kKB - 1) / kKB, KS = GT / 4, NJ = (NB + KS - 1) / KS;
      static_assert(kKB == 2 && kXR == 2, "store mapping below");
      const int kl = gt & 1, r2 = (gt >> 1) & 1, kb0 = gt >> 2;
      const size_t cstep = (size_t)a.Nz * (a.HxA / kKB) * a.Ny * kKB, kstep = (size_t)KS * a.Ny * kKB;
      double2* g0 = a.spec + (((size_t)z * (a.HxA / kKB) + kb0) * a.Ny + y0 + r2) * kKB + kl;
      const bool last = (kb0 + (NJ - 1) * KS) * kKB + kl < Hx;
      double2 val[NC][NJ];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int l = c * R + r2;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
          if (jj < NJ - 1 || last) val[c][jj] = fb[l * LP + SWZ(l, (kb0 + jj * KS) * kKB + kl)];
      }
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj)
          if (jj < NJ - 1 || last) g0[c * cstep + jj * kstep] = val[c][jj];
    }
    group_bar(grp);                                // fb is free for the group's next tile
  }
  if (MODE == XF_TANGENT_CG) {
    double rr2[1] = {red};
    reduce_finalize<1>(rr2, a.partials, a.sc, a.red_op, a.red_slot);
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

static int sm_count() {
  static int s = 0;
  if (!s) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    if (s <= 0) s = 148;
  }
  return s;
}

// returns FGD_OK and *done = false when the bulk-copy path does not apply (alignment)
// operands: CG (r, p, x, C); TANGENT (-, p, -, C); HELM (r, p, x, q in C)
static fgd_status launch_xtan(fgd_ctx* c, int mode, double* r, double* p, double* x, const double* Cp,
                              int red_op, int red_slot, bool* done, int first) {
  *done = false;
  const int Nx = c->n[0], Ny = c->n[1];
  const bool cmp = mode != XF_HELM_UPDATE && Cp == c->Cc;
  auto al = [](const void* q) { return ((uintptr_t)q & 15) == 0; };
  if (!al(p) || !al(Cp) || (mode != XF_TANGENT && (!al(r) || !al(x)))) return FGD_OK;
  static const int cw_env = [] {
    const char* e = std::getenv("FGD_XT_CW");
    return e ? std::atoi(e) : 128;
  }();
  const bool helm = mode == XF_HELM_UPDATE;
  // N = 512 (6 components): a row pair needs 24 line FFTs of 256 points -> 256 threads, 256-voxel chunks
  const int CW = helm ? Nx : std::min(Nx, std::max(16, Nx >= 512 ? 256 : cw_env));
  const int thr = (!helm && Nx >= 512) ? 256 : 128;
  const int R = helm ? std::min(Ny, 8) : kXR;
  const int nc = helm ? 1 : 6;
  const int nop = helm ? 4 : (mode == XF_TANGENT_CG ? 18 : 6) + (cmp ? 9 : 21);
  const size_t stage = (size_t)nop * CW * 8;
  size_t fixed = 0;
#define XTF(NN) fixed = xt_fixed_bytes<NN>(nc * R);
  FGD_DISPATCH_N(Nx, XTF)
#undef XTF
  // as many stages (2..4) as leave room for two CTAs per SM
  const size_t budget = 112 * 1024;
  int S = (int)std::min<size_t>(4, budget > fixed ? (budget - fixed) / stage : 0);
  if (S < 2) S = 2;
  static const int s_env = [] {
    const char* e = std::getenv("FGD_XT_S");
    return e ? std::atoi(e) : 0;
  }();
  if (helm) S = 3;   // measured: 3 stages of 8 KB beat 4 for the 1-component PCG pass (256^3)
  if (s_env >= 2 && s_env <= 8) S = s_env;
  const size_t smem = fixed + S * stage;
  if (smem > 227 * 1024) return FGD_OK;
  XTArgs a{c->guard ? c->sc : nullptr, Ny, c->nz_l, c->HxA, CW, S, R, first, c->nvox, r, p, x, Cp, c->specA, c->sc, c->partials, red_op, red_slot,
           c->tabs.tw[ilog2(Nx / 2)], c->tabs.tw[ilog2(Nx)]};
  const int ntiles = (Ny / R) * c->nz_l;
  KTimer kt(c, helm ? KC_XFWD1 : (mode == XF_TANGENT_CG && !first) ? KC_XFWD6_CG : KC_XFWD6);
  int grid = 1;
#define XTL(NN)                                                                                       \
  {                                                                                                   \
    auto kern = mode == XF_TANGENT_CG ? (cmp ? k_xtan<NN, XF_TANGENT_CG, true, kXR> : k_xtan<NN, XF_TANGENT_CG, false, kXR>) \
              : mode == XF_TANGENT    ? (cmp ? k_xtan<NN, XF_TANGENT, true, kXR> : k_xtan<NN, XF_TANGENT, false, kXR>)       \
              : R == 8                ? k_xtan<NN, XF_HELM_UPDATE, false, 8> : k_xtan<NN, XF_HELM_UPDATE, false, 4>;    \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);          \
    if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_xtan smem attr: ") + cudaGetErrorString(e)); \
    int occ = 0;                                                                                      \
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, thr, smem) != cudaSuccess || occ < 1) occ = 1; \
    grid = grid_cap(std::max(1, std::min(ntiles, sm_count() * occ)));                                 \
    if (red_op != RED_NONE) {                                                                         \
      fgd_status s_ = ensure_partials(c, (size_t)grid);                                               \
      if (s_ != FGD_OK) return s_;                                                                    \
      a.partials = c->partials;                                                                       \
    }                                                                                                 \
    c->launches++;                                                                                    \
    e = launch_pdl(kern, dim3(grid), dim3(thr), smem, c->stream, a);                                  \
    if (e == cudaSuccess) e = cudaGetLastError();                                                     \
    if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_xtan: ") + cudaGetErrorString(e));         \
  }
  static const int pp_env = [] {
    const char* e = std::getenv("FGD_XT_PP");
    return e ? std::atoi(e) : 1;   // 1: ping-pong kernel for N = 512 (k_xtan_pp)
  }();
  if (pp_env && !helm && Nx == 512 && Ny >= kXR) {
    auto kern = mode == XF_TANGENT_CG ? (cmp ? k_xtan_pp<512, XF_TANGENT_CG, true> : k_xtan_pp<512, XF_TANGENT_CG, false>)
                                      : (cmp ? k_xtan_pp<512, XF_TANGENT, true> : k_xtan_pp<512, XF_TANGENT, false>);
    const size_t smem_pp = mode == XF_TANGENT_CG ? (cmp ? xtpp_smem<512, XF_TANGENT_CG, true>() : xtpp_smem<512, XF_TANGENT_CG, false>())
                                                 : (cmp ? xtpp_smem<512, XF_TANGENT, true>() : xtpp_smem<512, XF_TANGENT, false>());
    if (smem_pp <= 227 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pp);
      if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_xtan_pp smem attr: ") + cudaGetErrorString(e));
      grid = grid_cap(std::max(1, std::min((ntiles + 1) / 2, sm_count())));
      if (red_op != RED_NONE) {
        fgd_status s_ = ensure_partials(c, (size_t)grid);
        if (s_ != FGD_OK) return s_;
        a.partials = c->partials;
      }
      c->launches++;
      e = launch_pdl(kern, dim3(grid), dim3(512), smem_pp, c->stream, a);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_xtan_pp: ") + cudaGetErrorString(e));
      *done = true;
      return FGD_OK;
    }
  }
  FGD_DISPATCH_N(Nx, XTL)
#undef XTL
  *done = true;
  return FGD_OK;
}

fgd_status launch_xfwd(fgd_ctx* c, int ncomp, int mode, const double* in0, const double* in1, double* out0,
                       const double* Cp, int red_op, int red_slot) {
  return launch_xfwd_io(c, ncomp, mode, in0, in1, out0, nullptr, Cp, red_op, red_slot);
}

fgd_status launch_xfwd_io(fgd_ctx* c, int ncomp, int mode, const double* in0, const double* in1, double* out0,
                          double* io1, const double* Cp, int red_op, int red_slot, int first) {
  if (mode == XF_PLAIN && ((uintptr_t)in0 & 15) == 0) return pipe_xfwd_plain(c, ncomp, in0);
  if (((ncomp == 6 && (mode == XF_TANGENT || mode == XF_TANGENT_CG)) || (ncomp == 1 && mode == XF_HELM_UPDATE)) &&
      !std::getenv("FGD_NO_XTAN")) {
    bool done = false;
    fgd_status s;
    if (mode == XF_TANGENT_CG)
      s = launch_xtan(c, mode, const_cast<double*>(in0), out0, io1, Cp, red_op, red_slot, &done, first);
    else if (mode == XF_TANGENT)
      s = launch_xtan(c, mode, nullptr, const_cast<double*>(in0), nullptr, Cp, red_op, red_slot, &done, 0);
    else   // HELM: x(out0) += alpha p(in0); r(io1) -= alpha q(in1)
      s = launch_xtan(c, mode, io1, const_cast<double*>(in0), out0, in1, red_op, red_slot, &done, 0);
    if (s != FGD_OK || done) return s;
  }
  if (first && mode == XF_TANGENT_CG) {
    // generic path: p_old = x = 0 make the update exact (alpha = beta = 0 after RED_MECH_INIT)
    FGD_CUDA(c, cudaMemsetAsync(out0, 0, 6 * c->nvox * sizeof(double), c->stream));
    FGD_CUDA(c, cudaMemsetAsync(io1, 0, 6 * c->nvox * sizeof(double), c->stream));
  }
  const int Nx = c->n[0], Ny = c->n[1], Nz = c->nz_l;
  const int TY = choose_TY(Nx, ncomp, Ny);
  const int nl = ncomp * TY;
  const int thr = std::min(kMaxThr, std::max(64, round32(nl * fft_TPL(Nx / 2))));
  const size_t smem = ((size_t)nl * xline(Nx / 2) + Nx / 2) * sizeof(double2);
  dim3 grid(Ny / TY, Nz);
  XArgs a{c->guard ? c->sc : nullptr, Ny, Nz, TY, c->HxA, c->nvox, in0, in1, out0, io1, nullptr, Cp, c->specA, c->sc, c->partials, red_op, red_slot,
          (Cp != nullptr && Cp == c->Cc) ? 1 : 0};
  if (red_op != RED_NONE) {
    fgd_status s = ensure_partials(c, (size_t)grid.x * grid.y);
    if (s != FGD_OK) return s;
    a.partials = c->partials;
  }
  const double2* tw = c->tabs.tw[ilog2(Nx / 2)];
  const double2* twN = c->tabs.tw[ilog2(Nx)];
  KTimer kt(c, ncomp == 6 ? ((mode == XF_TANGENT_CG && !first) ? KC_XFWD6_CG : KC_XFWD6) : KC_XFWD1);
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
