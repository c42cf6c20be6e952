// Persistent, double-buffered FFT passes (cp.async pipelines).
//
// Each CTA loops over tiles t = blockIdx.x, blockIdx.x + gridDim.x, ...; the global->shared
// copies of tile t+gridDim.x are issued (cp.async.cg, 16 B per complex double, any scatter
// pattern) BEFORE the FFT of tile t runs, so every SM keeps a full tile of loads in flight
// while it computes.  Stores are plain st.global (fire and forget).  The grid is sized to
// the number of CTAs the device keeps resident (SMs x occupancy).
//
// Passes (same layouts as passes.cu):
//   YP    C2C along y, A[c][z][kx][y] <-> B[c][kx][ky][z]        tile (c, kx, TZ z's)
//   ZP    C2C along z in place on B with the spectral multiply  tile (kx, TL ky's), NC comps
//   XI    C2R along x, one component per tile, with epilogue    tile (c, z, TY rows)
//   XF    R2C along x of a plain real field, one comp per tile  tile (c, z, TY rows)
#include "reduce.cuh"

namespace fgd {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// ---- shared per-line real <-> half-spectrum helpers (see passes.cu for the algebra) ----------
template <int N>
__device__ __forceinline__ void r2c_post_p(double2* line, int l, int k, const double2* twN) {
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
  const double2 WO = cmul(twN[k], O);
  line[SWZ(l, k)] = cadd(E, WO);
  if (k != M - k) line[SWZ(l, M - k)] = conjg(csub(E, WO));
}

template <int N>
__device__ __forceinline__ void c2r_pre_p(double2* line, int l, int k, const double2* twN) {
  constexpr int M = N / 2;
  if (k == 0) {
    const double x0 = line[SWZ(l, 0)].x, xm = line[SWZ(l, M)].x;
    line[SWZ(l, 0)] = make_double2(x0 + xm, x0 - xm);
    return;
  }
  const double2 xk = line[SWZ(l, k)], xm = line[SWZ(l, M - k)];
  const double2 A = cadd(xk, conjg(xm)), B = csub(xk, conjg(xm));
  const double2 w = conjg(twN[k]);
  const double2 iWB = mul_mi<true>(cmul(w, B));
  line[SWZ(l, k)] = cadd(A, iWB);
  if (k != M - k) line[SWZ(l, M - k)] = conjg(csub(A, iWB));
}

// ---------------------------------------------------------------------------------------------
// Y pass
// ---------------------------------------------------------------------------------------------
// Slab layout of the transposed spectra: P z-slabs of nzs planes in real space,
// P y-slabs of nys rows in the z pass.  The y pass writes S[r][s][c][kx][kyl][zl] (r = z-slab,
// s = destination y-slab), the all-to-all moves block S[r][s] to R[s][r], the z pass works on
// R[s][src][c][kx][kyl][zl].  P = 1 is the plain B[c][kx][ky][z] layout.
struct SlabL {
  int P, nys, nzs, lg_nys, lg_nzs;
};
__device__ __forceinline__ size_t slab_index(const SlabL& L, int C, int Hx, int c, int kx, int blk0_idx, int blk1_idx,
                                             int row, int col) {
  return (((((size_t)(blk0_idx * L.P + blk1_idx) * C + c) * Hx + kx) * L.nys + row) << L.lg_nzs) + col;
}
// S: y pass output / y-inv input, indexed by (c, kx, ky, z local)
__device__ __forceinline__ size_t s_index(const SlabL& L, int C, int Hx, int c, int kx, int ky, int z) {
  return slab_index(L, C, Hx, c, kx, z >> L.lg_nzs, ky >> L.lg_nys, ky & (L.nys - 1), z & (L.nzs - 1));
}
// R: z pass buffer, indexed by (c, kx, ky local, z global)
__device__ __forceinline__ size_t r_index(const SlabL& L, int C, int Hx, int c, int kx, int ky, int z) {
  return slab_index(L, C, Hx, c, kx, ky >> L.lg_nys, z >> L.lg_nzs, ky & (L.nys - 1), z & (L.nzs - 1));
}

struct YArgs {
  double2* A;
  double2* B;
  int Nz, Hx, TZ, ncomp, lgTZ;
  const double2* tw;
  SlabL L;
};

template <int N, bool INV>
__device__ __forceinline__ void y_issue(const YArgs& a, int t, double2* buf) {
  constexpr int LP = cline(N);
  const int nzt = a.Nz / a.TZ;
  const int zt = t % nzt, r = t / nzt, kx = r % a.Hx, c = r / a.Hx;
  const int z0 = zt * a.TZ, TZ = a.TZ;
  if (!INV) {
    for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
      const int zz = idx / N, y = idx % N;
      cp_async16(&buf[zz * LP + SWZ(zz, y)], &a.A[((size_t)(c * a.Nz + z0 + zz) * a.Hx + kx) * N + y]);
    }
  } else {
    for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
      const int zz = idx & (TZ - 1), ky = idx >> a.lgTZ;
      cp_async16(&buf[zz * LP + SWZ(zz, ky)], &a.B[s_index(a.L, a.ncomp, a.Hx, c, kx, ky, z0 + zz)]);
    }
  }
}

template <int N, bool INV>
__global__ void __launch_bounds__(256, 2) k_ypipe(YArgs a) {
  extern __shared__ double2 sm[];
  constexpr int LP = cline(N);
  const int TZ = a.TZ;
  double2* tws = sm + 2 * TZ * LP;
  build_pass_tables<N, true>(tws, a.tw);
  const int ntiles = a.ncomp * a.Hx * (a.Nz / TZ);
  int t = blockIdx.x;
  if (t < ntiles) y_issue<N, INV>(a, t, sm);
  cp_async_commit();
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) y_issue<N, INV>(a, tn, sm + ((i + 1) & 1) * TZ * LP);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* buf = sm + (i & 1) * TZ * LP;
    fft_lines<N, INV, true>(buf, TZ, LP, tws);
    __syncthreads();
    const int nzt = a.Nz / TZ;
    const int zt = t % nzt, r = t / nzt, kx = r % a.Hx, c = r / a.Hx;
    const int z0 = zt * TZ;
    if (!INV) {
      for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
        const int zz = idx & (TZ - 1), ky = idx >> a.lgTZ;
        a.B[s_index(a.L, a.ncomp, a.Hx, c, kx, ky, z0 + zz)] = buf[zz * LP + SWZ(zz, ky)];
      }
    } else {
      for (int idx = threadIdx.x; idx < TZ * N; idx += blockDim.x) {
        const int zz = idx / N, y = idx % N;
        a.A[((size_t)(c * a.Nz + z0 + zz) * a.Hx + kx) * N + y] = buf[zz * LP + SWZ(zz, y)];
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// Z pass with the spectral multiply
// ---------------------------------------------------------------------------------------------
struct ZPArgs {
  double2* B;
  SlabL SL;
  int ky_off;          // global index of the first local ky (distributed y-slab)
  int Nyl;             // local ky rows
  int Nx, Ny, Hx, TL, scheme, lgTL;
  double h[3], L[3];
  double scale;
  double shift[6];
  int mask[6];
  double mean_ell2;
  const double2* twx;
  const double2* twy;
  const double2* twz;
};

__device__ __forceinline__ void zsymbol(const ZPArgs& a, int Nz, int kx, int ky, int kz, double2* k,
                                        const double2* twz_s) {
  if (a.scheme == 1) {
    const double2 wx = __ldg(&a.twx[kx]), wy = __ldg(&a.twy[ky]), wz = twz_s[kz];
    const double2 ex = make_double2(wx.x, -wx.y), ey = make_double2(wy.x, -wy.y), ez = make_double2(wz.x, -wz.y);
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

// Galerkin projection G^*(xi) on 6 Mandel components held in shared memory
// v[c] points at component c (6 lines of the tile)
__device__ __forceinline__ void project6(const ZPArgs& a, double2* const* v, const double2* k, bool dc) {
  constexpr double S2 = 1.41421356237309504880, IS2 = 0.70710678118654752440;
  const double k2 = k[0].x * k[0].x + k[0].y * k[0].y + k[1].x * k[1].x + k[1].y * k[1].y + k[2].x * k[2].x +
                    k[2].y * k[2].y;
  if (dc) {
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const double2 t = *v[c];
      *v[c] = a.mask[c] ? cscale(make_double2(t.x - a.shift[c], t.y), a.scale) : make_double2(0.0, 0.0);
    }
    return;
  }
  if (k2 == 0.0) {
#pragma unroll
    for (int c = 0; c < 6; ++c) *v[c] = make_double2(0.0, 0.0);
    return;
  }
  const double2 kc0 = conjg(k[0]), kc1 = conjg(k[1]), kc2 = conjg(k[2]);
  double2 t0, t1, t2;
  {
    const double2 T00 = *v[0], T01 = cscale(*v[5], IS2), T02 = cscale(*v[4], IS2);
    t0 = cadd(cadd(cmul(T00, kc0), cmul(T01, kc1)), cmul(T02, kc2));
    const double2 T11 = *v[1], T12 = cscale(*v[3], IS2);
    t1 = cadd(cadd(cmul(T01, kc0), cmul(T11, kc1)), cmul(T12, kc2));
    const double2 T22 = *v[2];
    t2 = cadd(cadd(cmul(T02, kc0), cmul(T12, kc1)), cmul(T22, kc2));
  }
  const double2 s = cadd(cadd(cmul(kc0, t0), cmul(kc1, t1)), cmul(kc2, t2));
  const double inv = 1.0 / k2;
  const double2 hs = cscale(s, 0.5 * inv);
  const double f = 2.0 * inv * a.scale;          // output scale folded into u
  const double2 u0 = cscale(csub(t0, cmul(k[0], hs)), f);
  const double2 u1 = cscale(csub(t1, cmul(k[1], hs)), f);
  const double2 u2 = cscale(csub(t2, cmul(k[2], hs)), f);
  *v[0] = cmul(u0, k[0]);
  *v[1] = cmul(u1, k[1]);
  *v[2] = cmul(u2, k[2]);
  *v[3] = cscale(cadd(cmul(u1, k[2]), cmul(k[1], u2)), 0.5 * S2);
  *v[4] = cscale(cadd(cmul(u0, k[2]), cmul(k[0], u2)), 0.5 * S2);
  *v[5] = cscale(cadd(cmul(u0, k[1]), cmul(k[0], u1)), 0.5 * S2);
}

template <int N, int NC>
__device__ __forceinline__ void z_issue(const ZPArgs& a, int t, double2* buf) {
  constexpr int LP = cline(N);
  const int TL = a.TL;
  const int nyt = a.Nyl / TL;
  const int kx = t / nyt, ky0 = (t % nyt) * TL;
  for (int idx = threadIdx.x; idx < NC * TL * N; idx += blockDim.x) {
    const int kz = idx % N, rest = idx / N;
    const int ll = rest & (TL - 1), c = rest >> a.lgTL;
    cp_async16(&buf[(c * TL + ll) * LP + SWZ(c * TL + ll, kz)], &a.B[r_index(a.SL, NC, a.Hx, c, kx, ky0 + ll, kz)]);
  }
}

template <int N, int NC, int MODE>
__global__ void __launch_bounds__(192, 3) k_zpipe(ZPArgs a) {
  extern __shared__ double2 sm[];
  constexpr int LP = cline(N);
  const int TL = a.TL;
  double2* tws = sm + 2 * NC * TL * LP;    // e^{-2 pi i m/N} (symbol)
  double2* tpz = tws + N;                    // per-pass FFT twiddles
  load_table(tws, a.twz, N);
  build_pass_tables<N>(tpz, a.twz);
  const int nyt = a.Nyl / TL;
  const int ntiles = a.Hx * nyt;
  int t = blockIdx.x;
  if (t < ntiles) z_issue<N, NC>(a, t, sm);
  cp_async_commit();
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) z_issue<N, NC>(a, tn, sm + ((i + 1) & 1) * NC * TL * LP);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* buf = sm + (i & 1) * NC * TL * LP;
    const int kx = t / nyt, ky0 = (t % nyt) * TL;
    fft_lines<N, false>(buf, NC * TL, LP, tpz);
    __syncthreads();
    for (int idx = threadIdx.x; idx < TL * N; idx += blockDim.x) {
      const int kz = idx % N, ll = idx / N;
      const int ky = ky0 + ll + a.ky_off;
      double2 k[3];
      zsymbol(a, N, kx, ky, kz, k, tws);
      const bool dc = (kx == 0 && ky == 0 && kz == 0);
      if (MODE == Z_PRECOND) {
        double2* v = &buf[ll * LP + SWZ(ll, kz)];
        const double k2 = k[0].x * k[0].x + k[0].y * k[0].y + k[1].x * k[1].x + k[1].y * k[1].y + k[2].x * k[2].x +
                          k[2].y * k[2].y;
        *v = cscale(*v, a.scale / (1.0 + a.mean_ell2 * k2));
      } else {
        double2* v[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) v[c] = &buf[(c * TL + ll) * LP + SWZ(c * TL + ll, kz)];
        project6(a, v, k, dc);
      }
    }
    __syncthreads();
    fft_lines<N, true>(buf, NC * TL, LP, tpz);
    __syncthreads();
    for (int idx = threadIdx.x; idx < NC * TL * N; idx += blockDim.x) {
      const int kz = idx % N, rest = idx / N;
      const int ll = rest & (TL - 1), c = rest >> a.lgTL;
      a.B[r_index(a.SL, NC, a.Hx, c, kx, ky0 + ll, kz)] = buf[(c * TL + ll) * LP + SWZ(c * TL + ll, kz)];
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// X passes, one component per tile
// ---------------------------------------------------------------------------------------------
struct XPArgs {
  int Ny, Nz, TY, ncomp, lgTY;
  size_t nvox;
  double2* spec;
  const double* in0;   // XF: real input ; XI: p (MECH_CG) or r (HELM_Z)
  double* out0;        // XI: output q / z
  double* io1;         // XI MECH_CG: x
  double* io2;         // XI MECH_CG: r
  DevScalars* sc;
  double* partials;
  int red_op, red_slot;
  const double2* twM;
  const double2* twN;
};

template <int N>
__device__ __forceinline__ void xi_issue(const XPArgs& a, int t, double2* buf) {
  constexpr int M = N / 2, Hx = M + 1;
  constexpr int LP = xline(M);
  const int TY = a.TY, nyt = a.Ny / TY;
  const int yt = t % nyt, r = t / nyt, z = r % a.Nz, c = r / a.Nz;
  const int y0 = yt * TY;
  for (int idx = threadIdx.x; idx < Hx * TY; idx += blockDim.x) {
    const int yy = idx & (TY - 1), kx = idx >> a.lgTY;
    cp_async16(&buf[yy * LP + SWZ(yy, kx)], &a.spec[((size_t)(c * a.Nz + z) * Hx + kx) * a.Ny + y0 + yy]);
  }
}

template <int N, int MODE>
__global__ void __launch_bounds__(128, 4) k_xipipe(XPArgs a) {
  extern __shared__ double2 sm[];
  constexpr int M = N / 2;
  constexpr int LP = xline(M);
  const int TY = a.TY, nyt = a.Ny / TY;
  double2* twM = sm + 2 * TY * LP;
  double2* twN = twM + M;
  build_pass_tables<M>(twM, a.twM);
  load_table(twN, a.twN, N);
  const int ntiles = a.ncomp * a.Nz * nyt;
  const size_t n = a.nvox;
  double red[1] = {0.0};
  double alpha = 0.0;
  if (MODE == XI_MECH_CG) alpha = a.sc->alpha;
  int t = blockIdx.x;
  if (t < ntiles) xi_issue<N>(a, t, sm);
  cp_async_commit();
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) xi_issue<N>(a, tn, sm + ((i + 1) & 1) * TY * LP);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* buf = sm + (i & 1) * TY * LP;
    for (int idx = threadIdx.x; idx < TY * (M / 2 + 1); idx += blockDim.x) {
      const int k = idx % (M / 2 + 1), l = idx / (M / 2 + 1);
      c2r_pre_p<N>(buf + (size_t)l * LP, l, k, twN);
    }
    __syncthreads();
    fft_lines<M, true>(buf, TY, LP, twM);
    __syncthreads();
    const int yt = t % nyt, r = t / nyt, z = r % a.Nz, c = r / a.Nz;
    const int y0 = yt * TY;
    const double* bd = reinterpret_cast<const double*>(buf);
#pragma unroll 4
    for (int idx = threadIdx.x; idx < TY * N; idx += blockDim.x) {
      const int yy = idx / N, x = idx % N;
      const size_t g = (size_t)c * n + ((size_t)z * a.Ny + y0 + yy) * N + x;
      const double q = bd[(size_t)(yy * LP + SWZ(yy, x >> 1)) * 2 + (x & 1)];
      if (MODE == XI_STORE) {
        a.out0[g] = q;
      } else if (MODE == XI_STORE_RR) {
        a.out0[g] = q;
        red[0] = fma(q, q, red[0]);
      } else if (MODE == XI_MECH_CG) {
        const double p = a.in0[g], xo = a.io1[g], ro = a.io2[g];
        a.io1[g] = fma(alpha, p, xo);
        const double rn = fma(-alpha, q, ro);
        a.io2[g] = rn;
        red[0] = fma(rn, rn, red[0]);
      } else if (MODE == XI_HELM_Z) {
        a.out0[g] = q;
        red[0] = fma(a.in0[g], q, red[0]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if (MODE != XI_STORE) reduce_finalize<1>(red, a.partials, a.sc, a.red_op, a.red_slot);
}

template <int N>
__device__ __forceinline__ void xf_issue(const XPArgs& a, int t, double2* buf) {
  constexpr int M = N / 2;
  constexpr int LP = xline(M);
  const int TY = a.TY, nyt = a.Ny / TY;
  const int yt = t % nyt, r = t / nyt, z = r % a.Nz, c = r / a.Nz;
  const int y0 = yt * TY;
  const double2* src = reinterpret_cast<const double2*>(a.in0 + (size_t)c * a.nvox + ((size_t)z * a.Ny + y0) * N);
  for (int idx = threadIdx.x; idx < TY * M; idx += blockDim.x) {
    const int yy = idx / M, m = idx % M;
    cp_async16(&buf[yy * LP + SWZ(yy, m)], &src[(size_t)yy * M + m]);
  }
}

template <int N>
__global__ void __launch_bounds__(128, 4) k_xfpipe(XPArgs a) {
  extern __shared__ double2 sm[];
  constexpr int M = N / 2, Hx = M + 1;
  constexpr int LP = xline(M);
  const int TY = a.TY, nyt = a.Ny / TY;
  double2* twM = sm + 2 * TY * LP;
  double2* twN = twM + M;
  build_pass_tables<M>(twM, a.twM);
  load_table(twN, a.twN, N);
  const int ntiles = a.ncomp * a.Nz * nyt;
  int t = blockIdx.x;
  if (t < ntiles) xf_issue<N>(a, t, sm);
  cp_async_commit();
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) xf_issue<N>(a, tn, sm + ((i + 1) & 1) * TY * LP);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* buf = sm + (i & 1) * TY * LP;
    fft_lines<M, false>(buf, TY, LP, twM);
    __syncthreads();
    for (int idx = threadIdx.x; idx < TY * (M / 2 + 1); idx += blockDim.x) {
      const int k = idx % (M / 2 + 1), l = idx / (M / 2 + 1);
      r2c_post_p<N>(buf + (size_t)l * LP, l, k, twN);
    }
    __syncthreads();
    const int yt = t % nyt, r = t / nyt, z = r % a.Nz, c = r / a.Nz;
    const int y0 = yt * TY;
    for (int idx = threadIdx.x; idx < Hx * TY; idx += blockDim.x) {
      const int yy = idx & (TY - 1), kx = idx >> a.lgTY;
      a.spec[((size_t)(c * a.Nz + z) * Hx + kx) * a.Ny + y0 + yy] = buf[yy * LP + SWZ(yy, kx)];
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------------
static int num_sms() {
  static int s = 0;
  if (!s) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    if (s <= 0) s = 148;
  }
  return s;
}

static int p2floor(long v) {
  int p = 1;
  while ((long)p * 2 <= v) p *= 2;
  return p;
}
static int r32(int v) { return std::max(64, ((v + 31) / 32) * 32); }

template <typename K>
static fgd_status launch_persistent(fgd_ctx* c, K kernel, int threads, size_t smem, int ntiles, int* grid_out,
                                    const char* name) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string(name) + " smem attr: " + cudaGetErrorString(e));
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
  if (e != cudaSuccess || occ < 1) occ = 1;
  *grid_out = std::max(1, std::min(ntiles, num_sms() * occ));
  return FGD_OK;
}

#define FGD_PLAUNCH(ctx, kern, thr, smem, ntiles, ...)                                                  \
  do {                                                                                                  \
    int grid_ = 1;                                                                                      \
    fgd_status st_ = launch_persistent(ctx, kern, thr, smem, ntiles, &grid_, #kern);                     \
    if (st_ != FGD_OK) return st_;                                                                      \
    (ctx)->launches++;                                                                                  \
    kern<<<grid_, thr, smem, (ctx)->stream>>>(__VA_ARGS__);                                              \
    cudaError_t e_ = cudaGetLastError();                                                                \
    if (e_ != cudaSuccess) return set_err(ctx, FGD_ECUDA, std::string(#kern) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define FGD_PDISPATCH(Nval, MACRO)  \
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

static SlabL slab_layout(const fgd_ctx* c) {
  SlabL L{};
  L.P = c->P;
  L.nys = c->n[1] / c->P;
  L.nzs = c->n[2] / c->P;
  L.lg_nys = ilog2(L.nys);
  L.lg_nzs = ilog2(L.nzs);
  return L;
}

fgd_status pipe_y(fgd_ctx* c, int ncomp, bool inv) {
  const int Ny = c->n[1], Nz = c->nz_l;
  const int TPL = fft_TPL(Ny, true);
  int TZ = p2floor(std::max(1, 128 / TPL));
  TZ = std::min(TZ, std::min(Nz, c->n[2] / c->P));
  const int thr = std::min(256, r32(TZ * TPL));
  const size_t smem = (2 * (size_t)TZ * cline(Ny) + Ny) * sizeof(double2);
  const int ntiles = ncomp * c->Hx * (Nz / TZ);
  YArgs a{c->specA, c->specB, Nz, c->Hx, TZ, ncomp, ilog2(TZ), c->tabs.tw[ilog2(Ny)], slab_layout(c)};
  KTimer kt(c, inv ? (ncomp == 6 ? KC_YINV6 : KC_YINV1) : (ncomp == 6 ? KC_YFWD6 : KC_YFWD1));
#define YPP(NN)                                                                  \
  if (inv) FGD_PLAUNCH(c, (k_ypipe<NN, true>), thr, smem, ntiles, a);            \
  else FGD_PLAUNCH(c, (k_ypipe<NN, false>), thr, smem, ntiles, a);
  FGD_PDISPATCH(Ny, YPP)
#undef YPP
  return FGD_OK;
}

fgd_status pipe_z(fgd_ctx* c, int ncomp, int mode, double scale, const double* dc_shift, double mean_ell2) {
  const int Ny = c->n[1], Nz = c->n[2];
  const int Nyl = c->nranks > 1 ? Ny / c->P : Ny;
  const int TPL = fft_TPL(Nz);
  int TL = p2floor(std::max(1, 192 / (ncomp * TPL)));
  if (Nz == 1) TL = 32;
  TL = std::min(TL, Nyl);
  const int thr = std::min(192, std::max(r32(ncomp * TL * TPL), r32(std::min(TL * Nz, 192))));
  const size_t smem = (2 * (size_t)ncomp * TL * cline(Nz) + 2 * Nz) * sizeof(double2);
  const int ntiles = c->Hx * (Nyl / TL);
  ZPArgs a{};
  a.B = c->P > 1 ? c->specC : c->specB;
  a.SL = slab_layout(c);
  a.ky_off = c->nranks > 1 ? c->rank * (Ny / c->P) : 0;
  a.Nyl = Nyl;
  a.Nx = c->n[0];
  a.Ny = Ny;
  a.Hx = c->Hx;
  a.TL = TL;
  a.lgTL = ilog2(TL);
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
  a.twx = c->tabs.tw[ilog2(c->n[0])];
  a.twy = c->tabs.tw[ilog2(Ny)];
  a.twz = c->tabs.tw[ilog2(Nz)];
  KTimer kt(c, ncomp == 6 ? KC_Z6 : KC_Z1);
#define ZPP(NN)                                                                                          \
  if (ncomp == 6 && mode == Z_PROJECT) FGD_PLAUNCH(c, (k_zpipe<NN, 6, Z_PROJECT>), thr, smem, ntiles, a);      \
  else if (ncomp == 1 && mode == Z_PRECOND) FGD_PLAUNCH(c, (k_zpipe<NN, 1, Z_PRECOND>), thr, smem, ntiles, a); \
  else return set_err(c, FGD_EINVAL, "z mode");
  switch (Nz) {
    case 1: ZPP(1); break;
    case 2: ZPP(2); break;
    case 4: ZPP(4); break;
    case 8: ZPP(8); break;
    case 16: ZPP(16); break;
    case 32: ZPP(32); break;
    case 64: ZPP(64); break;
    case 128: ZPP(128); break;
    case 256: ZPP(256); break;
    case 512: ZPP(512); break;
    default: return set_err(c, FGD_EINVAL, "unsupported Nz");
  }
#undef ZPP
  return FGD_OK;
}

static int choose_TYp(int N, int Ny) {
  const int TPL = fft_TPL(N / 2);
  int TY = p2floor(std::max(1, 128 / TPL));
  TY = std::min(TY, 16);
  return std::min(TY, Ny);
}

fgd_status pipe_xinv(fgd_ctx* c, int ncomp, int mode, double* out0, double* io1, double* io2, const double* in1,
                     int red_op, int red_slot) {
  const int Nx = c->n[0], Ny = c->n[1], Nz = c->nz_l;
  const int TY = choose_TYp(Nx, Ny);
  const int thr = std::min(128, r32(TY * fft_TPL(Nx / 2)));
  const size_t smem = (2 * (size_t)TY * xline(Nx / 2) + Nx / 2 + Nx) * sizeof(double2);
  const int ntiles = ncomp * Nz * (Ny / TY);
  XPArgs a{Ny, Nz, TY, ncomp, ilog2(TY), c->nvox, c->specA, in1, out0, io1, io2, c->sc, nullptr, red_op, red_slot,
           c->tabs.tw[ilog2(Nx / 2)], c->tabs.tw[ilog2(Nx)]};
  if (mode != XI_STORE) {
    fgd_status s = ensure_partials(c, (size_t)num_sms() * 8);
    if (s != FGD_OK) return s;
    a.partials = c->partials;
  }
  KTimer kt(c, ncomp == 6 ? KC_XINV6 : KC_XINV1);
#define XIP(NN)                                                                                   \
  if (mode == XI_STORE) FGD_PLAUNCH(c, (k_xipipe<NN, XI_STORE>), thr, smem, ntiles, a);            \
  else if (mode == XI_STORE_RR) FGD_PLAUNCH(c, (k_xipipe<NN, XI_STORE_RR>), thr, smem, ntiles, a); \
  else if (mode == XI_MECH_CG) FGD_PLAUNCH(c, (k_xipipe<NN, XI_MECH_CG>), thr, smem, ntiles, a);   \
  else if (mode == XI_HELM_Z) FGD_PLAUNCH(c, (k_xipipe<NN, XI_HELM_Z>), thr, smem, ntiles, a);     \
  else return set_err(c, FGD_EINVAL, "xinv mode");
  FGD_PDISPATCH(Nx, XIP)
#undef XIP
  return FGD_OK;
}

fgd_status pipe_xfwd_plain(fgd_ctx* c, int ncomp, const double* in0) {
  const int Nx = c->n[0], Ny = c->n[1], Nz = c->nz_l;
  const int TY = choose_TYp(Nx, Ny);
  const int thr = std::min(128, r32(TY * fft_TPL(Nx / 2)));
  const size_t smem = (2 * (size_t)TY * xline(Nx / 2) + Nx / 2 + Nx) * sizeof(double2);
  const int ntiles = ncomp * Nz * (Ny / TY);
  XPArgs a{Ny, Nz, TY, ncomp, ilog2(TY), c->nvox, c->specA, in0, nullptr, nullptr, nullptr, c->sc, nullptr, RED_NONE, 0,
           c->tabs.tw[ilog2(Nx / 2)], c->tabs.tw[ilog2(Nx)]};
  KTimer kt(c, ncomp == 6 ? KC_XFWD6 : KC_XFWD1);
#define XFP(NN) FGD_PLAUNCH(c, (k_xfpipe<NN>), thr, smem, ntiles, a);
  FGD_PDISPATCH(Nx, XFP)
#undef XFP
  return FGD_OK;
}

}  // namespace fgd
