// Persistent, double-buffered FFT passes (cp.async pipelines).
//
// Each CTA loops over tiles t = blockIdx.x, blockIdx.x + gridDim.x, ...; the global->shared
// copies of tile t+gridDim.x are issued (cp.async.cg, 16 B per complex double, any scatter
// pattern) BEFORE the FFT of tile t runs, so every SM keeps a full tile of loads in flight
// while it computes.  Stores are plain st.global (fire and forget).  The grid is sized to
// the number of CTAs the device keeps resident (SMs x occupancy).
//
// Passes (same layouts as passes.cu):
//   YP    C2C along y, A[c][z][y][kx] <-> B[c][kx][ky][z]        tile (c, TK kx's, TZ z's)
//   ZP    C2C along z in place on B with the spectral multiply  tile (kx, TL ky's), NC comps
//   XI    C2R along x, one component per tile, with epilogue    tile (c, z, TY rows)
//   XF    R2C along x of a plain real field, one comp per tile  tile (c, z, TY rows)
#include <cooperative_groups.h>
#include <cstdlib>

#include "reduce.cuh"
#include "tma.cuh"

namespace fgd {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// The same 16-byte copy with an L2 prefetch hint: the L2 fetches the whole aligned 64 / 128 / 256 B
// block around the address (hint = 1 / 2 / 3; 0 = plain copy).  For the strided side of the y
// transposes, whose 32-64 B runs are completed by OTHER CTAs running at the same time: one wide
// DRAM access instead of several isolated sector reads.
__device__ __forceinline__ void cp_async16_l2(void* smem, const void* gmem, int hint) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (hint == 1) asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
  else if (hint == 2) asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
  else if (hint == 3) asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
  else asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
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

// A y-pass tile holds TK = kKB consecutive kx (one contiguous kKB * Ny run per plane of layout A) times TZ consecutive
// z (runs of TZ * 16 B in B, z fastest); line l = zz * TK + kk.  kx >= Hx (padding of the last kx
// block, HxA = Hx rounded up to 4) is neither loaded nor stored.
struct YArgs {
  const DevScalars* guard;   // non-null inside a guarded Krylov loop
  double2* A;
  double2* B;
  int Nz, Hx, HxA, TZ, TK, ncomp, lgTZ, lgTK;
  const double2* tw;
  SlabL L;
  int kb0, nkbc;   // kx blocks [kb0, kb0 + nkbc) of TK (or kKB) columns handled by this launch (kx chunk)
  int l2pf;        // inverse pass: L2 prefetch hint of the strided B-side cp.async reads (0 none, 1/2/3 = 64/128/256 B)
  int lgzf;        // 512 kernels: log2 of the z groups that vary fastest in the tile order (then kx blocks, then
                   // the remaining z groups, then components); < 0 or >= log2(z groups): all z groups fastest
  // Peer-store transposes (FGD_PEER=1, nranks > 1): npeer = P and peer[s] is rank s's
  // z-pass buffer R, offset so that the S index of an element of y-slab s addresses its place in block
  // R[s][r] of that rank.  The forward pass then stores straight into the peers' R (NVLink peer
  // stores), the inverse pass loads from it; no separate transpose.  npeer = 0: B is the local S.
  int npeer;
  double2* peer[kMaxPeers];
};
// B-side address of the element with S index `sidx` in y-slab `yb` (= ky >> lg_nys)
// tile -> (z group, kx block, component) for the 512 kernels (nzt z groups, a power of two).  The
// tiles that run at the same time (consecutive indices) then cover 2^lgzf neighbouring z groups x
// many neighbouring kx blocks: contiguous bytes in flight on BOTH strided sides of the transpose
// (A rows along kx, B runs along z) instead of on the B side only.
__device__ __forceinline__ void y512_tile(const YArgs& a, int nzt, int lg_nzt, int tile, int* zt, int* kb, int* c) {
  const int lf = (a.lgzf < 0 || a.lgzf > lg_nzt) ? lg_nzt : a.lgzf;
  const int lo = tile & ((1 << lf) - 1), r1 = tile >> lf;
  const int kbi = r1 % a.nkbc, r2 = r1 / a.nkbc;
  const int hi = r2 & ((nzt >> lf) - 1);
  *zt = (hi << lf) | lo;
  *kb = a.kb0 + kbi;
  *c = r2 >> (lg_nzt - lf);
}
__device__ __forceinline__ double2* yb_ptr(const YArgs& a, int yb, size_t sidx) {
  return (a.npeer ? a.peer[yb] : a.B) + sidx;
}

struct YTile {
  int c, kx0, z0;
};
__device__ __forceinline__ YTile y_tile(const YArgs& a, int t) {
  const int nzt = a.Nz / a.TZ, nkb = a.nkbc;
  const int zt = t % nzt, r = t / nzt;
  return YTile{r / nkb, (a.kb0 + r % nkb) * a.TK, zt * a.TZ};
}

template <int N, bool INV>
__device__ __forceinline__ void y_issue(const YArgs& a, int t, double2* buf) {
  constexpr int LP = cline(N);
  const YTile T = y_tile(a, t);
  const int TZ = a.TZ, TK = a.TK;
  if (!INV) {
    for (int idx = threadIdx.x; idx < TZ * TK * N; idx += blockDim.x) {
      // order (kk, y, zz): contiguous runs of TK * N elements in layout A when TK = kKB
      const int kk = idx & (TK - 1), y = (idx >> a.lgTK) & (N - 1), zz = idx >> (a.lgTK + ilog2(N));
      const int kx = T.kx0 + kk, l = zz * TK + kk;
      if (kx < a.Hx) cp_async16(&buf[l * LP + SWZ(l, y)], &a.A[aidx(a.HxA, N, a.Nz, T.c, T.z0 + zz, y, kx)]);
    }
  } else {
    for (int idx = threadIdx.x; idx < TZ * TK * N; idx += blockDim.x) {
      const int zz = idx & (TZ - 1), ky = (idx >> a.lgTZ) & (N - 1), kk = idx >> (a.lgTZ + ilog2(N));
      const int kx = T.kx0 + kk, l = zz * TK + kk;
      if (kx < a.Hx)
        cp_async16(&buf[l * LP + SWZ(l, ky)],
                   yb_ptr(a, ky >> a.L.lg_nys, s_index(a.L, a.ncomp, a.Hx, T.c, kx, ky, T.z0 + zz)));
    }
  }
}

template <int N, bool INV>
__global__ void __launch_bounds__(256, 2) k_ypipe(YArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int LP = cline(N);
  const int NL = a.TZ * a.TK;
  pdl_trigger();
  double2* tws = sm + 2 * NL * LP;
  build_pass_tables<N, true>(tws, a.tw);
  const int ntiles = a.ncomp * a.nkbc * (a.Nz / a.TZ);
  int t = blockIdx.x;
  pdl_wait();
  if (t < ntiles) y_issue<N, INV>(a, t, sm);
  cp_async_commit();
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) y_issue<N, INV>(a, tn, sm + ((i + 1) & 1) * NL * LP);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* buf = sm + (i & 1) * NL * LP;
    fft_lines<N, INV, true>(buf, NL, LP, tws);
    __syncthreads();
    const YTile T = y_tile(a, t);
    const int TZ = a.TZ, TK = a.TK;
    if (!INV) {
      for (int idx = threadIdx.x; idx < TZ * TK * N; idx += blockDim.x) {
        const int zz = idx & (TZ - 1), ky = (idx >> a.lgTZ) & (N - 1), kk = idx >> (a.lgTZ + ilog2(N));
        const int kx = T.kx0 + kk, l = zz * TK + kk;
        if (kx < a.Hx)
          *yb_ptr(a, ky >> a.L.lg_nys, s_index(a.L, a.ncomp, a.Hx, T.c, kx, ky, T.z0 + zz)) = buf[l * LP + SWZ(l, ky)];
      }
    } else {
      for (int idx = threadIdx.x; idx < TZ * TK * N; idx += blockDim.x) {
        const int kk = idx & (TK - 1), y = (idx >> a.lgTK) & (N - 1), zz = idx >> (a.lgTK + ilog2(N));
        const int kx = T.kx0 + kk, l = zz * TK + kk;
        if (kx < a.Hx) a.A[aidx(a.HxA, N, a.Nz, T.c, T.z0 + zz, y, kx)] = buf[l * LP + SWZ(l, y)];
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
  const DevScalars* guard;
  double2* B;
  SlabL SL;
  int ky_off;          // global index of the first local ky (distributed y-slab)
  int Nyl;             // local ky rows
  int Nx, Ny, Hx, TL, scheme, lgTL;
  int kx0, nkx;        // kx in [kx0, kx0 + nkx) handled by this launch (kx chunk); Hx stays the layout extent
  double h[3], L[3];
  double qh[3];        // 0.25 / h_j      (host-side reciprocals: no FP64 division in the passes)
  double qh2[3];       // 1 / (16 h_j^2)
  double tpl[3];       // 2 pi / L_j
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
    k[0] = cscale(cmul(dx, cmul(cy, cz)), a.qh[0]);
    k[1] = cscale(cmul(cx, cmul(dy, cz)), a.qh[1]);
    k[2] = cscale(cmul(cx, cmul(cy, dz)), a.qh[2]);
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
        k[j] = make_double2(0.0, a.tpl[j] * m);
      }
    }
  }
}

// Per-axis factors of |k|^2.  Willot: f[0] = (2 - 2 cos th) / (16 h^2), f[1] = 2 + 2 cos th, so
// that |k|^2 = f0x f1y f1z + f1x f0y f1z + f1x f1y f0z.  Continuous: f[0] = (2 pi m / L)^2.
__device__ __forceinline__ void zaxis(const ZPArgs& a, int j, int m, int Nj, const double2* tw_s, double* f) {
  if (a.scheme == 1) {
    const double cs = tw_s ? tw_s[m].x : __ldg(&(j == 0 ? a.twx : a.twy)[m]).x;
    f[0] = (2.0 - 2.0 * cs) * a.qh2[j];
    f[1] = 2.0 + 2.0 * cs;
  } else {
    if ((Nj % 2 == 0) && m == Nj / 2) {
      f[0] = 0.0;
    } else {
      if (m > Nj / 2) m -= Nj;
      const double x = a.tpl[j] * m;
      f[0] = x * x;
    }
    f[1] = 0.0;
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
  const int kx = a.kx0 + t / nyt, ky0 = (t % nyt) * TL;
  for (int idx = threadIdx.x; idx < NC * TL * N; idx += blockDim.x) {
    const int kz = idx % N, rest = idx / N;
    const int ll = rest & (TL - 1), c = rest >> a.lgTL;
    cp_async16(&buf[(c * TL + ll) * LP + SWZ(c * TL + ll, kz)], &a.B[r_index(a.SL, NC, a.Hx, c, kx, ky0 + ll, kz)]);
  }
}

template <int N, int NC, int MODE>
__global__ void __launch_bounds__(192, 3) k_zpipe(ZPArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int LP = cline(N);
  const int TL = a.TL;
  double2* tws = sm + 2 * NC * TL * LP;    // e^{-2 pi i m/N} (symbol)
  double2* tpz = tws + N;                    // per-pass FFT twiddles
  pdl_trigger();
  load_table(tws, a.twz, N);
  build_pass_tables<N>(tpz, a.twz);
  const int nyt = a.Nyl / TL;
  const int ntiles = a.nkx * nyt;
  int t = blockIdx.x;
  pdl_wait();
  if (t < ntiles) z_issue<N, NC>(a, t, sm);
  cp_async_commit();
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) z_issue<N, NC>(a, tn, sm + ((i + 1) & 1) * NC * TL * LP);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* buf = sm + (i & 1) * NC * TL * LP;
    const int kx = a.kx0 + t / nyt, ky0 = (t % nyt) * TL;
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
      } else if (MODE == Z_GRAD) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double2* v = &buf[(c * TL + ll) * LP + SWZ(c * TL + ll, kz)];
          *v = cscale(cmul(k[c], *v), a.scale);
        }
      } else if (MODE == Z_DIV) {
        double2 t = make_double2(0.0, 0.0);
#pragma unroll
        for (int c = 0; c < 3; ++c) t = cadd(t, cmul(conjg(k[c]), buf[(c * TL + ll) * LP + SWZ(c * TL + ll, kz)]));
        buf[ll * LP + SWZ(ll, kz)] = cscale(t, a.scale);
        buf[(TL + ll) * LP + SWZ(TL + ll, kz)] = make_double2(0.0, 0.0);
        buf[(2 * TL + ll) * LP + SWZ(2 * TL + ll, kz)] = make_double2(0.0, 0.0);
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
// Z pass for Nz = 256 as a register four-step FFT (256 = 16 x 16)
// ---------------------------------------------------------------------------------------------
// A z line is owned by 16 threads (half a warp); n = n1 + 16 n2, k = k2 + 16 k1.
//   forward: thread t (= n1) loads x[t + 16 j] straight from global memory (256 contiguous bytes
//   per half warp and j), DFT16 over j in registers, twiddle W256^{t k2}, 16 x 16 transpose
//   through shared memory, DFT16 -> thread t holds X[t + 16 k1], k1 = 0..15;
//   inverse: the mirror image, starting from the same "kz = t mod 16" layout and ending with a
//   coalesced store of z[t + 16 n2].
// Shared-memory traffic per element: 2 accesses per transform, +4 for the 6-component projection
// (which mixes the lines of one (kx, ky) and so goes through shared memory), against ~8 per
// transform for the three-pass Stockham of k_zpipe.  A line occupies 16 rows of 17 slots, so that
// row and column accesses of the transpose are both free of bank conflicts; the padded position of
// frequency kz is kz + kz / 16.
constexpr int kZRowPad = 17;
constexpr int kZLine = 16 * kZRowPad;

// PF (one slab: contiguous z lines): the two lines of each warp arrive by 1-D bulk copies (4 KB each)
// in the first 256 slots of their line buffers, completing on a per-warp mbarrier; the copies of the
// NEXT tile are issued once the warp has read the last exchange of the current one (see k_zreg512w).
template <int NC, int MODE, bool PF = false>
__global__ void __launch_bounds__(NC == 6 ? 96 : 128) __maxnreg__(NC == 6 ? 128 : 128) k_zreg256(ZPArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 256;
  const int TL = a.TL;
  const int nl = NC * TL;                       // blockDim.x == 16 * nl
  double2* tw = sm + (size_t)nl * kZLine;       // W256^{t k2} at (k2 - 1) * 16 + t
  double2* tws = tw + 240;                      // e^{-2 pi i m / 256} (symbol)
  uint64_t* bars = reinterpret_cast<uint64_t*>(tws + N);   // PF: one mbarrier per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  for (int i = threadIdx.x; i < 240; i += blockDim.x) tw[i] = __ldg(&a.twz[(i & 15) * (1 + (i >> 4))]);
  load_table(tws, a.twz, N);
  if (PF && lane == 0) {
    mbar_init(&bars[warp], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  const int line = threadIdx.x >> 4, t = threadIdx.x & 15;
  const int c = line >> a.lgTL, ll = line & (TL - 1);
  double2* ls = sm + (size_t)line * kZLine;
  const int nyt = a.Nyl / TL;
  const int ntiles = a.nkx * nyt;
  auto prefetch = [&](int tl) {
    const int kxp = a.kx0 + tl / nyt, kyp = (tl % nyt) * TL;
    mbar_arrive_expect_tx(&bars[warp], 2 * N * (unsigned)sizeof(double2));
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int lq = 2 * warp + q;
      bulk_g2s(sm + (size_t)lq * kZLine, a.B + r_index(a.SL, NC, a.Hx, lq >> a.lgTL, kxp, kyp + (lq & (TL - 1)), 0),
               N * (unsigned)sizeof(double2), &bars[warp]);
    }
  };
  unsigned phase = 0;
  if (PF && lane == 0 && (int)blockIdx.x < ntiles) prefetch(blockIdx.x);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int kx = a.kx0 + tile / nyt, ky0 = (tile % nyt) * TL;
    const int kyl = ky0 + ll;
    // z -> offset from the line start: z-slab block (z >> lg_nzs) of stride BS, then z within it
    double2* Bl = a.B + r_index(a.SL, NC, a.Hx, c, kx, kyl, 0);
    const int BS = NC * a.Hx * a.SL.nys * a.SL.nzs, zm = a.SL.nzs - 1, lgz = a.SL.lg_nzs;
    double2 v[16];
    if (PF) {
      mbar_wait(&bars[warp], phase);
      phase ^= 1u;
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = ls[t + 16 * j];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int z = t + 16 * j;
        v[j] = __ldcg(Bl + ((z >> lgz) * BS + (z & zm)));
      }
    }
    // ---- forward ----
    dft16<false>(v);
#pragma unroll
    for (int k2 = 1; k2 < 16; ++k2) v[k2] = cmul(v[k2], ld_tw(tw + (k2 - 1) * 16 + t));
    __syncwarp();
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) ls[k2 * kZRowPad + t] = v[k2];
    __syncwarp();
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) v[n1] = ls[t * kZRowPad + n1];
    dft16<false>(v);                            // v[k1] = X[t + 16 k1]
    // ---- spectral multiply ----
    const int ky = kyl + a.ky_off;
    if (MODE == Z_PRECOND) {
      // Pointwise multiply, one rolled loop over this thread's own column of the line buffer (no
      // cross-thread traffic; keeps the 16 divisions out of the unrolled register code).
      // |k|^2 from per-axis factors (same value as |zsymbol|^2 up to rounding):
      //   Willot: |k_1|^2 = (2 - 2 cos th1)(2 + 2 cos th2)(2 + 2 cos th3) / (16 h1^2), cyclic;
      //   continuous: sum_j (2 pi m_j / L_j)^2 with the Nyquist index zeroed (A-06).
      __syncwarp();
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) ls[k1 * kZRowPad + t] = v[k1];
      double fx[2], fy[2];
      zaxis(a, 0, kx, a.Nx, nullptr, fx);
      zaxis(a, 1, ky, a.Ny, nullptr, fy);
#pragma unroll 1
      for (int k1 = 0; k1 < 16; ++k1) {
        double fz[2];
        zaxis(a, 2, t + 16 * k1, N, tws, fz);
        const double k2 = a.scheme == 1 ? (fx[0] * fy[1] * fz[1] + fx[1] * fy[0] * fz[1] + fx[1] * fy[1] * fz[0])
                                        : fx[0] + fy[0] + fz[0];
        ls[k1 * kZRowPad + t] = cscale(ls[k1 * kZRowPad + t], a.scale / (1.0 + a.mean_ell2 * k2));
      }
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) v[k1] = ls[k1 * kZRowPad + t];
    } else {
      __syncwarp();
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) ls[k1 * kZRowPad + t] = v[k1];
      __syncthreads();
      // Willot symbol with the (kx, ky) factors hoisted (one ky per tile when TL = 1):
      // k0 = [(e^{ith1}-1)(1+e^{ith2}) qh0] (1+e^{ith3}), k1 = [(1+e^{ith1})(e^{ith2}-1) qh1] (1+e^{ith3}),
      // k2 = [(1+e^{ith1})(1+e^{ith2}) qh2] (e^{ith3}-1)
      double2 P0 = make_double2(0.0, 0.0), P1 = P0, P2 = P0;
      const bool hoist = a.scheme == 1 && TL == 1;
      if (hoist) {
        const double2 wx = __ldg(&a.twx[kx]), wy = __ldg(&a.twy[ky0 + a.ky_off]);
        const double2 ex = make_double2(wx.x, -wx.y), ey = make_double2(wy.x, -wy.y);
        const double2 dx = make_double2(ex.x - 1.0, ex.y), dy = make_double2(ey.x - 1.0, ey.y);
        const double2 cx = make_double2(ex.x + 1.0, ex.y), cy = make_double2(ey.x + 1.0, ey.y);
        P0 = cscale(cmul(dx, cy), a.qh[0]);
        P1 = cscale(cmul(cx, dy), a.qh[1]);
        P2 = cscale(cmul(cx, cy), a.qh[2]);
      }
      for (int idx = threadIdx.x; idx < TL * N; idx += blockDim.x) {
        const int kz = idx & (N - 1), l2 = idx >> 8;
        const int kyg = ky0 + l2 + a.ky_off;
        double2 k[3];
        if (hoist) {
          const double2 wz = tws[kz];
          const double2 cz = make_double2(wz.x + 1.0, -wz.y), dz = make_double2(wz.x - 1.0, -wz.y);
          k[0] = cmul(P0, cz);
          k[1] = cmul(P1, cz);
          k[2] = cmul(P2, dz);
        } else {
          zsymbol(a, N, kx, kyg, kz, k, tws);
        }
        double2* pv[6];
#pragma unroll
        for (int cc = 0; cc < 6; ++cc) pv[cc] = &sm[(size_t)(cc * TL + l2) * kZLine + kz + (kz >> 4)];
        project6(a, pv, k, kx == 0 && kyg == 0 && kz == 0);
      }
      __syncthreads();
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) v[k1] = ls[k1 * kZRowPad + t];
    }
    // ---- inverse ----
    dft16<true>(v);                             // v[n1] = U[k2 = t][n1]
#pragma unroll
    for (int n1 = 1; n1 < 16; ++n1) {
      double2 w = ld_tw(tw + (n1 - 1) * 16 + t);
      w.y = -w.y;
      v[n1] = cmul(v[n1], w);
    }
    __syncwarp();
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) ls[n1 * kZRowPad + t] = v[n1];
    __syncwarp();
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) v[k2] = ls[t * kZRowPad + k2];
    if (PF) {
      // the warp's line buffers are free from here on: refill them with the next tile's lines
      __syncwarp();
      if (lane == 0 && tile + (int)gridDim.x < ntiles) {
        fence_proxy_async();
        prefetch(tile + gridDim.x);
      }
    }
    dft16<true>(v);                             // v[n2] = z[t + 16 n2]
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) {
      const int z = t + 16 * n2;
      Bl[(z >> lgz) * BS + (z & zm)] = v[n2];
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Z pass with the Galerkin projection for the Willot scheme, Nz = 256: factorised form
// ---------------------------------------------------------------------------------------------
// Along a z line (fixed kx, ky) the rotated symbol factors as k_j(kz) = A_j m_j(kz) with per-line
// constants A_0 = (e^{ith1}-1)(1+e^{ith2})/(4h1), A_1 = (1+e^{ith1})(e^{ith2}-1)/(4h2),
// A_2 = (1+e^{ith1})(1+e^{ith2})/(4h3) and m_0 = m_1 = 1 + e^{ith3}, m_2 = e^{ith3} - 1 (A-04).
// Multiplying by e^{+ith3} is a shift z -> z+1, by e^{-ith3} a shift z -> z-1.  G^* needs tau only
// through t = tau^ conj(k) and returns sym(u (x) k):
//   t_i = F_z[d_i],   d_i(z) = sum_j conj(A_j) (tau_ij(z) + tau_ij(z-1))   (j = 0, 1)
//                                      + conj(A_2) (tau_i2(z-1) - tau_i2(z))
//   u_i = (2/|k|^2)(t_i - k_i s / (2|k|^2)),  s = conj(k) . t          (per kz)
//   U_i = F_z^{-1}[u_i],  eps_ij(z) = (A_j (U_i * m_j)(z) + A_i (U_j * m_i)(z)) / 2
//   with (U * m_0)(z) = U(z) + U(z+1), (U * m_2)(z) = U(z+1) - U(z).
// So each line transforms 3 components each way instead of 6 (exactly the same operator; only the
// association order of the sums changes).  Opt-in (FGD_ZFAC=1), see pipe_z.  The zero frequency (line kx = ky = 0, kz = 0) takes the
// mask branch: eps_c += mask_c (sum_z tau_c - N shift_c) scale on every z of that line.
__global__ void __launch_bounds__(96, 5) k_zfac256(ZPArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 256;
  constexpr double HS2 = 0.70710678118654752440;   // sqrt(2)/2 = 1/sqrt(2)
  double2* tw = sm + 6 * kZLine;                    // W256^{t k2} at (k2 - 1) * 16 + t
  double2* tws = tw + 240;                          // e^{-2 pi i m / 256}
  pdl_trigger();
  for (int i = threadIdx.x; i < 240; i += blockDim.x) tw[i] = __ldg(&a.twz[(i & 15) * (1 + (i >> 4))]);
  load_table(tws, a.twz, N);
  __syncthreads();
  pdl_wait();
  const int line = threadIdx.x >> 4, t = threadIdx.x & 15;   // line = Mandel component in phases A, B, G
  double2* ls = sm + (size_t)line * kZLine;
  const int ntiles = a.nkx * a.Nyl;
  const int BS = 6 * a.Hx * a.SL.nys * a.SL.nzs, zm = a.SL.nzs - 1, lgz = a.SL.lg_nzs;
  auto slot = [](int z) { return z + (z >> 4); };
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int kx = a.kx0 + tile / a.Nyl, kyl = tile % a.Nyl;
    const int ky = kyl + a.ky_off;
    double2* Bl = a.B + r_index(a.SL, 6, a.Hx, line, kx, kyl, 0);
    // per-line symbol factors
    const double2 wx = __ldg(&a.twx[kx]), wy = __ldg(&a.twy[ky]);
    const double2 ex = make_double2(wx.x, -wx.y), ey = make_double2(wy.x, -wy.y);
    const double2 A0 = cscale(cmul(make_double2(ex.x - 1.0, ex.y), make_double2(ey.x + 1.0, ey.y)), a.qh[0]);
    const double2 A1 = cscale(cmul(make_double2(ex.x + 1.0, ex.y), make_double2(ey.x - 1.0, ey.y)), a.qh[1]);
    const double2 A2 = cscale(cmul(make_double2(ex.x + 1.0, ex.y), make_double2(ey.x + 1.0, ey.y)), a.qh[2]);
    // ---- A: load tau_c(z), z = t + 16 j; B: to shared memory (natural z) ----
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int z = t + 16 * j;
      v[j] = __ldcg(Bl + ((z >> lgz) * BS + (z & zm)));
    }
    double2 tsum = make_double2(0.0, 0.0);
    const bool dcline = kx == 0 && ky == 0;
    if (dcline) {
#pragma unroll
      for (int j = 0; j < 16; ++j) tsum = cadd(tsum, v[j]);
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) {
        tsum.x += __shfl_xor_sync(0xffffffffu, tsum.x, o, 16);
        tsum.y += __shfl_xor_sync(0xffffffffu, tsum.y, o, 16);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) ls[slot(t + 16 * j)] = v[j];
    __syncthreads();
    // ---- C: d_i(z) for i = line < 3 ----
    const int i = line;
    if (i < 3) {
      // tensor row i in Mandel storage: (comp, factor) of tau_i0, tau_i1, tau_i2
      const int c0 = i == 0 ? 0 : i == 1 ? 5 : 4;
      const int c1 = i == 0 ? 5 : i == 1 ? 1 : 3;
      const int c2 = i == 0 ? 4 : i == 1 ? 3 : 2;
      const double f0 = i == 0 ? 1.0 : HS2, f1 = i == 1 ? 1.0 : HS2, f2 = i == 2 ? 1.0 : HS2;
      const double2 B0 = cscale(conjg(A0), f0), B1 = cscale(conjg(A1), f1), B2 = cscale(conjg(A2), f2);
      const double2* L0 = sm + (size_t)c0 * kZLine;
      const double2* L1 = sm + (size_t)c1 * kZLine;
      const double2* L2 = sm + (size_t)c2 * kZLine;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int z = t + 16 * j, zp = (z - 1) & (N - 1);
        const double2 g0 = cadd(L0[slot(z)], L0[slot(zp)]);
        const double2 g1 = cadd(L1[slot(z)], L1[slot(zp)]);
        const double2 g2 = csub(L2[slot(zp)], L2[slot(z)]);
        v[j] = cadd(cadd(cmul(B0, g0), cmul(B1, g1)), cmul(B2, g2));
      }
    }
    __syncthreads();
    // ---- D: forward z FFT of d_i (lines 0..2) -> t_i(kz = t + 16 k1) ----
    if (i < 3) {
      dft16<false>(v);
#pragma unroll
      for (int k2 = 1; k2 < 16; ++k2) v[k2] = cmul(v[k2], ld_tw(tw + (k2 - 1) * 16 + t));
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) ls[k2 * kZRowPad + t] = v[k2];
      __syncwarp(0x0000ffffu << (16 * (threadIdx.x >> 4 & 1)));
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) v[n1] = ls[t * kZRowPad + n1];
      dft16<false>(v);
      __syncwarp(0x0000ffffu << (16 * (threadIdx.x >> 4 & 1)));
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) ls[slot(t + 16 * k1)] = v[k1];
    }
    __syncthreads();
    // ---- E: per kz: u = (2/|k|^2)(t - k s/(2|k|^2)) scale, in place on lines 0..2 ----
    for (int kz = threadIdx.x; kz < N; kz += blockDim.x) {
      const double2 wz = tws[kz];
      const double2 cz = make_double2(wz.x + 1.0, -wz.y), dz = make_double2(wz.x - 1.0, -wz.y);
      const double2 k0 = cmul(A0, cz), k1 = cmul(A1, cz), k2 = cmul(A2, dz);
      const double kk = k0.x * k0.x + k0.y * k0.y + k1.x * k1.x + k1.y * k1.y + k2.x * k2.x + k2.y * k2.y;
      double2* p0 = sm + slot(kz);
      double2* p1 = p0 + kZLine;
      double2* p2 = p1 + kZLine;
      if (kk == 0.0) {
        *p0 = *p1 = *p2 = make_double2(0.0, 0.0);
      } else {
        const double2 t0 = *p0, t1 = *p1, t2 = *p2;
        const double2 sv = cadd(cadd(cmul(conjg(k0), t0), cmul(conjg(k1), t1)), cmul(conjg(k2), t2));
        const double inv = 1.0 / kk;
        const double2 hs = cscale(sv, 0.5 * inv);
        const double f = 2.0 * inv * a.scale;
        *p0 = cscale(csub(t0, cmul(k0, hs)), f);
        *p1 = cscale(csub(t1, cmul(k1, hs)), f);
        *p2 = cscale(csub(t2, cmul(k2, hs)), f);
      }
    }
    __syncthreads();
    // ---- F: inverse z FFT of u_i -> U_i(z), back to shared memory (natural z) ----
    if (i < 3) {
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) v[k1] = ls[slot(t + 16 * k1)];
      dft16<true>(v);
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) {
        double2 wv = ld_tw(tw + (n1 - 1) * 16 + t);
        wv.y = -wv.y;
        v[n1] = cmul(v[n1], wv);
      }
      __syncwarp(0x0000ffffu << (16 * (threadIdx.x >> 4 & 1)));
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) ls[n1 * kZRowPad + t] = v[n1];
      __syncwarp(0x0000ffffu << (16 * (threadIdx.x >> 4 & 1)));
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) v[k2] = ls[t * kZRowPad + k2];
      dft16<true>(v);                               // v[n2] = U_i(z = t + 16 n2)
      __syncwarp(0x0000ffffu << (16 * (threadIdx.x >> 4 & 1)));
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2) ls[slot(t + 16 * n2)] = v[n2];
    }
    __syncthreads();
    // ---- G: eps_c(z) from U (and the zero frequency on the kx = ky = 0 line), store ----
    {
      const int c = line;
      const double2* U0 = sm;
      const double2* U1 = sm + kZLine;
      const double2* U2 = sm + 2 * kZLine;
      double2 dcv = make_double2(0.0, 0.0);
      if (dcline && a.mask[c]) dcv = cscale(make_double2(tsum.x - a.shift[c], tsum.y), a.scale);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int z = t + 16 * j, zn = (z + 1) & (N - 1);
        const int s0 = slot(z), s1 = slot(zn);
        double2 e;
        if (c == 0) {
          e = cmul(A0, cadd(U0[s0], U0[s1]));
        } else if (c == 1) {
          e = cmul(A1, cadd(U1[s0], U1[s1]));
        } else if (c == 2) {
          e = cmul(A2, csub(U2[s1], U2[s0]));
        } else if (c == 3) {   // sqrt2 eps_12 = (A2 (U1 * m2) + A1 (U2 * m1)) / sqrt2
          e = cscale(cadd(cmul(A2, csub(U1[s1], U1[s0])), cmul(A1, cadd(U2[s0], U2[s1]))), HS2);
        } else if (c == 4) {   // sqrt2 eps_02
          e = cscale(cadd(cmul(A2, csub(U0[s1], U0[s0])), cmul(A0, cadd(U2[s0], U2[s1]))), HS2);
        } else {               // sqrt2 eps_01
          e = cscale(cadd(cmul(A1, cadd(U0[s0], U0[s1])), cmul(A0, cadd(U1[s0], U1[s1]))), HS2);
        }
        v[j] = cadd(e, dcv);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int z = t + 16 * j;
        Bl[(z >> lgz) * BS + (z & zm)] = v[j];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Y pass for Ny = 256 as a register four-step FFT (256 = 16 x 16), as the z pass below
// ---------------------------------------------------------------------------------------------
// Tile = (c, kx pair kx0 = kKB kb, TZ planes z0..): 2 TZ lines; warp w handles plane z0 + w, its
// half warps the two kx of the pair, so that the loads / stores on the A side (kKB x Ny
// contiguous per plane) are 512 B per warp instruction.  The B side (z fastest, runs of TZ x 16 B)
// goes through the line buffers in shared memory (line l = kl TZ + zz, conflict-free pitch).
//   fwd: global A -> registers -> DFT16, twiddle, 16 x 16 transpose (smem), DFT16 -> smem -> B
//   inv: B -> smem (cp.async) -> registers -> DFT16, twiddle, transpose (smem), DFT16 -> A
constexpr int kYLine = kZLine + 2;   // max pitch between lines (see ypitch)
// Line pitch of the y-pass line buffers: the B-side loops walk (z2 fastest, then ky), so 8
// consecutive threads touch TZ lines x 8/TZ consecutive ky: pitch = 1 mod 8 for TZ = 8 and
// 2 mod 8 for TZ = 4 keep those 8 16-B accesses in distinct bank groups.
__host__ __device__ constexpr int ypitch(int base, int TZ) { return base + (TZ >= 8 ? 1 : 2); }

// fwd: A rows go straight from HBM into registers (512 B per warp instruction); the line buffers
//      hold the exchange and the B-side output staging.
// inv: the NEXT tile's B-side input is staged by cp.async (double buffer, stage[b][l][slot(ky)])
//      while the current tile is transformed; the current stage buffer doubles as the exchange
//      buffer once its column has been read into registers.
__device__ __forceinline__ void y256_issue_inv(const YArgs& a, int tile, double2* buf) {
  constexpr int N = 256;
  const int TZ = a.TZ;
  const int nzt = a.Nz / TZ, nkb = a.nkbc;
  const int zt = tile % nzt, r = tile / nzt, kb = a.kb0 + r % nkb, c = r / nkb;
  const int z0 = zt * TZ, kx0 = kb * kKB;
  for (int idx = threadIdx.x; idx < 2 * N * TZ; idx += blockDim.x) {
    const int z2 = idx % TZ, ky = (idx / TZ) & (N - 1), k2l = idx / (TZ * N);
    const int kxo = kx0 + k2l;
    if (kxo < a.Hx)
      cp_async16_l2(&buf[(size_t)(k2l * TZ + z2) * ypitch(kZLine, TZ) + ky + (ky >> 4)],
                    yb_ptr(a, ky >> a.L.lg_nys, s_index(a.L, a.ncomp, a.Hx, c, kxo, ky, z0 + z2)), a.l2pf);
  }
}

template <bool INV>
__global__ void __launch_bounds__(256, 2) k_yreg256(YArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 256;
  const int TZ = a.TZ;                              // blockDim.x == 32 * TZ
  const int LPY = ypitch(kZLine, TZ);
  const size_t buf_sz = (size_t)2 * TZ * LPY;       // fwd: one line buffer; inv: two stage buffers
  double2* tw = sm + (INV ? 2 : 1) * buf_sz;        // W256^{t k2} at (k2 - 1) * 16 + t
  pdl_trigger();
  for (int i = threadIdx.x; i < 240; i += blockDim.x) tw[i] = __ldg(&a.tw[(i & 15) * (1 + (i >> 4))]);
  pdl_wait();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kl = lane >> 4, t = lane & 15, zz = w;
  const int l = kl * TZ + zz;
  const int nzt = a.Nz / TZ, nkb = a.nkbc;
  const int ntiles = a.ncomp * nkb * nzt;
  int tile = blockIdx.x;
  if (INV) {
    if (tile < ntiles) y256_issue_inv(a, tile, sm);
    cp_async_commit();
  }
  __syncthreads();
  double2 v[16];
  // fwd: the A-side loads of the next tile are issued into v as soon as v is dead (before the
  // B-side stores of the current tile), so they are in flight while the stores drain
  auto arow_of = [&](int tl) {
    const int zt = tl % nzt, r = tl / nzt, kb = a.kb0 + r % nkb, c = r / nkb;
    return a.A + aidx(a.HxA, N, a.Nz, c, zt * TZ + zz, 0, kb * kKB) + kl;
  };
  if (!INV && tile < ntiles) {
    const double2* A0 = arow_of(tile);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __ldcs(A0 + kKB * (t + 16 * j));
  }
  for (int i = 0; tile < ntiles; ++i, tile += gridDim.x) {
    const int zt = tile % nzt, r = tile / nzt, kb = a.kb0 + r % nkb, c = r / nkb;
    const int z0 = zt * TZ, kx0 = kb * kKB, kx = kx0 + kl;
    double2* Arow = a.A + aidx(a.HxA, N, a.Nz, c, z0 + zz, 0, kx0) + kl;   // element y at Arow[kKB * y]
    if (!INV) {
      double2* ls = sm + (size_t)l * LPY;
      dft16<false>(v);
#pragma unroll
      for (int k2 = 1; k2 < 16; ++k2) v[k2] = cmul(v[k2], ld_tw(tw + (k2 - 1) * 16 + t));
      __syncwarp();
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) ls[k2 * kZRowPad + t] = v[k2];
      __syncwarp();
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) v[n1] = ls[t * kZRowPad + n1];
      dft16<false>(v);                              // v[k1] = X[ky = t + 16 k1]
      __syncwarp();
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) ls[k1 * kZRowPad + t] = v[k1];
      __syncthreads();
      const int tn = tile + gridDim.x;
      if (tn < ntiles) {
        const double2* An = arow_of(tn);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __ldcs(An + kKB * (t + 16 * j));
      }
      // B side: z fastest
      for (int idx = threadIdx.x; idx < 2 * N * TZ; idx += blockDim.x) {
        const int z2 = idx % TZ, ky = (idx / TZ) & (N - 1), k2l = idx / (TZ * N);
        const int kxo = kx0 + k2l;
        if (kxo < a.Hx)
          *yb_ptr(a, ky >> a.L.lg_nys, s_index(a.L, a.ncomp, a.Hx, c, kxo, ky, z0 + z2)) =
              sm[(size_t)(k2l * TZ + z2) * LPY + ky + (ky >> 4)];
      }
      __syncthreads();
    } else {
      const int tn = tile + gridDim.x;
      if (tn < ntiles) y256_issue_inv(a, tn, sm + ((i + 1) & 1) * buf_sz);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      double2* ls = sm + (i & 1) * buf_sz + (size_t)l * LPY;
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) v[k1] = ls[k1 * kZRowPad + t];   // X[ky = t + 16 k1]
      dft16<true>(v);                               // v[n1] = U[k2 = t][n1]
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) {
        double2 wv = ld_tw(tw + (n1 - 1) * 16 + t);
        wv.y = -wv.y;
        v[n1] = cmul(v[n1], wv);
      }
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) ls[n1 * kZRowPad + t] = v[n1];
      __syncwarp();
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) v[k2] = ls[t * kZRowPad + k2];
      dft16<true>(v);                               // v[n2] = y-line value at y = t + 16 n2
      if (kx < a.Hx) {
#pragma unroll
        for (int n2 = 0; n2 < 16; ++n2) Arow[kKB * (t + 16 * n2)] = v[n2];
      }
      __syncthreads();                              // stage buffer free for the next issue
    }
  }
  if (INV) cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// 512-point lines as a register FFT 8 x 8 x 8: 64 threads per line, 8 points per thread, two
// shared-memory exchanges.  n = t + 64 j, t = t1 + 8 t2; k = ka + 8 kb + 64 kc:
//   S1 (thread t):           DFT8 over j -> ka, twiddle W512^{t ka}
//   S2 (thread ka + 8 t1):   DFT8 over t2 -> kb, twiddle W64^{t1 kb}
//   S3 (thread ka + 8 kb):   DFT8 over t1 -> kc        => thread t holds X[t + 64 kc]
// The inverse is the same algorithm with conjugate twiddles, applied to that layout, and returns
// thread t holding x[t + 64 m] -- the coalesced store layout.  Exchange slots (pitch 65, both
// sides conflict free):  E1 (ka, t) -> ka * 65 + t;  E2 (kb, ka, t1) -> kb * 65 + ka + 8 t1.
// Calls __syncthreads(): every thread of the CTA must call it.
constexpr int k512Line = 8 * 65;

constexpr bool kFft512TwProducts = true;

template <bool INV>
__device__ __forceinline__ void fft512_reg(double2 (&v)[8], int t, double2* ls, const double2* tw1,
                                           const double2* tw2, int bar, int nbar) {
  // the exchanges only involve the warps that carry this line: named barrier `bar` over `nbar` threads
  auto sync = [&]() {
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nbar) : "memory");
    FGD_JIT();
  };
  dft8<INV>(v);
  // twiddles W^{1,2,4} from the table, W^{3,5,6,7} as products (3 shared loads instead of 7 per
  // stage: the 512 y/z passes are shared-memory bound; products round to ~2 ulp)
  auto twiddle7 = [&](const double2* tab, int stride) {
    double2 w1 = ld_tw(tab), w2 = ld_tw(tab + stride), w4 = ld_tw(tab + 3 * stride);
    if (INV) {
      w1.y = -w1.y;
      w2.y = -w2.y;
      w4.y = -w4.y;
    }
    const double2 w3 = cmul(w1, w2);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    v[4] = cmul(v[4], w4);
    v[5] = cmul(v[5], cmul(w4, w1));
    v[6] = cmul(v[6], cmul(w4, w2));
    v[7] = cmul(v[7], cmul(w4, w3));
  };
  if (kFft512TwProducts) {
    twiddle7(tw1 + t, 64);
  } else {
#pragma unroll
    for (int ka = 1; ka < 8; ++ka) {
      double2 w = ld_tw(tw1 + (ka - 1) * 64 + t);
      if (INV) w.y = -w.y;
      v[ka] = cmul(v[ka], w);
    }
  }
#pragma unroll
  for (int ka = 0; ka < 8; ++ka) ls[ka * 65 + t] = v[ka];
  sync();
  const int ka = t & 7, hi = t >> 3;
#pragma unroll
  for (int t2 = 0; t2 < 8; ++t2) v[t2] = ls[ka * 65 + hi + 8 * t2];
  sync();
  dft8<INV>(v);
  if (kFft512TwProducts) {
    twiddle7(tw2 + hi, 8);
  } else {
#pragma unroll
    for (int kb = 1; kb < 8; ++kb) {
      double2 w = ld_tw(tw2 + (kb - 1) * 8 + hi);
      if (INV) w.y = -w.y;
      v[kb] = cmul(v[kb], w);
    }
  }
#pragma unroll
  for (int kb = 0; kb < 8; ++kb) ls[kb * 65 + ka + 8 * hi] = v[kb];
  sync();
#pragma unroll
  for (int t1 = 0; t1 < 8; ++t1) v[t1] = ls[hi * 65 + ka + 8 * t1];
  sync();
  dft8<INV>(v);
}

// twiddle tables of fft512_reg in shared memory: tw1[(ka-1)*64 + t] = W512^{t ka}, tw2[(kb-1)*8 + t1] = W64^{t1 kb}
__device__ __forceinline__ void fft512_tables(double2* tw1, double2* tw2, const double2* __restrict__ w512) {
  for (int i = threadIdx.x; i < 448; i += blockDim.x) tw1[i] = __ldg(&w512[(i & 63) * (1 + (i >> 6))]);
  for (int i = threadIdx.x; i < 56; i += blockDim.x) tw2[i] = __ldg(&w512[8 * (i & 7) * (1 + (i >> 3))]);
}

// Z pass, Nz = 512: one (kx, ky) per tile, NC lines of 64 threads.
template <int NC, int MODE>
__global__ void __launch_bounds__(NC * 64, NC == 6 ? 2 : 8) k_zreg512(ZPArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 512;
  double2* tw1 = sm + (size_t)NC * k512Line;
  double2* tw2 = tw1 + 448;
  double2* tws = tw2 + 56;                      // e^{-2 pi i m / 512} (symbol)
  pdl_trigger();
  fft512_tables(tw1, tw2, a.twz);
  load_table(tws, a.twz, N);
  __syncthreads();
  pdl_wait();
  const int c = threadIdx.x >> 6, t = threadIdx.x & 63;
  double2* ls = sm + (size_t)c * k512Line;
  const int ntiles = a.nkx * a.Nyl;
  const int BS = NC * a.Hx * a.SL.nys * a.SL.nzs, zm = a.SL.nzs - 1, lgz = a.SL.lg_nzs;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int kx = a.kx0 + tile / a.Nyl, kyl = tile % a.Nyl;
    double2* Bl = a.B + r_index(a.SL, NC, a.Hx, c, kx, kyl, 0);
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int z = t + 64 * j;
      v[j] = __ldcg(Bl + ((z >> lgz) * BS + (z & zm)));
    }
    fft512_reg<false>(v, t, ls, tw1, tw2, 1 + c, 64);   // v[kc] = X[t + 64 kc]
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) ls[kc * 65 + t] = v[kc];
    __syncthreads();
    const int ky = kyl + a.ky_off;
    // Willot symbol with the (kx, ky) factors hoisted out of the kz loop (one line per tile):
    // k0 = P0 (1+e^{ith3}), k1 = P1 (1+e^{ith3}), k2 = P2 (e^{ith3}-1)
    const bool hoist = a.scheme == 1;
    double2 P0 = make_double2(0.0, 0.0), P1 = P0, P2 = P0;
    if (hoist) {
      const double2 wx = __ldg(&a.twx[kx]), wy = __ldg(&a.twy[ky]);
      const double2 ex = make_double2(wx.x, -wx.y), ey = make_double2(wy.x, -wy.y);
      const double2 dx = make_double2(ex.x - 1.0, ex.y), dy = make_double2(ey.x - 1.0, ey.y);
      const double2 cx = make_double2(ex.x + 1.0, ex.y), cy = make_double2(ey.x + 1.0, ey.y);
      P0 = cscale(cmul(dx, cy), a.qh[0]);
      P1 = cscale(cmul(cx, dy), a.qh[1]);
      P2 = cscale(cmul(cx, cy), a.qh[2]);
    }
    for (int kz = threadIdx.x; kz < N; kz += blockDim.x) {
      double2 k[3];
      if (hoist) {
        const double2 wz = tws[kz];
        const double2 cz = make_double2(wz.x + 1.0, -wz.y), dz = make_double2(wz.x - 1.0, -wz.y);
        k[0] = cmul(P0, cz);
        k[1] = cmul(P1, cz);
        k[2] = cmul(P2, dz);
      } else {
        zsymbol(a, N, kx, ky, kz, k, tws);
      }
      const int slot = (kz >> 6) * 65 + (kz & 63);
      if (MODE == Z_PRECOND) {
        const double k2 = k[0].x * k[0].x + k[0].y * k[0].y + k[1].x * k[1].x + k[1].y * k[1].y + k[2].x * k[2].x +
                          k[2].y * k[2].y;
        sm[slot] = cscale(sm[slot], a.scale / (1.0 + a.mean_ell2 * k2));
      } else {
        double2* pv[6];
#pragma unroll
        for (int cc = 0; cc < 6; ++cc) pv[cc] = &sm[(size_t)cc * k512Line + slot];
        project6(a, pv, k, kx == 0 && ky == 0 && kz == 0);
      }
    }
    __syncthreads();
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) v[kc] = ls[kc * 65 + t];
    __syncthreads();
    fft512_reg<true>(v, t, ls, tw1, tw2, 1 + c, 64);    // v[m] = z[t + 64 m]
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int z = t + 64 * m;
      Bl[(z >> lgz) * BS + (z & zm)] = v[m];
    }
  }
}

// Z pass, Nz = 512, wide plan: 16 threads per line, 32 points per thread and ONE shared-memory
// exchange per transform (512 = 32 x 16), instead of the 8 x 8 x 8 plan of k_zreg512 (64 threads
// per line, two exchanges per transform).  Thread t loads x[t + 16 m] (m < 32, 256 B per
// half-warp instruction), runs a register DFT32 over m, multiplies by W512^{t k2}, and one
// transpose through the line buffer (32 rows k2 x 16 columns t, pitch 17: row and column
// accesses conflict free) gives it rows k2 = t and t + 16, whose DFT16 over t yields
// X[k2 + 32 k1].  The inverse runs the mirror image and ends in the coalesced store layout.
// Shared accesses per element: 2 per transform + 4 for the six-component projection (was 4 + 4).
// Line buffer of 512 slots, no padding: exchange element (row r, column n) at r * 16 + (n ^ (r & 15))
// (XOR swizzle: row accesses and column accesses are both conflict free), staged frequency kz at kz;
// twiddle W512^{t k2} at (k2 - 1) * 16 + (t ^ (k2 & 15)).  55.75 KB per six-component CTA, so four
// CTAs fit on an SM.
constexpr int kZ5Line = 512;
__device__ __forceinline__ int z5x(int r, int n) { return r * 16 + (n ^ (r & 15)); }
__device__ __forceinline__ int z5slot(int kz) { return kz; }

// SLAB = false (one slab, P = 1): the z offsets are compile-time immediates from one base pointer
// (otherwise 32 64-bit addresses stay live across the tile and the kernel spills).
// PF (one slab only): the two z lines of each warp arrive by 1-D bulk copies (8 KB each, the TMA
// engine) in the warp's own line buffers, completing on a per-warp mbarrier; the copies of the NEXT
// tile are issued as soon as the warp has read the last exchange of the current one, so they run
// under the inverse DFT32 and the 32 stores per thread (and under the other CTAs' phases).
template <int NC, int MODE, bool SLAB, bool PF = false>
__global__ void __launch_bounds__(NC == 6 ? 96 : 128, NC == 6 ? 4 : 2) k_zreg512w(ZPArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  static_assert(!(PF && SLAB), "prefetched lines must be contiguous (one slab)");
  extern __shared__ double2 sm[];
  constexpr int N = 512;
  const int TL = a.TL;
  const int nl = NC * TL;                       // blockDim.x == 16 * nl
  double2* tw = sm + (size_t)nl * kZ5Line;      // W512^{t k2} at (k2 - 1) * 16 + (t ^ (k2 & 15)), k2 in [1, 32)
  uint64_t* bars = reinterpret_cast<uint64_t*>(tw + 31 * 16);   // PF: one mbarrier per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  for (int i = threadIdx.x; i < 31 * 16; i += blockDim.x) {
    const int k2 = 1 + (i >> 4), tt = i & 15;
    tw[(k2 - 1) * 16 + (tt ^ (k2 & 15))] = __ldg(&a.twz[tt * k2]);
  }
  if (PF && lane == 0) {
    mbar_init(&bars[warp], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  const int line = threadIdx.x >> 4, t = threadIdx.x & 15;
  const int c = line >> a.lgTL, ll = line & (TL - 1);
  double2* ls = sm + (size_t)line * kZ5Line;
  const int nyt = a.Nyl / TL;
  const int ntiles = a.nkx * nyt;
  const int BS = NC * a.Hx * a.SL.nys * a.SL.nzs, zm = a.SL.nzs - 1, lgz = a.SL.lg_nzs;
  // PF: lane 0 of a warp copies the warp's lines 2 warp, 2 warp + 1 of tile tl into their buffers
  auto prefetch = [&](int tl) {
    const int kxp = a.kx0 + tl / nyt, kyp = (tl % nyt) * TL;
    mbar_arrive_expect_tx(&bars[warp], 2 * N * (unsigned)sizeof(double2));
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int lq = 2 * warp + q;
      bulk_g2s(sm + (size_t)lq * kZ5Line, a.B + r_index(a.SL, NC, a.Hx, lq >> a.lgTL, kxp, kyp + (lq & (TL - 1)), 0),
               N * (unsigned)sizeof(double2), &bars[warp]);
    }
  };
  unsigned phase = 0;
  if (PF && lane == 0 && (int)blockIdx.x < ntiles) prefetch(blockIdx.x);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int kx = a.kx0 + tile / nyt, ky0 = (tile % nyt) * TL;
    const int kyl = ky0 + ll;
    double2* Bl = a.B + r_index(a.SL, NC, a.Hx, c, kx, kyl, 0) + (SLAB ? 0 : t);
    auto zoff = [&](int z) -> size_t { return SLAB ? (size_t)((z >> lgz) * BS + (z & zm)) : (size_t)(z - t); };
    double2 v[32];
    if (PF) {
      mbar_wait(&bars[warp], phase);
      phase ^= 1u;
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = ls[t + 16 * m];
    } else {
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = __ldcg(Bl + zoff(t + 16 * m));
    }
    // ---- forward: DFT32 over m, twiddle, transpose, DFT16 over t ----
    // (each group of 8 outputs of the DFT32 is twiddled and stored at once: register footprint)
    dft32_stage1<false>(v);
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      dft8<false>(v + 8 * k1);                               // v[8 k1 + j] = Y[t][k2 = k1 + 4 j]
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k2 = k1 + 4 * j;
        double2 y = v[8 * k1 + j];
        if (k2 > 0) y = cmul(y, ld_tw(tw + (k2 - 1) * 16 + (t ^ (k2 & 15))));
        ls[z5x(k2, t)] = y;
      }
    }
    __syncwarp();
    const int ky = kyl + a.ky_off;
#pragma unroll
    for (int h = 0; h < 2; ++h) {                            // rows k2 = t, t + 16
      double2 u[16];
#pragma unroll
      for (int n = 0; n < 16; ++n) u[n] = ls[z5x(t + 16 * h, n)];
      dft16<false>(u);                                       // u[k1] = X[t + 16 h + 32 k1]
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) v[16 * h + k1] = u[k1];
    }
    // ---- spectral multiply ----
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) {
      ls[z5slot(t + 32 * k1)] = v[k1];
      ls[z5slot(t + 16 + 32 * k1)] = v[16 + k1];
    }
    if (MODE == Z_PRECOND) {
      // own slots only (no cross-thread traffic); |k|^2 from the per-axis factors as in k_zreg256
      double fx[2], fy[2];
      zaxis(a, 0, kx, a.Nx, nullptr, fx);
      zaxis(a, 1, ky, a.Ny, nullptr, fy);
#pragma unroll 1
      for (int j = 0; j < 32; ++j) {
        const int kz = t + 16 * (j & 1) + 32 * (j >> 1);
        double fz[2];
        if (a.scheme == 1) {
          const double cs = __ldg(&a.twz[kz]).x;
          fz[0] = (2.0 - 2.0 * cs) * a.qh2[2];
          fz[1] = 2.0 + 2.0 * cs;
        } else {
          zaxis(a, 2, kz, N, nullptr, fz);
        }
        const double k2 = a.scheme == 1 ? (fx[0] * fy[1] * fz[1] + fx[1] * fy[0] * fz[1] + fx[1] * fy[1] * fz[0])
                                        : fx[0] + fy[0] + fz[0];
        ls[z5slot(kz)] = cscale(ls[z5slot(kz)], a.scale / (1.0 + a.mean_ell2 * k2));
      }
    } else {
      __syncthreads();
      // Willot symbol with the (kx, ky) factors hoisted (TL = 1: one ky per tile)
      double2 P0 = make_double2(0.0, 0.0), P1 = P0, P2 = P0;
      const bool hoist = a.scheme == 1 && TL == 1;
      if (hoist) {
        const double2 wx = __ldg(&a.twx[kx]), wy = __ldg(&a.twy[ky0 + a.ky_off]);
        const double2 ex = make_double2(wx.x, -wx.y), ey = make_double2(wy.x, -wy.y);
        const double2 dx = make_double2(ex.x - 1.0, ex.y), dy = make_double2(ey.x - 1.0, ey.y);
        const double2 cx = make_double2(ex.x + 1.0, ex.y), cy = make_double2(ey.x + 1.0, ey.y);
        P0 = cscale(cmul(dx, cy), a.qh[0]);
        P1 = cscale(cmul(cx, dy), a.qh[1]);
        P2 = cscale(cmul(cx, cy), a.qh[2]);
      }
      for (int idx = threadIdx.x; idx < TL * N; idx += blockDim.x) {
        const int kz = idx & (N - 1), l2 = idx >> 9;
        const int kyg = ky0 + l2 + a.ky_off;
        double2 k[3];
        if (hoist) {
          const double2 wz = __ldg(&a.twz[kz]);
          const double2 cz = make_double2(wz.x + 1.0, -wz.y), dz = make_double2(wz.x - 1.0, -wz.y);
          k[0] = cmul(P0, cz);
          k[1] = cmul(P1, cz);
          k[2] = cmul(P2, dz);
        } else {
          zsymbol(a, N, kx, kyg, kz, k, a.twz);
        }
        double2* pv[6];
#pragma unroll
        for (int cc = 0; cc < 6; ++cc) pv[cc] = &sm[(size_t)(cc * TL + l2) * kZ5Line + z5slot(kz)];
        project6(a, pv, k, kx == 0 && kyg == 0 && kz == 0);
      }
      __syncthreads();
    }
    // ---- inverse: DFT16 over k1, conjugate twiddle, transpose, DFT32 over k2 ----
    // rows k2 = t + 16 h: read the 16 frequencies k1 from the staging slots, inverse DFT16, twiddle
    // and put them back in the exchange layout (row k2, column n) -- the staging slots of the line
    // are all read before any exchange slot is written (the two layouts overlap)
    double2 u[2][16];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) u[h][k1] = ls[z5slot(t + 16 * h + 32 * k1)];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      dft16<true>(u[h]);                                     // u[h][n] = Z[k2 = t + 16 h][n]
      const int k2 = t + 16 * h;
#pragma unroll
      for (int n = 0; n < 16; ++n) {
        double2 y = u[h][n];
        if (n > 0) {
          double2 w = ld_tw(tw + (k2 > 0 ? k2 - 1 : 0) * 16 + (n ^ (k2 & 15)));
          if (k2 == 0) w = make_double2(1.0, 0.0);
          w.y = -w.y;
          y = cmul(y, w);
        }
        ls[z5x(k2, n)] = y;
      }
    }
    __syncwarp();
#pragma unroll
    for (int k2 = 0; k2 < 32; ++k2) v[k2] = ls[z5x(k2, t)];
    if (PF) {
      // the warp's line buffers are free from here on: refill them with the next tile's lines
      __syncwarp();
      if (lane == 0 && tile + (int)gridDim.x < ntiles) {
        fence_proxy_async();
        prefetch(tile + gridDim.x);
      }
    }
    dft32_stage1<true>(v);
    // slab layout: the store offsets are recomputed from an opaque copy of the slab stride, so that
    // the 32 load offsets are not kept live (as 64-bit registers) across the whole tile -- they spilled
    int BSs = BS;
    if (SLAB) asm volatile("" : "+r"(BSs));
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      dft8<true>(v + 8 * k1);                                // v[8 k1 + j] = z[t + 16 (k1 + 4 j)]
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int z = t + 16 * (k1 + 4 * j);
        Bl[SLAB ? (size_t)((z >> lgz) * BSs + (z & zm)) : zoff(z)] = v[8 * k1 + j];
      }
    }
  }
}

// Y pass, Ny = 512: tile (c, kx pair, TZ planes), 2 TZ lines of 64 threads.  Warp w carries 16
// threads of each kx of the pair for plane zz = w / 4 (t = 16 (w % 4) + lane % 16), so that the
// A-side loads / stores are 512 B per warp instruction.  Line l = kl TZ + zz at pitch k512Line + 1.
constexpr int kY512Line = k512Line + 2;   // max pitch (see ypitch)

// Y pass forward, Ny = 512, wide plan (the 32 x 16 decomposition of k_zreg512w): tile (c, kx pair,
// TZ = 4 planes), 8 lines of 16 threads (warp w = plane, half-warp = kx of the pair, so that an A-row
// load of one m is 512 contiguous bytes per warp instruction).  One exchange per transform (swizzled
// rows), the spectrum staged at slot ky of the line (pitch 513: the z-fastest B-side stores read
// TZ lines at one ky conflict free), the next tile's A rows loaded into the registers while the
// B-side stores of this tile run.  Shared accesses per element ~5 (8x8x8 plan: ~8).
constexpr int kY5Pitch = 513;
__global__ void __launch_bounds__(128, 3) k_yreg512w(YArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 512, TZ = 4;
  double2* tw = sm + (size_t)2 * TZ * kY5Pitch;   // W512^{t k2} at (k2 - 1) * 16 + (t ^ (k2 & 15))
  pdl_trigger();
  for (int i = threadIdx.x; i < 31 * 16; i += blockDim.x) {
    const int k2 = 1 + (i >> 4), tt = i & 15;
    tw[(k2 - 1) * 16 + (tt ^ (k2 & 15))] = __ldg(&a.tw[tt * k2]);
  }
  __syncthreads();
  pdl_wait();
  const int zz = threadIdx.x >> 5, lane = threadIdx.x & 31, kl = lane >> 4, t = lane & 15;
  double2* ls = sm + (size_t)(kl * TZ + zz) * kY5Pitch;
  const int nzt = a.Nz / TZ, nkb = a.nkbc, lg_nzt = 31 - __clz(nzt);   // Nz is a power of two
  const int ntiles = a.ncomp * nkb * nzt;
  auto arow_of = [&](int tl) {
    int zt, kb, c;
    y512_tile(a, nzt, lg_nzt, tl, &zt, &kb, &c);
    return a.A + aidx(a.HxA, N, a.Nz, c, zt * TZ + zz, 0, kb * kKB) + kl + kKB * t;
  };
  double2 v[32];
  if ((int)blockIdx.x < ntiles) {
    const double2* A0 = arow_of(blockIdx.x);
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = __ldcs(A0 + kKB * 16 * m);
  }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int zt, kb, c;
    y512_tile(a, nzt, lg_nzt, tile, &zt, &kb, &c);
    const int z0 = zt * TZ, kx0 = kb * kKB;
    // ---- DFT32 over m, twiddle, transpose (row k2, column t), DFT16 over t ----
    dft32_stage1<false>(v);
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      dft8<false>(v + 8 * k1);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k2 = k1 + 4 * j;
        double2 y = v[8 * k1 + j];
        if (k2 > 0) y = cmul(y, ld_tw(tw + (k2 - 1) * 16 + (t ^ (k2 & 15))));
        ls[z5x(k2, t)] = y;
      }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 u[16];
#pragma unroll
      for (int n = 0; n < 16; ++n) u[n] = ls[z5x(t + 16 * h, n)];
      dft16<false>(u);                                     // u[k1] = X[ky = t + 16 h + 32 k1]
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) v[16 * h + k1] = u[k1];
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) ls[t + 16 * h + 32 * k1] = v[16 * h + k1];
    __syncthreads();
    const int tn = tile + gridDim.x;                       // next tile's A rows in flight during the stores
    if (tn < ntiles) {
      const double2* An = arow_of(tn);
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = __ldcs(An + kKB * 16 * m);
    }
    // B-side stores: element idx = tid + 128 it is (z2, ky, k2l) = (tid % 4, tid / 4 + 32 (it % 16), it / 16);
    // the slab terms that do not depend on ky are formed once per tile (no per-element s_index)
    {
      const int z = z0 + (threadIdx.x & 3), kyb = threadIdx.x >> 2;
      const int zl = z & (a.L.nzs - 1), zb = z >> a.L.lg_nzs;
      const size_t row0 = ((size_t)(zb * a.L.P) * a.ncomp + c) * a.Hx + kx0, ybstep = (size_t)a.ncomp * a.Hx;
      const double2* sp = sm + (size_t)(threadIdx.x & 3) * kY5Pitch + kyb;
#pragma unroll
      for (int k2l = 0; k2l < 2; ++k2l) {
        if (kx0 + k2l < a.Hx) {
#pragma unroll 4
          for (int j = 0; j < 16; ++j) {
            const int ky = kyb + 32 * j;
            const size_t rr = (row0 + k2l + (size_t)(ky >> a.L.lg_nys) * ybstep) * a.L.nys + (ky & (a.L.nys - 1));
            *yb_ptr(a, ky >> a.L.lg_nys, (rr << a.L.lg_nzs) + zl) = sp[(size_t)k2l * TZ * kY5Pitch + 32 * j];
          }
        }
      }
    }
    __syncthreads();
  }
}


template <bool INV>
__global__ void __launch_bounds__(512, 2) k_yreg512(YArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 512;
  const int TZ = a.TZ;                             // blockDim.x == 128 * TZ
  const int LPY = ypitch(k512Line, TZ);
  double2* tw1 = sm + (size_t)2 * TZ * LPY;
  double2* tw2 = tw1 + 448;
  pdl_trigger();
  fft512_tables(tw1, tw2, a.tw);
  pdl_wait();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kl = lane >> 4, t = 16 * (w & 3) + (lane & 15), zz = w >> 2;
  const int l = kl * TZ + zz;
  double2* ls = sm + (size_t)l * LPY;
  const int nzt = a.Nz / TZ, nkb = a.nkbc;
  const int ntiles = a.ncomp * nkb * nzt;
  __syncthreads();
  double2 v[8];
  auto arow_of = [&](int tl) {
    const int zt = tl % nzt, r = tl / nzt, kb = a.kb0 + r % nkb, c = r / nkb;
    return a.A + aidx(a.HxA, N, a.Nz, c, zt * TZ + zz, 0, kb * kKB) + kl;
  };
  if (!INV && (int)blockIdx.x < ntiles) {
    const double2* A0 = arow_of(blockIdx.x);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(A0 + kKB * (t + 64 * j));
  }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int zt = tile % nzt, r = tile / nzt, kb = a.kb0 + r % nkb, c = r / nkb;
    const int z0 = zt * TZ, kx0 = kb * kKB, kx = kx0 + kl;
    double2* Arow = a.A + aidx(a.HxA, N, a.Nz, c, z0 + zz, 0, kx0) + kl;   // element y at Arow[kKB * y]
    if (!INV) {
      fft512_reg<false>(v, t, ls, tw1, tw2, 1 + zz, 128);   // v[kc] = X[ky = t + 64 kc]
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) ls[kc * 65 + t] = v[kc];
      __syncthreads();
      const int tn = tile + gridDim.x;           // next tile's A rows in flight during the stores
      if (tn < ntiles) {
        const double2* An = arow_of(tn);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldcs(An + kKB * (t + 64 * j));
      }
      for (int idx = threadIdx.x; idx < 2 * N * TZ; idx += blockDim.x) {
        const int z2 = idx % TZ, ky = (idx / TZ) & (N - 1), k2l = idx / (TZ * N);
        const int kxo = kx0 + k2l;
        if (kxo < a.Hx)
          *yb_ptr(a, ky >> a.L.lg_nys, s_index(a.L, a.ncomp, a.Hx, c, kxo, ky, z0 + z2)) =
              sm[(size_t)(k2l * TZ + z2) * LPY + (ky >> 6) * 65 + (ky & 63)];
      }
      __syncthreads();
    } else {
      // the staging loop below writes EVERY line buffer, and the previous tile's inverse FFT
      // synchronises only the warps of its own plane (named barrier): wait for all planes first
      __syncthreads();
      for (int idx = threadIdx.x; idx < 2 * N * TZ; idx += blockDim.x) {
        const int z2 = idx % TZ, ky = (idx / TZ) & (N - 1), k2l = idx / (TZ * N);
        const int kxo = kx0 + k2l;
        if (kxo < a.Hx)
          cp_async16(&sm[(size_t)(k2l * TZ + z2) * LPY + (ky >> 6) * 65 + (ky & 63)],
                     yb_ptr(a, ky >> a.L.lg_nys, s_index(a.L, a.ncomp, a.Hx, c, kxo, ky, z0 + z2)));
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) v[kc] = ls[kc * 65 + t];
      __syncthreads();
      fft512_reg<true>(v, t, ls, tw1, tw2, 1 + zz, 128);    // v[m] = y-line value at y = t + 64 m
      if (kx < a.Hx) {
#pragma unroll
        for (int m = 0; m < 8; ++m) Arow[kKB * (t + 64 * m)] = v[m];
      }
    }
  }
}

// Y pass inverse, Ny = 512, double-buffered: the NEXT tile's B-side input (TZ runs of 16 B per ky,
// z fastest) is staged by cp.async into the second set of line buffers while the current tile is
// transformed (k_yreg512<true> waits for its own staging before every tile: long-scoreboard bound).
// TZ = 2 (256 threads, two buffers of 4 lines, three CTAs per SM); the current buffer doubles as the
// exchange buffer once its column has been read into registers.
__global__ void __launch_bounds__(256, 3) k_yreg512i(YArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 512;
  const int TZ = a.TZ;                             // blockDim.x == 128 * TZ
  const int LPY = ypitch(k512Line, TZ);
  const int NLB = 2 * TZ;                          // lines per buffer
  double2* tw1 = sm + (size_t)2 * NLB * LPY;
  double2* tw2 = tw1 + 448;
  pdl_trigger();
  fft512_tables(tw1, tw2, a.tw);
  pdl_wait();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kl = lane >> 4, t = 16 * (w & 3) + (lane & 15), zz = w >> 2;
  const int l = kl * TZ + zz;
  const int nzt = a.Nz / TZ, nkb = a.nkbc;
  const int ntiles = a.ncomp * nkb * nzt;
  // B-side staging: element idx = tid + 128 TZ it (it < 8) is (z2, ky, k2l) = (tid % TZ, tid / TZ + 128 (it % 4),
  // it / 4): z2 and ky mod 128 are fixed per thread, so the thread's four ky addresses are formed once
  // per tile and the second kx of the pair is one slab row further (the per-element index arithmetic
  // with its runtime divisions made up half of this kernel's instructions)
  const int lg_nzt = 31 - __clz(nzt);              // Nz and TZ are powers of two
  const int z2t = threadIdx.x & (TZ - 1), ky0 = threadIdx.x >> a.lgTZ;
  const int soff = z2t * LPY + (ky0 >> 6) * 65 + (ky0 & 63);
  const size_t kxstep = (size_t)a.L.nys << a.L.lg_nzs;
  auto issue = [&](int tile, double2* buf) {
    int zt, kb, c;
    y512_tile(a, nzt, lg_nzt, tile, &zt, &kb, &c);
    const int z = zt * TZ + z2t, kx0 = kb * kKB;
    const bool two = kx0 + 1 < a.Hx;
    double2* sb = buf + soff;
    if (kx0 >= a.Hx) return;                       // padding block of layout A (HxA = Hx rounded up to 4)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2* g = yb_ptr(a, (ky0 + 128 * j) >> a.L.lg_nys, s_index(a.L, a.ncomp, a.Hx, c, kx0, ky0 + 128 * j, z));
      cp_async16_l2(sb + 130 * j, g, a.l2pf);
      if (two) cp_async16_l2(sb + 130 * j + TZ * LPY, g + kxstep, a.l2pf);
    }
  };
  int i = 0;
  if ((int)blockIdx.x < ntiles) issue(blockIdx.x, sm);
  cp_async_commit();
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
    double2* cur = sm + (size_t)(i & 1) * NLB * LPY;
    double2* nxt = sm + (size_t)((i + 1) & 1) * NLB * LPY;
    // every thread is done with `nxt` (the previous tile's exchanges) before it is refilled
    __syncthreads();
    const int tn = tile + gridDim.x;
    if (tn < ntiles) issue(tn, nxt);
    cp_async_commit();
    cp_async_wait<1>();                            // this tile's staging has landed
    __syncthreads();
    int zt, kb, c;
    y512_tile(a, nzt, lg_nzt, tile, &zt, &kb, &c);
    const int z0 = zt * TZ, kx = kb * kKB + kl;
    double2* ls = cur + (size_t)l * LPY;
    double2 v[8];
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) v[kc] = ls[kc * 65 + t];
    __syncthreads();
    // CTA-wide barrier 0 inside the FFT (both planes run in step): a constant barrier id keeps the
    // kernel at one hardware barrier (runtime ids reserve all 16 and cap the CTAs per SM)
    fft512_reg<true>(v, t, ls, tw1, tw2, 0, 128 * TZ);     // v[m] = y-line value at y = t + 64 m
    if (kx < a.Hx) {
      double2* Arow = a.A + aidx(a.HxA, N, a.Nz, c, z0 + zz, 0, kb * kKB) + kl;
#pragma unroll
      for (int m = 0; m < 8; ++m) Arow[kKB * (t + 64 * m)] = v[m];
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// One-component preconditioner, N2 = N3 = 256, one GPU: the y-forward, z (with the multiply) and
// y-inverse passes fused into ONE kernel per kx plane with a thread-block cluster of 8 CTAs and
// distributed shared memory.  Opt-in (FGD_YZY=1): on the 256^3 sweep it is slower than the three
// streaming passes (see launch_precond_yz).  CTA r of the cluster holds the (z in [32 r, 32 r + 32), all y)
// block of the kx plane (128 KB):
//   1. y-forward FFT of its 32 z rows (A -> registers -> 16x16 register FFT -> local block, ky)
//   2. cluster barrier; z-lines ky in [32 r, 32 r + 32): the 16 threads of a z-line read their 16
//      points z = t + 16 j straight from the 8 blocks of the cluster (DSMEM), z FFT, multiply by
//      scale / (1 + <l^2>|k|^2), inverse z FFT, and write the points back where they came from
//   3. cluster barrier; inverse y FFT of the 32 local rows -> A
// HBM: the spectrum of the plane is read and written once (16 B per complex value) instead of
// three read+write passes through the transposed buffer B.
// Block slot of (row l, ky): l * 256 + (ky ^ (l & 15)) -- the z-line reads (16 rows, one ky) and
// the row accesses are both conflict free.
namespace cg = cooperative_groups;
constexpr int kYZCl = 8;
constexpr size_t kYZSmem = (size_t)(32 * 256 + 16 * kZLine + 240) * sizeof(double2) + 2 * 256 * sizeof(double);

struct YZArgs {
  double2* A;
  int Nz, Hx, HxA;
  ZPArgs z;   // symbol / multiply parameters (twx, twy, twz, h, scheme, scale, mean_ell2)
};

__device__ __forceinline__ double rcp_pos(double x) {
  // 1/x for x >= 1 without the division slow path: float seed + two Newton steps (rel. err ~1e-28)
  double r = (double)__frcp_rn((float)x);
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

__global__ void __cluster_dims__(kYZCl, 1, 1) __launch_bounds__(512, 1) k_yzy256(YZArgs a) {
  if (guard_done(a.z.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int N = 256;
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int kx = blockIdx.x / kYZCl;
  double2* D = sm;                                  // [32 rows][256]
  double2* scr = D + 32 * 256;                      // [16 z-lines][kZLine] exchange scratch
  double2* tw = scr + 16 * kZLine;                  // W256^{t k2} at (k2 - 1) * 16 + t
  double* fz0 = reinterpret_cast<double*>(tw + 240);
  double* fz1 = fz0 + 256;
  for (int i = threadIdx.x; i < 240; i += blockDim.x) tw[i] = __ldg(&a.z.twz[(i & 15) * (1 + (i >> 4))]);
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    double f[2];
    zaxis(a.z, 2, m, N, nullptr, f);
    fz0[m] = f[0];
    fz1[m] = f[1];
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane & 15;
  const int l = 2 * w + (lane >> 4);                // phase 1 / 3: local row (z = 32 r + l)
  const int z = 32 * r + l;
  const int sw = l & 15;
  double2* row = D + l * 256;
  double2* Arow = a.A + aidx(a.HxA, N, a.Nz, 0, z, 0, kx);   // element y at Arow[kKB * y]
  __syncthreads();
  double2 v[16];
  // ---- 1. y forward ----
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = Arow[kKB * (t + 16 * j)];
  dft16<false>(v);
#pragma unroll
  for (int k2 = 1; k2 < 16; ++k2) v[k2] = cmul(v[k2], ld_tw(tw + (k2 - 1) * 16 + t));
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) row[k2 * 16 + (t ^ k2)] = v[k2];
  __syncwarp();
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) v[n1] = row[t * 16 + (n1 ^ t)];
  dft16<false>(v);                                  // v[k1] = X[ky = t + 16 k1]
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) row[(t + 16 * k1) ^ sw] = v[k1];
  cluster.sync();
  // ---- 2. z lines ky in [32 r, 32 r + 32), two rounds of 16 ----
  if (threadIdx.x < 256) {
    const int lz = threadIdx.x >> 4;                // z-line within the round
    double2* sl = scr + lz * kZLine;
    double fx[2], fy[2];
    zaxis(a.z, 0, kx, a.z.Nx, nullptr, fx);
    for (int round = 0; round < 2; ++round) {
      const int ky = 32 * r + 16 * round + lz;
      zaxis(a.z, 1, ky, a.z.Ny, nullptr, fy);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int zl = t + 16 * (j & 1);
        v[j] = *cluster.map_shared_rank(D + zl * 256 + (ky ^ (zl & 15)), j >> 1);
      }
      dft16<false>(v);
#pragma unroll
      for (int k2 = 1; k2 < 16; ++k2) v[k2] = cmul(v[k2], ld_tw(tw + (k2 - 1) * 16 + t));
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) sl[k2 * kZRowPad + t] = v[k2];
      __syncwarp();
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) v[n1] = sl[t * kZRowPad + n1];
      dft16<false>(v);                              // v[k1] = X[kz = t + 16 k1]
      const double A2 = a.z.scheme == 1 ? fx[0] * fy[1] + fx[1] * fy[0] : 0.0;
      const double B2 = a.z.scheme == 1 ? fx[1] * fy[1] : 0.0;
      const double C2 = a.z.scheme == 1 ? 0.0 : fx[0] + fy[0];
#pragma unroll
      for (int k1 = 0; k1 < 16; ++k1) {
        const int kz = t + 16 * k1;
        const double k2v = a.z.scheme == 1 ? fma(A2, fz1[kz], B2 * fz0[kz]) : C2 + fz0[kz];
        v[k1] = cscale(v[k1], a.z.scale * rcp_pos(fma(a.z.mean_ell2, k2v, 1.0)));
      }
      dft16<true>(v);                               // v[n1] = U[k2 = t][n1]
#pragma unroll
      for (int n1 = 1; n1 < 16; ++n1) {
        double2 wv = ld_tw(tw + (n1 - 1) * 16 + t);
        wv.y = -wv.y;
        v[n1] = cmul(v[n1], wv);
      }
      __syncwarp();
#pragma unroll
      for (int n1 = 0; n1 < 16; ++n1) sl[n1 * kZRowPad + t] = v[n1];
      __syncwarp();
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) v[k2] = sl[t * kZRowPad + k2];
      dft16<true>(v);                               // v[n2] = value at z = t + 16 n2
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int zl = t + 16 * (j & 1);
        *cluster.map_shared_rank(D + zl * 256 + (ky ^ (zl & 15)), j >> 1) = v[j];
      }
      __syncwarp();
    }
  }
  cluster.sync();
  // ---- 3. y inverse ----
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) v[k1] = row[(t + 16 * k1) ^ sw];
  dft16<true>(v);
#pragma unroll
  for (int n1 = 1; n1 < 16; ++n1) {
    double2 wv = ld_tw(tw + (n1 - 1) * 16 + t);
    wv.y = -wv.y;
    v[n1] = cmul(v[n1], wv);
  }
  __syncwarp();
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) row[n1 * 16 + (t ^ n1)] = v[n1];
  __syncwarp();
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) v[k2] = row[t * 16 + (k2 ^ t)];
  dft16<true>(v);                                   // v[n2] = y-line value at y = t + 16 n2
  if (kx < a.Hx) {
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) Arow[kKB * (t + 16 * n2)] = v[n2];
  }
}

// ---------------------------------------------------------------------------------------------
// X passes, one component per tile
// ---------------------------------------------------------------------------------------------
struct XPArgs {
  const DevScalars* guard;
  int Ny, Nz, TY, ncomp, lgTY, HxA;
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

// Modes whose epilogue reads one real operand row per output row (MECH_CG: r, HELM_Z: r of the
// PCG): that operand is staged by cp.async together with the spectrum of the tile.
// (N = 256 loads its epilogue operand into registers ahead of the FFT instead; see k_xipipe)
template <int N, int MODE>
__host__ __device__ constexpr bool xi_prefetch() {
  return (MODE == XI_MECH_CG || MODE == XI_HELM_Z) && N != 256 && N != 512;
}

template <int N, int MODE>
__device__ __forceinline__ void xi_issue(const XPArgs& a, int t, double2* buf, double* ebuf) {
  constexpr int M = N / 2, Hx = M + 1;
  constexpr int LP = xline(M);
  const int TY = a.TY, nyt = a.Ny / TY;
  const int yt = t % nyt, r = t / nyt, z = r % a.Nz, c = r / a.Nz;
  const int y0 = yt * TY;
  constexpr int NB = (Hx + kKB - 1) / kKB;
  const int kbs = blockDim.x >> (1 + a.lgTY);   // kx blocks per sweep of the CTA (kKB = 2)
  if (kbs > 0) {
    // order (kx % kKB, yy, kx / kKB): runs of TY * kKB contiguous elements of layout A.  (kl, yy) and the
    // first kx block are fixed per thread: one base address per tile, then constant steps
    static_assert(kKB == 2, "thread mapping below");
    const int kl = threadIdx.x & 1, yy = (threadIdx.x >> 1) & (TY - 1);
    int kb = threadIdx.x >> (1 + a.lgTY);
    const double2* g = a.spec + (((size_t)(c * a.Nz + z) * (a.HxA / kKB) + kb) * a.Ny + y0 + yy) * kKB + kl;
    const size_t gstep = (size_t)kbs * a.Ny * kKB;
    double2* sb = buf + yy * LP;
    for (; kb < NB; kb += kbs, g += gstep) {
      const int kx = kb * kKB + kl;
      if (kx < Hx) cp_async16(sb + SWZ(yy, kx), g);
    }
  } else {
    for (int idx = threadIdx.x; idx < NB * TY * kKB; idx += blockDim.x) {
      const int kl = idx % kKB, yy = (idx / kKB) & (TY - 1), kx = (idx / kKB >> a.lgTY) * kKB + kl;
      if (kx < Hx) cp_async16(&buf[yy * LP + SWZ(yy, kx)], &a.spec[aidx(a.HxA, a.Ny, a.Nz, c, z, y0 + yy, kx)]);
    }
  }
  if constexpr (xi_prefetch<N, MODE>()) {
    // rows y0 .. y0 + TY - 1 of plane z are contiguous: TY * N doubles
    const double* src = a.in0 + (size_t)c * a.nvox + ((size_t)z * a.Ny + y0) * N;
    for (int idx = threadIdx.x; idx < TY * N / 2; idx += blockDim.x) cp_async16(ebuf + 2 * idx, src + 2 * idx);
  }
}

template <int N, int MODE>
__global__ void __launch_bounds__((N == 256 || N == 512) ? 128 : 256, (N == 256 || N == 512) ? 3 : 2) k_xipipe(XPArgs a) {
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  pdl_trigger();
  constexpr int M = N / 2;
  constexpr int LP = xline(M);
  const int TY = a.TY, nyt = a.Ny / TY;
  double2* twM = sm + 2 * TY * LP;
  double2* twN = twM + M;
  double* ebuf = reinterpret_cast<double*>(twN + N);   // [2][TY * N] epilogue operand (xi_prefetch)
  double2* tw128 = reinterpret_cast<double2*>(ebuf + (xi_prefetch<N, MODE>() ? 2 * TY * N : 0));   // M = 128 only
  build_pass_tables<M>(twM, a.twM);
  load_table(twN, a.twN, N);
  if constexpr (M == 128)
    for (int k = threadIdx.x; k < 120; k += blockDim.x) tw128[k] = __ldg(&a.twM[(k & 7) * (1 + (k >> 3))]);
  if constexpr (M == 256) fft_reg_tables<M>(tw128, a.twM);   // W256^{t k2} at (k2 - 1) * 16 + t
  const int ntiles = a.ncomp * a.Nz * nyt;
  const size_t n = a.nvox;
  double red[1] = {0.0};
  double alpha = 0.0;
  pdl_wait();
  if (MODE == XI_MECH_CG) alpha = a.sc->alpha;
  int t = blockIdx.x;
  if (t < ntiles) xi_issue<N, MODE>(a, t, sm, ebuf);
  cp_async_commit();
  for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < ntiles) xi_issue<N, MODE>(a, tn, sm + ((i + 1) & 1) * TY * LP, ebuf + ((i + 1) & 1) * TY * N);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    double2* buf = sm + (i & 1) * TY * LP;
    for (int idx = threadIdx.x; idx < TY * (M / 2 + 1); idx += blockDim.x) {
      const int k = idx % (M / 2 + 1), l = idx / (M / 2 + 1);
      c2r_pre_p<N>(buf + (size_t)l * LP, l, k, twN);
    }
    __syncthreads();
    const int yt = t % nyt, r = t / nyt, z = r % a.Nz, c = r / a.Nz;
    const int y0 = yt * TY;
    const double* eb = ebuf + (i & 1) * TY * N;
    if constexpr (M == 128) {
      // register FFT 128 = 16 x 8 (8 threads per line, 16 points each, one exchange), epilogue
      // straight from the registers: thread (yy, tt) ends with z[n], n = tt + 16 k1 and tt + 8 + 16 k1,
      // z[n] = x[2n] + i x[2n+1]
      if (threadIdx.x < TY * 8) {
        const int yy = threadIdx.x >> 3, tt = threadIdx.x & 7;
        double2* ln = buf + (size_t)yy * LP;
        const size_t grow = (size_t)c * n + ((size_t)z * a.Ny + y0 + yy) * N;
        // epilogue operand (r) of this thread's 16 output pairs, in flight during the FFT
        double2 ro[16];
        if (MODE == XI_MECH_CG || MODE == XI_HELM_Z) {
          const double* rs = a.in0 + grow;
#pragma unroll
          for (int h = 0; h < 16; ++h) {
            const int nn = (h < 8 ? tt : tt + 8) + 16 * (h & 7);
            ro[h] = __ldcs(reinterpret_cast<const double2*>(rs + 2 * nn));
          }
        }
        double2 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ln[SWZ(yy, tt + 8 * j)];
        dft16<true>(v);
#pragma unroll
        for (int k2 = 1; k2 < 16; ++k2) {
          double2 w = ld_tw(tw128 + (k2 - 1) * 8 + tt);
          w.y = -w.y;
          v[k2] = cmul(v[k2], w);
        }
        __syncwarp();
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) ln[k2 * 9 + tt] = v[k2];
        __syncwarp();
        double2 u0[8], u1[8];
#pragma unroll
        for (int n1 = 0; n1 < 8; ++n1) {
          u0[n1] = ln[tt * 9 + n1];
          u1[n1] = ln[(tt + 8) * 9 + n1];
        }
        dft8<true>(u0);
        dft8<true>(u1);
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          const int nn = (h < 8 ? tt : tt + 8) + 16 * (h & 7);
          const double2 q2 = h < 8 ? u0[h & 7] : u1[h & 7];
          const int x = 2 * nn;
          double2* o2;
          if (MODE == XI_MECH_CG) {
            const double2 rn = make_double2(fma(-alpha, q2.x, ro[h].x), fma(-alpha, q2.y, ro[h].y));
            o2 = reinterpret_cast<double2*>(a.io2 + grow + x);
            *o2 = rn;
            red[0] = fma(rn.x, rn.x, fma(rn.y, rn.y, red[0]));
          } else {
            o2 = reinterpret_cast<double2*>(a.out0 + grow + x);
            *o2 = q2;
            if (MODE == XI_STORE_RR) red[0] = fma(q2.x, q2.x, fma(q2.y, q2.y, red[0]));
            if (MODE == XI_HELM_Z) red[0] = fma(ro[h].x, q2.x, fma(ro[h].y, q2.y, red[0]));
          }
        }
      }
      __syncthreads();
      continue;
    }
    if constexpr (M == 256) {
      // register FFT 256 = 16 x 16 (16 threads per line, one exchange), epilogue from registers:
      // thread (yy, tt) ends with z[n], n = tt + 16 k1, z[n] = x[2n] + i x[2n+1]
      if (threadIdx.x < TY * 16) {
        const int yy = threadIdx.x >> 4, tt = threadIdx.x & 15;
        double2* ln = buf + (size_t)yy * LP;
        const size_t grow = (size_t)c * n + ((size_t)z * a.Ny + y0 + yy) * N;
        double2 ro[16];
        if (MODE == XI_MECH_CG || MODE == XI_HELM_Z) {
          const double* rs = a.in0 + grow;
#pragma unroll
          for (int h = 0; h < 16; ++h) ro[h] = __ldcs(reinterpret_cast<const double2*>(rs + 2 * (tt + 16 * h)));
        }
        double2 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ln[SWZ(yy, tt + 16 * j)];
        dft16<true>(v);
#pragma unroll
        for (int k2 = 1; k2 < 16; ++k2) {
          double2 w = ld_tw(tw128 + (k2 - 1) * 16 + tt);
          w.y = -w.y;
          v[k2] = cmul(v[k2], w);
        }
        __syncwarp();
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) ln[k2 * 17 + tt] = v[k2];
        __syncwarp();
#pragma unroll
        for (int n1 = 0; n1 < 16; ++n1) v[n1] = ln[tt * 17 + n1];
        dft16<true>(v);
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          const int x = 2 * (tt + 16 * h);
          const double2 q2 = v[h];
          if (MODE == XI_MECH_CG) {
            const double2 rn = make_double2(fma(-alpha, q2.x, ro[h].x), fma(-alpha, q2.y, ro[h].y));
            *reinterpret_cast<double2*>(a.io2 + grow + x) = rn;
            red[0] = fma(rn.x, rn.x, fma(rn.y, rn.y, red[0]));
          } else {
            *reinterpret_cast<double2*>(a.out0 + grow + x) = q2;
            if (MODE == XI_STORE_RR) red[0] = fma(q2.x, q2.x, fma(q2.y, q2.y, red[0]));
            if (MODE == XI_HELM_Z) red[0] = fma(ro[h].x, q2.x, fma(ro[h].y, q2.y, red[0]));
          }
        }
      }
      __syncthreads();
      continue;
    }
    fft_lines<M, true>(buf, TY, LP, twM);
    __syncthreads();
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
        const double rn = fma(-alpha, q, eb[idx]);
        a.io2[g] = rn;
        red[0] = fma(rn, rn, red[0]);
      } else if (MODE == XI_HELM_Z) {
        a.out0[g] = q;
        red[0] = fma(eb[idx], q, red[0]);
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
  if (guard_done(a.guard)) return;   // converged Krylov loop: skip
  extern __shared__ double2 sm[];
  constexpr int M = N / 2, Hx = M + 1;
  constexpr int LP = xline(M);
  const int TY = a.TY, nyt = a.Ny / TY;
  double2* twM = sm + 2 * TY * LP;
  double2* twN = twM + M;
  pdl_trigger();
  build_pass_tables<M>(twM, a.twM);
  load_table(twN, a.twN, N);
  const int ntiles = a.ncomp * a.Nz * nyt;
  int t = blockIdx.x;
  pdl_wait();
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
    constexpr int NB = (Hx + kKB - 1) / kKB;
    for (int idx = threadIdx.x; idx < NB * TY * kKB; idx += blockDim.x) {
      const int kl = idx % kKB, yy = (idx / kKB) & (TY - 1), kx = (idx / kKB >> a.lgTY) * kKB + kl;
      if (kx < Hx) a.spec[aidx(a.HxA, a.Ny, a.Nz, c, z, y0 + yy, kx)] = buf[yy * LP + SWZ(yy, kx)];
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
  *grid_out = grid_cap(std::max(1, std::min(ntiles, (num_sms() - c->sm_reserve) * occ)));
  return FGD_OK;
}

#define FGD_PLAUNCH(ctx, kern, thr, smem, ntiles, ...)                                                  \
  do {                                                                                                  \
    int grid_ = 1;                                                                                      \
    fgd_status st_ = launch_persistent(ctx, kern, thr, smem, ntiles, &grid_, #kern);                     \
    if (st_ != FGD_OK) return st_;                                                                      \
    (ctx)->launches++;                                                                                  \
    cudaError_t e_ = launch_pdl(kern, dim3(grid_), dim3(thr), smem, (ctx)->stream, __VA_ARGS__);          \
    if (e_ == cudaSuccess) e_ = cudaGetLastError();                                                     \
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

// Peer-store transposes: rank s's R base, offset by (r - s) blocks, so that the S index of an element
// of y-slab s (block s of the local S layout) lands in block r of rank s's R (same intra-block offset).
static void fill_peers(const fgd_ctx* c, int ncomp, YArgs* a) {
  a->npeer = 0;
  if (!c->peer_on || !c->peer_ready) return;
  const int P = c->nranks;
  const long long blk = (long long)ncomp * c->Hx * (c->n[1] / P) * (c->n[2] / P);
  a->npeer = P;
  for (int s = 0; s < P; ++s) a->peer[s] = c->peerC[s] + (long long)(c->rank - s) * blk;
}

// L2 prefetch hint of the y-inverse B-side reads (FGD_Y_L2PF = 0..3; local buffers only: a peer's
// memory is not cached in this GPU's L2 the same way)
static int y_l2pf(const fgd_ctx* c) {
  static const int v = [] {
    const char* e = std::getenv("FGD_Y_L2PF");
    return e ? std::atoi(e) : 0;
  }();
  return (c->peer_on || c->nranks > 1) ? 0 : v;
}

fgd_status pipe_y(fgd_ctx* c, int ncomp, bool inv, int kxa, int kxb) {
  const int Ny = c->n[1], Nz = c->nz_l;
  if (kxb < 0) kxb = c->HxA;   // kx chunk [kxa, kxb): multiples of 4 (kx blocks of kKB or TK <= 4)
  if (Ny == 512 && !std::getenv("FGD_NO_YREG")) {
    const int TZ = std::min(4, std::min(Nz, c->n[2] / c->P));
    const int thr = 128 * TZ;
    const size_t smem = ((size_t)2 * TZ * kY512Line + 448 + 56) * sizeof(double2);
    const int ntiles = ncomp * ((kxb - kxa) / kKB) * (Nz / TZ);
    YArgs a{c->guard ? c->sc : nullptr, c->specA, c->specB, Nz, c->Hx, c->HxA, TZ, kKB, ncomp, ilog2(TZ), ilog2(kKB), c->tabs.tw[ilog2(Ny)],
            slab_layout(c), kxa / kKB, (kxb - kxa) / kKB};
    fill_peers(c, ncomp, &a);
    a.l2pf = y_l2pf(c);
    {
      // tile order of the 512 kernels (y512_tile): FGD_Y512_ZF = log2 of the z groups that vary fastest
      const char* e = std::getenv("FGD_Y512_ZF");
      a.lgzf = e ? std::atoi(e) : -1;
    }
    KTimer kt(c, inv ? (ncomp == 6 ? KC_YINV6 : KC_YINV1) : (ncomp == 6 ? KC_YFWD6 : KC_YFWD1));
    static const int y512i = [] {
      const char* e = std::getenv("FGD_Y512I");
      return e ? std::atoi(e) : 1;   // 1: double-buffered inverse (k_yreg512i, TZ = 2)
    }();
    if (inv && y512i && std::min(Nz, c->n[2] / c->P) >= 2) {
      const int TZi = 2;
      YArgs ai = a;
      ai.TZ = TZi;
      ai.lgTZ = 1;
      const size_t smem_i = ((size_t)4 * TZi * ypitch(k512Line, TZi) + 448 + 56) * sizeof(double2);
      const int nt_i = ncomp * ((kxb - kxa) / kKB) * (Nz / TZi);
      FGD_PLAUNCH(c, k_yreg512i, 128 * TZi, smem_i, nt_i, ai);
      return FGD_OK;
    }
    static const int y512w = [] {
      const char* e = std::getenv("FGD_Y512W");
      return e ? std::atoi(e) : 1;   // 1: wide 32 x 16 forward (k_yreg512w, TZ = 4)
    }();
    if (!inv && y512w && std::min(Nz, c->n[2] / c->P) >= 4) {
      YArgs aw = a;
      aw.TZ = 4;
      aw.lgTZ = 2;
      const size_t smem_w = ((size_t)8 * kY5Pitch + 31 * 16) * sizeof(double2);
      const int nt_w = ncomp * ((kxb - kxa) / kKB) * (Nz / 4);
      FGD_PLAUNCH(c, k_yreg512w, 128, smem_w, nt_w, aw);
      return FGD_OK;
    }
    if (inv) FGD_PLAUNCH(c, k_yreg512<true>, thr, smem, ntiles, a);
    else FGD_PLAUNCH(c, k_yreg512<false>, thr, smem, ntiles, a);
    return FGD_OK;
  }
  if (Ny == 256 && !std::getenv("FGD_NO_YREG")) {
    // 4 planes per tile (64 B runs on the B side; 128-thread CTAs, up to 4 per SM).  Measured on
    // the 256^3 sweep, 6-component forward: 4 planes 3.88 ms, 8 planes 4.09 ms, 2 planes 4.41 ms.
    static const int tzf = [] {
      const char* e = std::getenv("FGD_YF_TZ");
      return e ? std::atoi(e) : 4;
    }();
    const int TZ = std::min(inv ? 4 : tzf, std::min(Nz, c->n[2] / c->P));
    const int thr = 32 * TZ;
    const size_t smem = ((inv ? 2 : 1) * (size_t)2 * TZ * kYLine + 240) * sizeof(double2);
    const int ntiles = ncomp * ((kxb - kxa) / kKB) * (Nz / TZ);
    YArgs a{c->guard ? c->sc : nullptr, c->specA, c->specB, Nz, c->Hx, c->HxA, TZ, kKB, ncomp, ilog2(TZ), ilog2(kKB), c->tabs.tw[ilog2(Ny)],
            slab_layout(c), kxa / kKB, (kxb - kxa) / kKB};
    fill_peers(c, ncomp, &a);
    a.l2pf = y_l2pf(c);
    KTimer kt(c, inv ? (ncomp == 6 ? KC_YINV6 : KC_YINV1) : (ncomp == 6 ? KC_YFWD6 : KC_YFWD1));
    if (inv) FGD_PLAUNCH(c, k_yreg256<true>, thr, smem, ntiles, a);
    else FGD_PLAUNCH(c, k_yreg256<false>, thr, smem, ntiles, a);
    return FGD_OK;
  }
  const int TPL = fft_TPL(Ny, true);
  static const int nl_env = [] {
    const char* e = std::getenv("FGD_YL");
    return e ? std::atoi(e) : 8;
  }();
  static const int tk_env = [] {
    const char* e = std::getenv("FGD_YTK");
    return e ? std::atoi(e) : kKB;
  }();
  // lines per tile = TZ * TK; at least 8 so that both sides of the transpose move >= 64 B runs
  const int NL = std::max(8, p2floor(std::max(1, std::min(nl_env, 256) * 16 / TPL)));
  int TK = p2floor(std::max(1, std::min(std::min(tk_env, NL), 4)));
  int TZ = std::min(NL / TK, std::min(Nz, c->n[2] / c->P));
  TK = std::min(NL / TZ, 4);
  const int thr = std::min(256, r32(TZ * TK * TPL));
  const size_t smem = (2 * (size_t)TZ * TK * cline(Ny) + Ny) * sizeof(double2);
  const int ntiles = ncomp * ((kxb - kxa) / TK) * (Nz / TZ);
  YArgs a{c->guard ? c->sc : nullptr, c->specA, c->specB, Nz, c->Hx, c->HxA, TZ, TK, ncomp, ilog2(TZ), ilog2(TK), c->tabs.tw[ilog2(Ny)],
          slab_layout(c), kxa / TK, (kxb - kxa) / TK};
  fill_peers(c, ncomp, &a);
  KTimer kt(c, inv ? (ncomp == 6 ? KC_YINV6 : KC_YINV1) : (ncomp == 6 ? KC_YFWD6 : KC_YFWD1));
#define YPP(NN)                                                                  \
  if (inv) FGD_PLAUNCH(c, (k_ypipe<NN, true>), thr, smem, ntiles, a);            \
  else FGD_PLAUNCH(c, (k_ypipe<NN, false>), thr, smem, ntiles, a);
  FGD_PDISPATCH(Ny, YPP)
#undef YPP
  return FGD_OK;
}

fgd_status pipe_z(fgd_ctx* c, int ncomp, int mode, double scale, const double* dc_shift, double mean_ell2, int kxa,
                  int kxb) {
  kxb = kxb < 0 ? c->Hx : std::min(kxb, c->Hx);
  const int nkx = kxb - kxa;
  if (nkx <= 0) return FGD_OK;
  const int Ny = c->n[1], Nz = c->n[2];
  const int Nyl = c->nranks > 1 ? Ny / c->P : Ny;
  const int TPL = fft_TPL(Nz);
  int TL = p2floor(std::max(1, 192 / (ncomp * TPL)));
  if (Nz == 1) TL = 32;
  TL = std::min(TL, Nyl);
  const int thr = std::min(192, std::max(r32(ncomp * TL * TPL), r32(std::min(TL * Nz, 192))));
  const size_t smem = (2 * (size_t)ncomp * TL * cline(Nz) + 2 * Nz) * sizeof(double2);
  const int ntiles = nkx * (Nyl / TL);
  ZPArgs a{};
  a.guard = c->guard ? c->sc : nullptr;
  a.B = c->P > 1 ? c->specC : c->specB;
  a.SL = slab_layout(c);
  a.ky_off = c->nranks > 1 ? c->rank * (Ny / c->P) : 0;
  a.Nyl = Nyl;
  a.Nx = c->n[0];
  a.Ny = Ny;
  a.Hx = c->Hx;
  a.kx0 = kxa;
  a.nkx = nkx;
  a.TL = TL;
  a.lgTL = ilog2(TL);
  a.scheme = c->scheme;
  for (int i = 0; i < 3; ++i) {
    a.h[i] = c->h[i];
    a.L[i] = c->L[i];
    a.qh[i] = 0.25 / c->h[i];
    a.qh2[i] = 0.0625 / (c->h[i] * c->h[i]);
    a.tpl[i] = 2.0 * 3.14159265358979323846 / c->L[i];
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
  // 1 (default): the wide 512 z pass takes its lines by bulk copies issued one tile ahead (PF variant;
  // one slab only).  Measured at 512^3: z6 4.22 -> 3.85 ms per launch.  2: the 256 kernels too.
  static const int zpf = [] {
    const char* e = std::getenv("FGD_ZPF");
    return e ? std::atoi(e) : 1;
  }();
  static const int z512w = [] {
    const char* e = std::getenv("FGD_Z512");
    return e ? std::atoi(e) : 1;   // 1: wide 32 x 16 plan (k_zreg512w), 0: 8 x 8 x 8 plan (k_zreg512)
  }();
  // measured at 512^3 (per sweep): 6 components 49.6 -> 46.2 ms with the wide plan; the 1-component
  // preconditioner pass 8.1 -> 10.8 ms (16-thread lines, 8 lines per CTA: too little parallelism per
  // SM), so it keeps the 8 x 8 x 8 plan unless FGD_Z512=2
  if (Nz == 512 && z512w && ((ncomp == 6 && mode == Z_PROJECT) || (ncomp == 1 && mode == Z_PRECOND && z512w == 2))) {
    const int TLr = std::min(ncomp == 6 ? 1 : 8, Nyl);
    a.TL = TLr;
    a.lgTL = ilog2(TLr);
    const int thr_r = 16 * ncomp * TLr;
    const size_t smem_r = ((size_t)ncomp * TLr * kZ5Line + 31 * 16 + 8) * sizeof(double2);
    const int nt_r = nkx * (Nyl / TLr);
    if (c->P > 1) {
      if (ncomp == 6) FGD_PLAUNCH(c, (k_zreg512w<6, Z_PROJECT, true>), thr_r, smem_r, nt_r, a);
      else FGD_PLAUNCH(c, (k_zreg512w<1, Z_PRECOND, true>), thr_r, smem_r, nt_r, a);
    } else if (ncomp == 6 && zpf) {
      FGD_PLAUNCH(c, (k_zreg512w<6, Z_PROJECT, false, true>), thr_r, smem_r, nt_r, a);
    } else {
      if (ncomp == 6) FGD_PLAUNCH(c, (k_zreg512w<6, Z_PROJECT, false>), thr_r, smem_r, nt_r, a);
      else FGD_PLAUNCH(c, (k_zreg512w<1, Z_PRECOND, false>), thr_r, smem_r, nt_r, a);
    }
    return FGD_OK;
  }
  if (Nz == 512 && ((ncomp == 6 && mode == Z_PROJECT) || (ncomp == 1 && mode == Z_PRECOND))) {
    const int thr_r = 64 * ncomp;
    const size_t smem_r = ((size_t)ncomp * k512Line + 448 + 56 + 512) * sizeof(double2);
    const int nt_r = nkx * Nyl;
    if (ncomp == 6) FGD_PLAUNCH(c, (k_zreg512<6, Z_PROJECT>), thr_r, smem_r, nt_r, a);
    else FGD_PLAUNCH(c, (k_zreg512<1, Z_PRECOND>), thr_r, smem_r, nt_r, a);
    return FGD_OK;
  }
  if (Nz == 256 && ((ncomp == 6 && mode == Z_PROJECT) || (ncomp == 1 && mode == Z_PRECOND))) {
    const int TLr = std::min(ncomp == 6 ? 1 : 8, Nyl);
    a.TL = TLr;
    a.lgTL = ilog2(TLr);
    const int thr_r = 16 * ncomp * TLr;
    const size_t smem_r = ((size_t)ncomp * TLr * kZLine + 240 + 256 + 8) * sizeof(double2);
    const int nt_r = nkx * (Nyl / TLr);
    // measured at 256^3: no gain from the prefetch (z6 0.432 vs 0.433 ms, z1 0.078 vs 0.082 ms: five
    // CTAs per SM already hide the 4 KB line loads), so the 256 kernels take it only with FGD_ZPF=2
    const bool pf = zpf == 2 && c->P == 1 && (ncomp * TLr) % 2 == 0;
    // factorised form (3 transformed components each way) is opt-in: measured 7.66 vs 4.72 ms per
    // 256^3 sweep -- its serial phases leave half of the CTA idle and spill; the FP64 saving does
    // not pay for that at this occupancy
    if (ncomp == 6 && c->scheme == 1 && TLr == 1 && std::getenv("FGD_ZFAC"))
      FGD_PLAUNCH(c, k_zfac256, 96, smem_r, nt_r, a);
    else if (ncomp == 6 && pf) FGD_PLAUNCH(c, (k_zreg256<6, Z_PROJECT, true>), thr_r, smem_r, nt_r, a);
    else if (ncomp == 6) FGD_PLAUNCH(c, (k_zreg256<6, Z_PROJECT>), thr_r, smem_r, nt_r, a);
    else if (pf) FGD_PLAUNCH(c, (k_zreg256<1, Z_PRECOND, true>), thr_r, smem_r, nt_r, a);
    else FGD_PLAUNCH(c, (k_zreg256<1, Z_PRECOND>), thr_r, smem_r, nt_r, a);
    return FGD_OK;
  }
#define ZPP(NN)                                                                                         \
  if (ncomp == 6 && mode == Z_PROJECT) FGD_PLAUNCH(c, (k_zpipe<NN, 6, Z_PROJECT>), thr, smem, ntiles, a);      \
  else if (ncomp == 1 && mode == Z_PRECOND) FGD_PLAUNCH(c, (k_zpipe<NN, 1, Z_PRECOND>), thr, smem, ntiles, a); \
  else if (ncomp == 3 && mode == Z_GRAD) FGD_PLAUNCH(c, (k_zpipe<NN, 3, Z_GRAD>), thr, smem, ntiles, a);       \
  else if (ncomp == 3 && mode == Z_DIV) FGD_PLAUNCH(c, (k_zpipe<NN, 3, Z_DIV>), thr, smem, ntiles, a);         \
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
  static const int ty_env = [] {
    const char* e = std::getenv("FGD_XI_TY");
    return e ? std::atoi(e) : 0;
  }();
  const int TY = ty_env > 0 ? std::min(Ny, ty_env) : choose_TYp(Nx, Ny);
  const int thr = std::min(256, r32(TY * fft_TPL(Nx / 2)));
  const bool pre = (mode == XI_MECH_CG || mode == XI_HELM_Z) && Nx != 256 && Nx != 512;
  const size_t smem = (2 * (size_t)TY * xline(Nx / 2) + Nx / 2 + Nx + (Nx == 256 ? 120 : Nx == 512 ? 240 : 0)) * sizeof(double2) +
                      (pre ? 2 * (size_t)TY * Nx * sizeof(double) : 0);
  const double* eop = in1;
  if (pre && ((uintptr_t)eop & 15) != 0) return set_err(c, FGD_EINVAL, "xinv: epilogue operand not 16 B aligned");
  const int ntiles = ncomp * Nz * (Ny / TY);
  XPArgs a{c->guard ? c->sc : nullptr, Ny, Nz, TY, ncomp, ilog2(TY), c->HxA, c->nvox, c->specA, in1, out0, io1, io2, c->sc, nullptr, red_op, red_slot,
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
  XPArgs a{c->guard ? c->sc : nullptr, Ny, Nz, TY, ncomp, ilog2(TY), c->HxA, c->nvox, c->specA, in0, nullptr, nullptr, nullptr, c->sc, nullptr, RED_NONE, 0,
           c->tabs.tw[ilog2(Nx / 2)], c->tabs.tw[ilog2(Nx)]};
  KTimer kt(c, ncomp == 6 ? KC_XFWD6 : KC_XFWD1);
#define XFP(NN) FGD_PLAUNCH(c, (k_xfpipe<NN>), thr, smem, ntiles, a);
  FGD_PDISPATCH(Nx, XFP)
#undef XFP
  return FGD_OK;
}

// y forward, z with the preconditioner multiply, y inverse of the one-component spectrum:
// fused cluster kernel when N2 = N3 = 256 on one GPU, else the three passes (+ exchanges).
fgd_status launch_precond_yz(fgd_ctx* c, double scale, double mean_ell2) {
  const int Ny = c->n[1], Nz = c->n[2];
  // opt-in (FGD_YZY=1): measured 3.70 ms vs 2.43 ms per 256^3 sweep for the three separate passes
  // (one 205 KB CTA per SM serialises load, DSMEM exchange and store; kept as the cluster variant)
  const bool yzy = std::getenv("FGD_YZY") != nullptr;
  if (yzy && Ny == 256 && Nz == 256 && c->P == 1) {
    YZArgs a{};
    a.z.guard = c->guard ? c->sc : nullptr;
    a.A = c->specA;
    a.Nz = c->nz_l;
    a.Hx = c->Hx;
    a.HxA = c->HxA;
    a.z.Nx = c->n[0];
    a.z.Ny = Ny;
    a.z.Hx = c->Hx;
    a.z.scheme = c->scheme;
    for (int i = 0; i < 3; ++i) {
      a.z.h[i] = c->h[i];
      a.z.L[i] = c->L[i];
      a.z.qh[i] = 0.25 / c->h[i];
      a.z.qh2[i] = 0.0625 / (c->h[i] * c->h[i]);
      a.z.tpl[i] = 2.0 * 3.14159265358979323846 / c->L[i];
    }
    a.z.scale = scale;
    a.z.mean_ell2 = mean_ell2;
    a.z.twx = c->tabs.tw[ilog2(c->n[0])];
    a.z.twy = c->tabs.tw[ilog2(Ny)];
    a.z.twz = c->tabs.tw[ilog2(Nz)];
    cudaError_t e = cudaFuncSetAttribute(k_yzy256, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kYZSmem);
    if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_yzy256 smem attr: ") + cudaGetErrorString(e));
    KTimer kt(c, KC_Z1);
    c->launches++;
    k_yzy256<<<c->Hx * kYZCl, 512, kYZSmem, c->stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_yzy256: ") + cudaGetErrorString(e));
    return FGD_OK;
  }
  return yz_round_trip(c, 1, Z_PRECOND, scale, nullptr, mean_ell2);
}

}  // namespace fgd
