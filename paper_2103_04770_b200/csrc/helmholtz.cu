// Real-space heterogeneous Helmholtz operator for the Willot rotated scheme.
//
// With k_j the symbol of the rotated finite difference (A-04), D_j is the real
// stencil "forward difference along j at the voxel vertex, averaged over the 4 cells that
// share the vertex":  (D_j a)(x) = 1/(4h_j) sum_{v in {0,1}^3} s_j(v) a(x+v), s_j = +1 if v_j = 1
// else -1, and D_j^T has symbol conj(k_j).  Hence the paper's Fourier-space operator
//   L^(a^) = a^ + sum_j conj(k_j) F(l^2 F^-1(k_j a^))            (A-09)
// is EXACTLY the real-space operator  L a = a + sum_j D_j^T (l^2 D_j a): a 27-point stencil
// that needs no FFT.  One kernel: load a 3D tile of a with a one-voxel halo into shared
// memory, form the vertex fluxes f_j = l^2(P) (D_j a)(P) for the tile plus its low halo, and
// gather L a.  The PCG variant builds p = z + beta p_old on the fly (halo included), writes p and
// q = L p and reduces p.q.  HBM traffic: read a (8 B) + phase (1 B) + write (8 B) per voxel.
#include <cstdlib>

#include "reduce.cuh"

namespace fgd {

#define TRYH(x)                   \
  do {                            \
    fgd_status s_ = (x);          \
    if (s_ != FGD_OK) return s_;  \
  } while (0)
#define FGD_CHECK_K(c, name)                                                                       \
  do {                                                                                             \
    cudaError_t e_ = cudaGetLastError();                                                           \
    if (e_ != cudaSuccess) return set_err(c, FGD_ECUDA, std::string(name) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct SArgs {
  const DevScalars* guard;
  int Nx, Ny, Nz, TX, TY, TZ;   // Nz: local planes
  size_t nvox;
  double ih[3];          // 1 / (4 h_j)
  double lut[kMaxPhases];  // l^2 per phase
  int dist;              // 1: z-slab of a multi-GPU run -> planes -1 and Nz come from the halos
  const double* a_lo;
  const double* a_hi;
  const double* p_lo;
  const double* p_hi;
  const uint8_t* ph_lo;
};

enum StencilMode : int { ST_APPLY = 0, ST_PCG = 1 };

// periodic wrap for power-of-two extents (i >= -n)
__device__ __forceinline__ int wrapi(int i, int n) { return (i + n) & (n - 1); }

// z-marching register-blocked stencil.  A CTA of 32 x 8 threads owns a 32 x 8 column block
// and marches over TZ output levels.  Per level it stages one (TX+2) x (TY+2) plane of `a`
// (a = z + beta p_old for PCG) in shared memory; every thread keeps the 3 x 3 neighbourhood of
// the current and next plane and the vertex fluxes of the previous level in registers:
//   f_j(P) = l^2(P) (D_j a)(P)  at the 4 corners P in {x-1, x} x {y-1, y} of level z,
//   (L a)(x) = a(x) + sum_j ih_j sum_{v in {0,1}^3} s_j(v) f_j(x - v)   (levels z and z-1).
// Shared-memory reads: 9 per voxel (vs ~45 for a flux-tile formulation).
constexpr int SBX = 32, SBY = 8;

__device__ __forceinline__ void corner_flux(const double (&A0)[3][3], const double (&A1)[3][3], int cx, int cy,
                                            double l2, const double* ih, double* f) {
  // corner P = (x-1+cx, y-1+cy): a(P + v) with v in {0,1}^3 -> A{vz}[cy+vy][cx+vx]
  const double a000 = A0[cy][cx], a100 = A0[cy][cx + 1], a010 = A0[cy + 1][cx], a110 = A0[cy + 1][cx + 1];
  const double a001 = A1[cy][cx], a101 = A1[cy][cx + 1], a011 = A1[cy + 1][cx], a111 = A1[cy + 1][cx + 1];
  f[0] = l2 * ih[0] * ((a100 - a000) + (a110 - a010) + (a101 - a001) + (a111 - a011));
  f[1] = l2 * ih[1] * ((a010 - a000) + (a110 - a100) + (a011 - a001) + (a111 - a101));
  f[2] = l2 * ih[2] * ((a001 - a000) + (a101 - a100) + (a011 - a010) + (a111 - a110));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit_s() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait_s() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// Planes of `a` (and p_old for PCG) arrive in a ring of kRing shared-memory slots by cp.async, up
// to kRing - 2 planes ahead of the level being computed, so that every SM keeps several planes of
// loads in flight through the z march.
//
// Each thread owns a column of RY voxels (x, y0' .. y0' + RY - 1) and keeps the (RY + 2) x 3
// neighbourhood of levels z and z + 1 in registers.  Per level it forms the vertex fluxes of the
// 2 x (RY + 1) vertices around its column ONCE (instead of 4 corners per voxel) and scatters them
// with the D^T signs into two accumulators: the voxels of level z (complete after this level) and
// of level z + 1 (seeded for the next level).  Vertex V(xv, yv, zl) sits at the far corner of voxel
// (xv, yv, zl), uses a on {xv, xv+1} x {yv, yv+1} x {zl, zl+1} and l^2 of voxel (xv, yv, zl).
constexpr int kRing = 5;

// phase ids of a plane: rows y0-1 .. y0+TY-1, 4-byte words covering x0-4 .. x0+TX+3 (aligned, so
// that the periodic wrap never splits a word); byte of x at (x - x0 + 4)
constexpr int kPhW = SBX + 8;
template <int RY>
constexpr size_t stencil_smem(int na) {
  return (size_t)kRing * na * (SBX + 2) * (SBY * RY + 2) * sizeof(double) + (size_t)kRing * (SBY * RY + 1) * kPhW;
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}

template <int MODE, int RY>
__global__ void __launch_bounds__(256, RY == 4 ? 2 : 3) k_stencil(SArgs s, const double* __restrict__ ain, const double* __restrict__ pold,
                                                     double* __restrict__ pout, double* __restrict__ q,
                                                     const uint8_t* __restrict__ phase, DevScalars* sc, double* partials,
                                                     int red_op, int red_slot) {
  if (guard_done(s.guard)) return;   // converged Krylov loop: skip
  constexpr int NA = MODE == ST_PCG ? 2 : 1;
  constexpr int PX = SBX + 2, PY = SBY * RY + 2, PL = PX * PY, PHL = (SBY * RY + 1) * kPhW;
  extern __shared__ double ring[];                 // [kRing][NA][PL], then phase ids [kRing][PHL]
  uint8_t* phs = reinterpret_cast<uint8_t*>(ring + (size_t)kRing * NA * PL);
  __shared__ double lut[kMaxPhases];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * SBX + tx, nthr = SBX * blockDim.y;
  const int TX = s.TX, TY = s.TY, TZ = s.TZ;      // TY = blockDim.y * RY
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, z0 = blockIdx.z * TZ;
  const int Nx = s.Nx, Ny = s.Ny, Nz = s.Nz;
  pdl_trigger();
  if (tid < kMaxPhases) lut[tid] = s.lut[tid];
  pdl_wait();
  const double beta = (MODE == ST_PCG) ? sc->beta : 0.0;
  const bool act = tx < TX;
  const int gx = x0 + tx, gyb = y0 + ty * RY;
  // D^T D carries 1/(4h_j) twice
  const double w0 = s.ih[0] * s.ih[0], w1 = s.ih[1] * s.ih[1], w2 = s.ih[2] * s.ih[2];
  const int PW = TX + 2, PN = (TY + 2) * PW;
  // plane index pi = 0 .. TZ + 1 <-> level z0 - 1 + pi; one commit group per plane (possibly empty)
  auto issue = [&](int pi) {
    if (pi <= TZ + 1) {
      const int zl = z0 - 1 + pi;
      const double* pa;
      const double* pp;
      if (s.dist && zl < 0) {
        pa = s.a_lo;
        pp = s.p_lo;
      } else if (s.dist && zl >= Nz) {
        pa = s.a_hi;
        pp = s.p_hi;
      } else {
        const size_t base = (size_t)wrapi(zl, Nz) * Ny * Nx;
        pa = ain + base;
        pp = pold + base;
      }
      double* d = ring + (size_t)(pi % kRing) * NA * PL;
      for (int e = tid; e < PN; e += nthr) {
        const int py = e / PW, px = e - py * PW;
        const size_t r = (size_t)wrapi(y0 - 1 + py, Ny) * Nx + wrapi(x0 - 1 + px, Nx);
        cp_async8(d + py * PX + px, pa + r);
        if (MODE == ST_PCG) cp_async8(d + PL + py * PX + px, pp + r);
      }
      const uint8_t* pb = (s.dist && zl < 0) ? s.ph_lo : phase + (size_t)wrapi(zl, Nz) * Ny * Nx;
      uint8_t* dph = phs + (size_t)(pi % kRing) * PHL;
      const int nw = (TX + 8) / 4;                 // words per row (TX is a multiple of 4)
      for (int e = tid; e < (TY + 1) * nw; e += nthr) {
        const int row = e / nw, wd = e - row * nw;
        const size_t r = (size_t)wrapi(y0 - 1 + row, Ny) * Nx + wrapi(x0 - 4 + 4 * wd, Nx);
        cp_async4(dph + row * kPhW + 4 * wd, pb + r);
      }
    }
    cp_async_commit_s();
  };
  double Alo[RY + 2][3], Ahi[RY + 2][3];   // rows gyb-1 .. gyb+RY, columns x-1 .. x+1; levels z, z+1
  auto readcol = [&](int pi, double (&A)[RY + 2][3]) {
    const double* pa = ring + (size_t)(pi % kRing) * NA * PL;
#pragma unroll
    for (int r = 0; r < RY + 2; ++r)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int o = (ty * RY + r) * PX + tx + dx;
        A[r][dx] = MODE == ST_PCG ? fma(beta, pa[PL + o], pa[o]) : pa[o];
      }
  };
  // fluxes of the vertices of level zl (between Alo = level zl and Ahi = level zl + 1):
  // cur[k] += contribution to voxel (x, gyb + k, zl), nxt[k] += contribution to voxel (.., zl + 1)
  auto vertices = [&](int pi, double* cur, double* nxt) {
    const uint8_t* ph = phs + (size_t)(pi % kRing) * PHL + ty * RY * kPhW + tx + 3;
#pragma unroll
    for (int vr = 0; vr <= RY; ++vr) {            // vertex row yv = gyb - 1 + vr: A rows vr, vr + 1
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {            // xv = x - 1 + cx: A columns cx, cx + 1
        const double l2 = lut[ph[vr * kPhW + cx]];
        const double a000 = Alo[vr][cx], a100 = Alo[vr][cx + 1], a010 = Alo[vr + 1][cx], a110 = Alo[vr + 1][cx + 1];
        const double a001 = Ahi[vr][cx], a101 = Ahi[vr][cx + 1], a011 = Ahi[vr + 1][cx], a111 = Ahi[vr + 1][cx + 1];
        const double f0 = l2 * w0 * ((a100 - a000) + (a110 - a010) + (a101 - a001) + (a111 - a011));
        const double f1 = l2 * w1 * ((a010 - a000) + (a110 - a100) + (a011 - a001) + (a111 - a101));
        const double f2 = l2 * w2 * ((a001 - a000) + (a101 - a100) + (a011 - a010) + (a111 - a110));
        const double ex = cx == 0 ? f0 : -f0;      // + from xv = x - 1, - from xv = x
        if (vr < RY) {                             // voxel row yv + 1: + f1
          cur[vr] += (ex + f1) - f2;
          nxt[vr] += (ex + f1) + f2;
        }
        if (vr >= 1) {                             // voxel row yv: - f1
          cur[vr - 1] += (ex - f1) - f2;
          nxt[vr - 1] += (ex - f1) + f2;
        }
      }
    }
  };
  double cur[RY], nxt[RY];
  double red = 0.0;
#pragma unroll
  for (int k = 0; k < RY; ++k) nxt[k] = 0.0;
  for (int pi = 0; pi < kRing; ++pi) issue(pi);
  cp_async_wait_s<kRing - 2>();       // planes 0 and 1 (levels z0 - 1, z0) have landed
  __syncthreads();
  if (act) {
    readcol(0, Alo);
    readcol(1, Ahi);
    double scratch[RY];
#pragma unroll
    for (int k = 0; k < RY; ++k) scratch[k] = 0.0;
    vertices(0, scratch, nxt);
  }
  __syncthreads();                    // planes 0 and 1 have been read by every thread
  for (int zz = 0; zz < TZ; ++zz) {
    const int z = z0 + zz;
    cp_async_wait_s<kRing - 3>();     // plane zz + 2 (level z + 1) has landed
    __syncthreads();
    // the slot of plane zz was last read at iteration zz - 1 (its phase ids, by vertices(zz)) or in
    // the prologue: every thread has passed the barrier above since, so it can be refilled now
    issue(zz + kRing);
    if (act) {
#pragma unroll
      for (int r = 0; r < RY + 2; ++r)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) Alo[r][dx] = Ahi[r][dx];
      readcol(zz + 2, Ahi);
#pragma unroll
      for (int k = 0; k < RY; ++k) {
        cur[k] = nxt[k];
        nxt[k] = 0.0;
      }
      vertices(zz + 1, cur, nxt);                // vertex level z = plane zz + 1
#pragma unroll
      for (int k = 0; k < RY; ++k) {
        const double ac = Alo[k + 1][1];
        const double out = ac + cur[k];
        const size_t g = ((size_t)z * Ny + gyb + k) * Nx + gx;
        __stcs(q + g, out);
        if (MODE == ST_PCG) {
          __stcs(pout + g, ac);
          red = fma(ac, out, red);
        }
      }
    }
  }
  cp_async_wait_s<0>();
  if (MODE == ST_PCG) {
    double rr[1] = {red};
    reduce_finalize<1>(rr, partials, sc, red_op, red_slot);
  }
}

// ---------------------------------------------------------------------------------------------
// Fourier form of the Helmholtz operator (the paper's L^ of P:716-718 / A-09 for ANY derivative
// symbol; required by the continuous scheme k_j = i xi_j, which is not a stencil):
//   y = a + F^-1 [ sum_j conj(k_j) F( l^2(x) F^-1( k_j F a ) ) ]
// as two 3-component FFT round trips of the library's passes: forward transform of three copies of
// a, z pass Z_GRAD (comp j *= k_j / N), inverse -> g_j = D_j a; g_j *= l^2(phase); forward, z pass
// Z_DIV (comp 0 = sum_j conj(k_j) g^_j / N), inverse of comp 0; y = a + that.  The PCG variant first
// forms p = z + beta p_old (written to pout) and reduces p.y.
// ---------------------------------------------------------------------------------------------
__global__ void k_hf_prep(const DevScalars* guard, size_t n, const double* a, const double* zin, const double* pold,
                          const DevScalars* sc, double* pout, double* g) {
  if (guard_done(guard)) return;
  const double beta = zin ? sc->beta : 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double v = zin ? fma(beta, pold[i], zin[i]) : a[i];
    if (pout) pout[i] = v;
    g[i] = v;
    g[n + i] = v;
    g[2 * n + i] = v;
  }
}
__global__ void k_hf_ell2(const DevScalars* guard, size_t n, double* g, const uint8_t* phase, SArgs s) {
  if (guard_done(guard)) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double l2 = s.lut[phase[i]];
    g[i] *= l2;
    g[n + i] *= l2;
    g[2 * n + i] *= l2;
  }
}
__global__ void k_hf_add(const DevScalars* guard, size_t n, const double* a, const double* t, double* y) {
  if (guard_done(guard)) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = a[i] + t[i];
}

fgd_status helm_fourier(fgd_ctx* c, int field, const double* a, const double* zin, const double* pold, double* pout,
                        double* y, int red_op) {
  const size_t n = c->nvox;
  if (!c->hg && cudaMalloc((void**)&c->hg, 3 * n * sizeof(double) + 16) != cudaSuccess)
    return set_err(c, FGD_ENOMEM, "Fourier-form Helmholtz gradient field");
  TRYH(ensure_spectral(c));
  const DevScalars* guard = c->guard ? c->sc : nullptr;
  const int nb = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
  // p (or a) into the three gradient slots; the value of a itself stays in pout (PCG) or a
  const double* av = zin ? pout : a;
  c->launches++;
  k_hf_prep<<<nb, 256, 0, c->stream>>>(guard, n, a, zin, pold, c->sc, zin ? pout : nullptr, c->hg);
  FGD_CHECK_K(c, "k_hf_prep");
  const double inv = 1.0 / (double)c->nvox_g;
  TRYH(pipe_xfwd_plain(c, 3, c->hg));
  TRYH(yz_round_trip(c, 3, Z_GRAD, inv, nullptr, 0.0));
  TRYH(pipe_xinv(c, 3, XI_STORE, c->hg, nullptr, nullptr, nullptr, RED_NONE, 0));
  SArgs s{};
  for (int p = 0; p < kMaxPhases; ++p) s.lut[p] = (p < c->nphases) ? c->ell[field][p] * c->ell[field][p] : 0.0;
  c->launches++;
  k_hf_ell2<<<nb, 256, 0, c->stream>>>(guard, n, c->hg, c->phase, s);
  FGD_CHECK_K(c, "k_hf_ell2");
  TRYH(pipe_xfwd_plain(c, 3, c->hg));
  TRYH(yz_round_trip(c, 3, Z_DIV, inv, nullptr, 0.0));
  TRYH(pipe_xinv(c, 1, XI_STORE, c->hg, nullptr, nullptr, nullptr, RED_NONE, 0));   // div term -> hg[0..n)
  c->launches++;
  k_hf_add<<<nb, 256, 0, c->stream>>>(guard, n, av, c->hg, y);
  FGD_CHECK_K(c, "k_hf_add");
  // p.y with the caller's reduction (the caller runs post_reduce, as after launch_stencil)
  if (red_op != RED_NONE) TRYH(launch_dot(c, n, av, y, red_op_for(c, red_op), red_slot_for(c, red_op, 0)));
  return FGD_OK;
}

double mean_ell2(const fgd_ctx* c, int field) {
  double s = 0.0;
  for (int q = 0; q < c->nphases; ++q) s += (double)c->phase_count[q] * c->ell[field][q] * c->ell[field][q];
  return s / (double)c->nvox_g;
}

fgd_status launch_stencil(fgd_ctx* c, int field, int mode, const double* a, const double* zin, const double* pold,
                          double* pout, double* q, int red_op) {
  // the 27-point stencil is the Willot symbol's exact real-space form (R-HELM); any other scheme
  // (continuous k = i xi, A-06) takes the Fourier form of the operator
  if (c->scheme != 1)
    return mode == ST_APPLY ? helm_fourier(c, field, a, nullptr, nullptr, nullptr, q, red_op)
                            : helm_fourier(c, field, nullptr, zin, pold, pout, q, red_op);
  SArgs s{};
  s.guard = c->guard ? c->sc : nullptr;
  s.Nx = c->n[0];
  s.Ny = c->n[1];
  s.Nz = c->nz_l;
  // rows per thread: 4 when the tile can be 32 rows high, else 2 / 1
  static const int ry_env = [] {
    const char* e = std::getenv("FGD_ST_RY");
    return e ? std::atoi(e) : 2;   // measured at 256^3: RY 2 / 32 levels 2.32 ms, RY 4 / 16 levels 2.43 ms
  }();
  const int RY = (s.Ny >= 4 * SBY && ry_env >= 4) ? 4 : (s.Ny >= 2 * SBY && ry_env >= 2 ? 2 : 1);
  const int WY = std::min(SBY, s.Ny / RY);
  s.TX = std::min(SBX, s.Nx);
  s.TY = WY * RY;
  static const int tz_env = [] {
    const char* e = std::getenv("FGD_ST_TZ");
    return e ? std::atoi(e) : 32;
  }();
  s.TZ = std::min(tz_env, s.Nz);
  s.nvox = c->nvox;
  for (int j = 0; j < 3; ++j) s.ih[j] = 0.25 / c->h[j];
  for (int p = 0; p < kMaxPhases; ++p) s.lut[p] = (p < c->nphases) ? c->ell[field][p] * c->ell[field][p] : 0.0;
  dim3 grid(s.Nx / s.TX, s.Ny / s.TY, s.Nz / s.TZ);
  dim3 block(SBX, WY);
  if (c->nranks > 1) {
    const size_t plane = (size_t)s.Nx * s.Ny;
    if (!c->halo && cudaMalloc((void**)&c->halo, 4 * plane * sizeof(double)) != cudaSuccess)
      return set_err(c, FGD_ENOMEM, "halo planes");
    s.dist = 1;
    s.a_lo = c->halo;
    s.a_hi = c->halo + plane;
    s.p_lo = c->halo + 2 * plane;
    s.p_hi = c->halo + 3 * plane;
    s.ph_lo = c->phase_halo;
    const double* src = (mode == ST_APPLY) ? a : zin;
    fgd_status st = halo_exchange(c, src, plane * sizeof(double), c->halo, c->halo + plane);
    if (st != FGD_OK) return st;
    if (mode == ST_PCG) {
      st = halo_exchange(c, pold, plane * sizeof(double), c->halo + 2 * plane, c->halo + 3 * plane);
      if (st != FGD_OK) return st;
    }
  }
  if (mode == ST_PCG) {
    fgd_status st = ensure_partials(c, (size_t)grid.x * grid.y * grid.z);
    if (st != FGD_OK) return st;
  }
  c->launches++;
  KTimer kt(c, KC_STENCIL);
  const int rop = red_op_for(c, red_op), rslot = red_slot_for(c, red_op, 0);
  cudaError_t e = cudaSuccess;
#define STL(RYV)                                                                                                  \
  {                                                                                                               \
    const size_t smem = stencil_smem<RYV>(mode == ST_PCG ? 2 : 1);                                               \
    if (mode == ST_APPLY) {                                                                                       \
      e = cudaFuncSetAttribute(k_stencil<ST_APPLY, RYV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e == cudaSuccess)                                                                                       \
        e = launch_pdl(k_stencil<ST_APPLY, RYV>, grid, block, smem, c->stream, s, a, (const double*)nullptr,     \
                       (double*)nullptr, q, (const uint8_t*)c->phase, c->sc, c->partials, rop, rslot);           \
    } else {                                                                                                      \
      e = cudaFuncSetAttribute(k_stencil<ST_PCG, RYV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
      if (e == cudaSuccess)                                                                                       \
        e = launch_pdl(k_stencil<ST_PCG, RYV>, grid, block, smem, c->stream, s, zin, pold, pout, q,              \
                       (const uint8_t*)c->phase, c->sc, c->partials, rop, rslot);                                \
    }                                                                                                             \
  }
  if (RY == 4) STL(4) else if (RY == 2) STL(2) else STL(1)
#undef STL
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_stencil: ") + cudaGetErrorString(e));
  return FGD_OK;
}

}  // namespace fgd
