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
#include "reduce.cuh"

namespace fgd {

struct SArgs {
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
constexpr int kRing = 6;
constexpr int kPlane = (SBY + 2) * (SBX + 2);

template <int MODE>
__global__ void __launch_bounds__(256, 2) k_stencil(SArgs s, const double* __restrict__ ain, const double* __restrict__ pold,
                                                     double* __restrict__ pout, double* __restrict__ q,
                                                     const uint8_t* __restrict__ phase, DevScalars* sc, double* partials,
                                                     int red_op, int red_slot) {
  constexpr int NA = MODE == ST_PCG ? 2 : 1;
  __shared__ double ring[kRing][NA][kPlane];
  __shared__ double lut[kMaxPhases];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * SBX + tx;
  const int TX = s.TX, TY = s.TY, TZ = s.TZ;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, z0 = blockIdx.z * TZ;
  const int Nx = s.Nx, Ny = s.Ny, Nz = s.Nz;
  const double beta = (MODE == ST_PCG) ? sc->beta : 0.0;
  if (tid < kMaxPhases) lut[tid] = s.lut[tid];
  const bool act = (tx < TX) && (ty < TY);
  const int gx = x0 + tx, gy = y0 + ty;
  const int xm = wrapi(gx - 1, Nx), ym = wrapi(gy - 1, Ny);
  const double ih[3] = {s.ih[0], s.ih[1], s.ih[2]};
  // plane elements staged by this thread (at most 2 of (TY+2) x (TX+2) <= 340), stored at the
  // fixed (SBY+2) x (SBX+2) pitch
  const int PW = TX + 2, PN = (TY + 2) * PW;
  const int i0 = tid, i1 = tid + SBX * SBY;
  const int py0 = i0 / PW, px0 = i0 - py0 * PW, py1 = i1 / PW, px1 = i1 - py1 * PW;
  const int o0 = py0 * (SBX + 2) + px0, o1 = py1 * (SBX + 2) + px1;
  const size_t r0 = (size_t)wrapi(y0 - 1 + py0, Ny) * Nx + wrapi(x0 - 1 + px0, Nx);
  const size_t r1 = (size_t)wrapi(y0 - 1 + py1, Ny) * Nx + wrapi(x0 - 1 + px1, Nx);
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
      double* d = ring[pi % kRing][0];
      if (i0 < PN) cp_async8(d + o0, pa + r0);
      if (i1 < PN) cp_async8(d + o1, pa + r1);
      if (MODE == ST_PCG) {
        double* dp = ring[pi % kRing][NA - 1];
        if (i0 < PN) cp_async8(dp + o0, pp + r0);
        if (i1 < PN) cp_async8(dp + o1, pp + r1);
      }
    }
    cp_async_commit_s();
  };
  double A0[3][3], A1[3][3];      // a at (x-1..x+1, y-1..y+1) of levels z and z+1
  double fp[4][3], fc[4][3];      // fluxes of the 4 corners at levels z-1 (fp) and z (fc)
  double red = 0.0;
  auto read3 = [&](int pi, double (&A)[3][3]) {
    const double* pa = ring[pi % kRing][0];
    const double* pp = ring[pi % kRing][NA - 1];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int o = (ty + dy) * (SBX + 2) + tx + dx;
        A[dy][dx] = MODE == ST_PCG ? fma(beta, pp[o], pa[o]) : pa[o];
      }
  };
  auto fluxes = [&](int zl, double (&F)[4][3]) {
    const uint8_t* pb = (s.dist && zl < 0) ? s.ph_lo : phase + (size_t)wrapi(zl, Nz) * Ny * Nx;
    const size_t row0 = (size_t)ym * Nx, row1 = (size_t)gy * Nx;
    const double l00 = lut[__ldg(pb + row0 + xm)], l10 = lut[__ldg(pb + row0 + gx)];
    const double l01 = lut[__ldg(pb + row1 + xm)], l11 = lut[__ldg(pb + row1 + gx)];
    corner_flux(A0, A1, 0, 0, l00, ih, F[0]);   // corner (x-1, y-1)
    corner_flux(A0, A1, 1, 0, l10, ih, F[1]);   // corner (x,   y-1)
    corner_flux(A0, A1, 0, 1, l01, ih, F[2]);   // corner (x-1, y)
    corner_flux(A0, A1, 1, 1, l11, ih, F[3]);   // corner (x,   y)
  };
  for (int pi = 0; pi < kRing; ++pi) issue(pi);
  cp_async_wait_s<kRing - 2>();       // planes 0 and 1 (levels z0 - 1, z0) have landed
  __syncthreads();
  if (act) {
    read3(0, A0);
    read3(1, A1);
    fluxes(z0 - 1, fp);
  }
  for (int zz = 0; zz < TZ; ++zz) {
    const int z = z0 + zz;
    __syncthreads();                  // all threads are done with the slot of plane zz
    issue(zz + kRing);                // into that slot
    cp_async_wait_s<kRing - 2>();     // plane zz + 2 (level z + 1) has landed
    __syncthreads();
    if (act) {
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) A0[dy][dx] = A1[dy][dx];
      read3(zz + 2, A1);
      fluxes(z, fc);
      // D^T gather: corner c = cx + 2 cy (cx = 1 - vx, cy = 1 - vy); level z (vz = 0) / z-1 (vz = 1)
      const double tx_ = (fc[0][0] - fc[1][0]) + (fc[2][0] - fc[3][0]) + (fp[0][0] - fp[1][0]) + (fp[2][0] - fp[3][0]);
      const double ty_ = (fc[0][1] - fc[2][1]) + (fc[1][1] - fc[3][1]) + (fp[0][1] - fp[2][1]) + (fp[1][1] - fp[3][1]);
      const double tz_ = (fp[0][2] - fc[0][2]) + (fp[1][2] - fc[1][2]) + (fp[2][2] - fc[2][2]) + (fp[3][2] - fc[3][2]);
      const double ac = A0[1][1];
      const double out = ac + tx_ * ih[0] + ty_ * ih[1] + tz_ * ih[2];
      const size_t g = ((size_t)z * Ny + gy) * Nx + gx;
      __stcs(q + g, out);
      if (MODE == ST_PCG) {
        __stcs(pout + g, ac);
        red = fma(ac, out, red);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j) fp[c][j] = fc[c][j];
    }
  }
  cp_async_wait_s<0>();
  if (MODE == ST_PCG) {
    double rr[1] = {red};
    reduce_finalize<1>(rr, partials, sc, red_op, red_slot);
  }
}

double mean_ell2(const fgd_ctx* c, int field) {
  double s = 0.0;
  for (int q = 0; q < c->nphases; ++q) s += (double)c->phase_count[q] * c->ell[field][q] * c->ell[field][q];
  return s / (double)c->nvox_g;
}

fgd_status launch_stencil(fgd_ctx* c, int field, int mode, const double* a, const double* zin, const double* pold,
                          double* pout, double* q, int red_op) {
  SArgs s{};
  s.Nx = c->n[0];
  s.Ny = c->n[1];
  s.Nz = c->nz_l;
  s.TX = std::min(SBX, s.Nx);
  s.TY = std::min(SBY, s.Ny);
  s.TZ = std::min(32, s.Nz);
  s.nvox = c->nvox;
  for (int j = 0; j < 3; ++j) s.ih[j] = 0.25 / c->h[j];
  for (int p = 0; p < kMaxPhases; ++p) s.lut[p] = (p < c->nphases) ? c->ell[field][p] * c->ell[field][p] : 0.0;
  dim3 grid(s.Nx / s.TX, s.Ny / s.TY, s.Nz / s.TZ);
  dim3 block(SBX, SBY);
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
  if (mode == ST_APPLY)
    k_stencil<ST_APPLY><<<grid, block, 0, c->stream>>>(s, a, nullptr, nullptr, q, c->phase, c->sc, c->partials, rop, rslot);
  else
    k_stencil<ST_PCG><<<grid, block, 0, c->stream>>>(s, zin, pold, pout, q, c->phase, c->sc, c->partials, rop, rslot);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_stencil: ") + cudaGetErrorString(e));
  return FGD_OK;
}

}  // namespace fgd
