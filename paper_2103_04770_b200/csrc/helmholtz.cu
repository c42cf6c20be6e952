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
#include "tma.cuh"

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
// BULK staging (TMA engine, 1-D bulk copies): plane rows at pitch SBX + 4 holding x0-2 .. x0+TX+1
// (16 B aligned runs), phase rows at pitch kPhWB holding x0-16 .. x0+TX-1
constexpr int kPhWB = SBX + 16;
// plane staging: per-thread cp.async (SG_CP), 1-D bulk copies per row (SG_BULK), or one tensor-map
// TMA box per array and plane (SG_TENSOR; ring slots padded to 128 B multiples, the TMA destination
// alignment)
enum StencilStage : int { SG_CP = 0, SG_BULK = 1, SG_TENSOR = 2 };
constexpr int pad16(int n) { return (n + 15) / 16 * 16; }
template <int RY>
constexpr int stencil_pl(int stg) {
  return stg == SG_TENSOR ? pad16((SBX + 4) * (SBY * RY + 2)) : (stg == SG_BULK ? (SBX + 4) : (SBX + 2)) * (SBY * RY + 2);
}
template <int RY>
constexpr int stencil_phl(int stg) {
  return stg == SG_TENSOR ? pad16((SBY * RY + 1) * kPhWB / 8) * 8 : (SBY * RY + 1) * (stg == SG_BULK ? kPhWB : kPhW);
}
template <int RY>
constexpr size_t stencil_smem(int na, int stg = SG_CP) {
  return (size_t)kRing * na * stencil_pl<RY>(stg) * sizeof(double) + (size_t)kRing * stencil_phl<RY>(stg) +
         (stg == SG_TENSOR ? 128 : 0);
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// SG_TENSOR, CTAs on the cell boundary: one plane (a, p_old if NA = 2, phase ids) into a ring slot of
// the wide layout by per-thread cp.async with the periodic wrap.  Out of line, so that its index
// registers are not live through the z march of the interior CTAs (which spilled otherwise).
template <int NA>
__device__ __noinline__ void stage_plane_wrap(int TX, int TY, int Nx, int Ny, const double* pa, const double* pp,
                                              const uint8_t* pb, double* d, uint8_t* dph, int PL) {
  constexpr int PX = SBX + 4;
  const int tx = threadIdx.x, ty = threadIdx.y, WYb = blockDim.y;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const bool cp1 = tx + 32 < TX + 2;
  const int cx0 = wrapi(x0 - 1 + tx, Nx), cx1 = wrapi(x0 + 31 + tx, Nx);
  for (int py = ty; py < TY + 2; py += WYb) {
    const size_t r = (size_t)wrapi(y0 - 1 + py, Ny) * Nx;
    double* drow = d + py * PX + 1;
    cp_async8(drow + tx, pa + r + cx0);
    if (NA == 2) cp_async8(drow + PL + tx, pp + r + cx0);
    if (cp1) {
      cp_async8(drow + tx + 32, pa + r + cx1);
      if (NA == 2) cp_async8(drow + PL + tx + 32, pp + r + cx1);
    }
  }
  if (tx < (TX + 8) / 4) {
    const int cw = wrapi(x0 - 4 + 4 * tx, Nx);
    for (int row = ty; row < TY + 1; row += WYb)
      cp_async4(dph + row * kPhWB + 12 + 4 * tx, pb + (size_t)wrapi(y0 - 1 + row, Ny) * Nx + cw);
  }
}

// FACT = true (default): the vertex fluxes and their D^T scatter in factored form.  D_j = Delta_j A_k A_l
// (forward difference along j, 2-point sums along the other two axes; all of them commute), so per
// level the 2 x 2 x 2 cube of a vertex is reduced through the z pair sums / differences
// S = a(z+1) + a(z), Dd = a(z+1) - a(z) of each column, their y pair sums and x pair sums, which the
// neighbouring vertices of the thread share:  D_x ~ sy(c+1) - sy(c), D_y ~ sx(r+1) - sx(r),
// D_z ~ dy(c) + dy(c+1).  The scatter D_j^T is factored the same way: per vertex row
// P = f_x(x-1) - f_x(x), Q = f_y(x-1) + f_y(x), R = f_z(x-1) + f_z(x); voxel row k takes
// E = (P + Q)(k) + (P - Q)(k+1) and Fz = R(k) + R(k+1), i.e. E - Fz on this level and E + Fz on the
// next.  Same operator, ~64 instead of ~113 FP64 operations per voxel (RY = 2); the
// additions are associated differently, so results agree with FACT = false to rounding only.
//
// BULK = true (opt-in, FGD_ST_BULK=1; needs N1 % 16 == 0): each plane of the ring arrives by 1-D bulk copies (the TMA
// engine; one per row and array, split in two or three only where the row wraps periodically),
// issued by warp 0 and completed on the slot's mbarrier -- no per-element copy instructions or index
// arithmetic in the other warps.  Measured and rejected at 512^3: 2.73 vs 1.73 ms per PCG stencil --
// ~100 row copies of 16-288 B per plane keep the bulk-copy engine busy far longer than the same bytes
// as per-thread 8 B cp.async.
template <int MODE, int RY, bool FACT, int STG>
__global__ void __launch_bounds__(256, RY == 4 ? 2 : 3) k_stencil(SArgs s, const double* __restrict__ ain, const double* __restrict__ pold,
                                                     double* __restrict__ pout, double* __restrict__ q,
                                                     const uint8_t* __restrict__ phase, DevScalars* sc, double* partials,
                                                     int red_op, int red_slot, const __grid_constant__ StencilMaps tm) {
  if (guard_done(s.guard)) return;   // converged Krylov loop: skip
  constexpr int NA = MODE == ST_PCG ? 2 : 1;
  constexpr bool BULK = STG == SG_BULK;
  constexpr bool WIDE = STG != SG_CP;              // ring rows hold x0-2 .. x0+TX+1, phase rows x0-16 .. x0+TX-1
  constexpr int PHW = WIDE ? kPhWB : kPhW;
  constexpr int PX = WIDE ? SBX + 4 : SBX + 2, PL = stencil_pl<RY>(STG), PHL = stencil_phl<RY>(STG);
  constexpr int XO = WIDE ? 1 : 0, PO = WIDE ? 15 : 3;   // ring column of x - 1, phase byte of x - 1
  extern __shared__ __align__(128) double ring_raw[];
  // [kRing][NA][PL], then phase ids [kRing][PHL]; SG_TENSOR: 128 B aligned slots
  double* ring = ring_raw + (STG == SG_TENSOR ? ((128u - (smem_u32(ring_raw) & 127u)) & 127u) / 8u : 0u);
  uint8_t* phs = reinterpret_cast<uint8_t*>(ring + (size_t)kRing * NA * PL);
  __shared__ uint64_t fullb[kRing];
  __shared__ double lut[kMaxPhases];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * SBX + tx, nthr = SBX * blockDim.y;
  const int TX = s.TX, TY = s.TY, TZ = s.TZ;      // TY = blockDim.y * RY
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, z0 = blockIdx.z * TZ;
  const int Nx = s.Nx, Ny = s.Ny, Nz = s.Nz;
  pdl_trigger();
  const bool iso = FACT && s.ih[0] == s.ih[1] && s.ih[1] == s.ih[2];
  if (tid < kMaxPhases) {
    lut[tid] = iso ? s.lut[tid] * (s.ih[0] * s.ih[0]) : s.lut[tid];   // FACT + iso: l^2 w
  }
  if ((BULK || STG == SG_TENSOR) && tid == 0) {
    for (int i = 0; i < kRing; ++i) mbar_init(&fullb[i], 1);
    fence_mbar_init();
  }
  if (BULK || STG == SG_TENSOR) __syncthreads();
  pdl_wait();
  const double beta = (MODE == ST_PCG) ? sc->beta : 0.0;
  const bool act = tx < TX;
  const int gx = x0 + tx, gyb = y0 + ty * RY;
  // D^T D carries 1/(4h_j) twice
  const double w0 = s.ih[0] * s.ih[0], w1 = s.ih[1] * s.ih[1], w2 = s.ih[2] * s.ih[2];
  const int PW = TX + 2, WYb = blockDim.y;
  const bool cp0 = tx < PW, cp1 = tx + 32 < PW;
  const int cx0 = wrapi(x0 - 1 + tx, Nx), cx1 = cp1 ? wrapi(x0 + 31 + tx, Nx) : 0;
  const int nw = (TX + 8) / 4, cw = tx < nw ? wrapi(x0 - 4 + 4 * tx, Nx) : 0;
  // bytes of one ring slot (BULK): the split copies of a wrapping row add up to the same total
  const unsigned slot_bytes = (unsigned)((TY + 2) * (TX + 4) * 8 * NA + (TY + 1) * (16 + TX));
  const bool wl = x0 == 0, wr = x0 + TX == Nx;
  // one plane row (global row start g) -> ring row d: x0-2 .. x0+TX+1
  auto copy_row = [&](double* d, const double* g, uint64_t* bar) {
    if (!wl && !wr) {
      bulk_g2s(d, g + x0 - 2, (unsigned)(TX + 4) * 8, bar);
    } else {
      bulk_g2s(d, g + (wl ? Nx - 2 : x0 - 2), 16, bar);
      bulk_g2s(d + 2, g + x0, (unsigned)TX * 8, bar);
      bulk_g2s(d + TX + 2, g + (wr ? 0 : x0 + TX), 16, bar);
    }
  };
  auto issue_bulk = [&](int pi) {
    if (pi > TZ + 1 || ty != 0) return;
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
    const uint8_t* pb = (s.dist && zl < 0) ? s.ph_lo : phase + (size_t)wrapi(zl, Nz) * Ny * Nx;
    const int slot = pi % kRing;
    double* d = ring + (size_t)slot * NA * PL;
    uint8_t* dph = phs + (size_t)slot * PHL;
    uint64_t* bar = &fullb[slot];
    if (tx == 0) {
      fence_proxy_async();                        // the slot's earlier generic reads before the async writes
      mbar_arrive_expect_tx(bar, slot_bytes);
    }
    __syncwarp();
    for (int row = tx; row < TY + 2; row += 32) {
      const size_t r = (size_t)wrapi(y0 - 1 + row, Ny) * Nx;
      copy_row(d + row * PX, pa + r, bar);
      if (MODE == ST_PCG) copy_row(d + PL + row * PX, pp + r, bar);
      if (row < TY + 1) {                         // phase bytes x0-16 .. x0+TX-1
        if (!wl) {
          bulk_g2s(dph + row * PHW, pb + r + x0 - 16, (unsigned)(16 + TX), bar);
        } else {
          bulk_g2s(dph + row * PHW, pb + r + Nx - 16, 16, bar);
          bulk_g2s(dph + row * PHW + 16, pb + r, (unsigned)TX, bar);
        }
      }
    }
  };
  // plane index pi = 0 .. TZ + 1 <-> level z0 - 1 + pi; one commit group per plane (possibly empty)
  // SG_TENSOR: CTAs whose haloed tile lies inside the periodic cell take each plane as one TMA box
  // per array (a, p_old, phase ids) on the slot's mbarrier, issued by one thread -- no per-element
  // copy instructions or index arithmetic; CTAs on the cell boundary (the box would need the
  // periodic wrap) stage the same ring layout with the per-thread cp.async copies below.
  const bool tmi = STG == SG_TENSOR && x0 >= 16 && x0 + TX + 2 <= Nx && y0 >= 1 && y0 + TY + 1 <= Ny;
  auto issue_tensor = [&](int pi) {
    if (pi > TZ + 1 || tid != 0) return;
    const int zw = wrapi(z0 - 1 + pi, Nz), slot = pi % kRing;
    uint64_t* bar = &fullb[slot];
    fence_proxy_async();                          // the slot's earlier generic reads before the async writes
    mbar_arrive_expect_tx(bar, (unsigned)((TY + 2) * (TX + 4) * 8 * NA + (TY + 1) * (16 + TX)));
    tma_load_3d(ring + (size_t)slot * NA * PL, &tm.a, x0 - 2, y0 - 1, zw, bar);
    if (MODE == ST_PCG) tma_load_3d(ring + (size_t)slot * NA * PL + PL, &tm.p, x0 - 2, y0 - 1, zw, bar);
    tma_load_3d(phs + (size_t)slot * PHL, &tm.ph, x0 - 16, y0 - 1, zw, bar);
  };
  auto issue = [&](int pi) {
    if (BULK) {
      issue_bulk(pi);
      return;
    }
    if (tmi) {
      issue_tensor(pi);
      return;
    }
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
      if (STG == SG_TENSOR) {                       // boundary CTA of the tensor variant (single slab)
        stage_plane_wrap<NA>(TX, TY, Nx, Ny, pa, pp, phase + (size_t)wrapi(zl, Nz) * Ny * Nx, ring + (size_t)(pi % kRing) * NA * PL,
                             phs + (size_t)(pi % kRing) * PHL, PL);
        cp_async_commit_s();
        return;
      }
      // thread (tx, ty) copies columns px = tx and px = tx + 32 (the two right halo columns when
      // TX = 32) of the rows py = ty, ty + WY, ...; the column offsets are fixed per thread (no
      // per-element index arithmetic: it dominated the instruction mix)
      double* d = ring + (size_t)(pi % kRing) * NA * PL;
      for (int py = ty; py < TY + 2; py += WYb) {
        const size_t r = (size_t)wrapi(y0 - 1 + py, Ny) * Nx;
        double* drow = d + py * PX;
        if (cp0) {
          cp_async8(drow + tx + XO, pa + r + cx0);
          if (MODE == ST_PCG) cp_async8(drow + PL + tx + XO, pp + r + cx0);
        }
        if (cp1) {
          cp_async8(drow + tx + 32 + XO, pa + r + cx1);
          if (MODE == ST_PCG) cp_async8(drow + PL + tx + 32 + XO, pp + r + cx1);
        }
      }
      const uint8_t* pb = (s.dist && zl < 0) ? s.ph_lo : phase + (size_t)wrapi(zl, Nz) * Ny * Nx;
      uint8_t* dph = phs + (size_t)(pi % kRing) * PHL;
      if (tx < nw)                                  // words per row: (TX + 8) / 4 <= 10
        for (int row = ty; row < TY + 1; row += WYb)
          cp_async4(dph + row * PHW + (WIDE ? 12 : 0) + 4 * tx, pb + (size_t)wrapi(y0 - 1 + row, Ny) * Nx + cw);
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
        const int o = (ty * RY + r) * PX + tx + dx + XO;
        A[r][dx] = MODE == ST_PCG ? fma(beta, pa[PL + o], pa[o]) : pa[o];
      }
  };
  // fluxes of the vertices of level zl (between Alo = level zl and Ahi = level zl + 1):
  // cur[k] += contribution to voxel (x, gyb + k, zl), nxt[k] += contribution to voxel (.., zl + 1)
  auto vertices = [&](int pi, double* cur, double* nxt) {
    const uint8_t* ph = phs + (size_t)(pi % kRing) * PHL + ty * RY * PHW + tx + PO;
#pragma unroll
    for (int vr = 0; vr <= RY; ++vr) {            // vertex row yv = gyb - 1 + vr: A rows vr, vr + 1
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {            // xv = x - 1 + cx: A columns cx, cx + 1
        const double l2 = lut[ph[vr * PHW + cx]];
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
  // factored form of vertices() (see the note above the kernel)
  auto vertices_f = [&](int pi, double* cur, double* nxt) {
    const uint8_t* ph = phs + (size_t)(pi % kRing) * PHL + ty * RY * PHW + tx + PO;
    double Sp[3], Dp[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Sp[c] = Ahi[0][c] + Alo[0][c];
      Dp[c] = Ahi[0][c] - Alo[0][c];
    }
    double sxp0 = Sp[0] + Sp[1], sxp1 = Sp[1] + Sp[2];
    double Up = 0.0, Rp = 0.0;
#pragma unroll
    for (int vr = 0; vr <= RY; ++vr) {            // vertex row yv = gyb - 1 + vr: A rows vr, vr + 1
      double Sn[3], Dn[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        Sn[c] = Ahi[vr + 1][c] + Alo[vr + 1][c];
        Dn[c] = Ahi[vr + 1][c] - Alo[vr + 1][c];
      }
      const double sxn0 = Sn[0] + Sn[1], sxn1 = Sn[1] + Sn[2];
      const double sy0 = Sp[0] + Sn[0], sy1 = Sp[1] + Sn[1], sy2 = Sp[2] + Sn[2];
      const double dy0 = Dp[0] + Dn[0], dy1 = Dp[1] + Dn[1], dy2 = Dp[2] + Dn[2];
      // one l^2 per vertex (times the common w = 1/(4h)^2 when h_x = h_y = h_z, else the three
      // weights scale the row sums P, Q, R below)
      const double l0 = lut[ph[vr * PHW]], l1 = lut[ph[vr * PHW + 1]];
      // vertex xv = x - 1 (columns 0, 1) and xv = x (columns 1, 2)
      const double fx0 = l0 * (sy1 - sy0), fx1 = l1 * (sy2 - sy1);
      const double fy0 = l0 * (sxn0 - sxp0), fy1 = l1 * (sxn1 - sxp1);
      const double fz0 = l0 * (dy0 + dy1), fz1 = l1 * (dy1 + dy2);
      double P = fx0 - fx1, Q = fy0 + fy1, R = fz0 + fz1;
      if (!iso) {
        P *= w0;
        Q *= w1;
        R *= w2;
      }
      const double U = P + Q, V = P - Q;
      if (vr >= 1) {                              // voxel row vr - 1: vertex rows vr - 1 (U) and vr (V)
        const double E = Up + V, Fz = Rp + R;
        cur[vr - 1] += E - Fz;
        nxt[vr - 1] += E + Fz;
      }
      Up = U;
      Rp = R;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        Sp[c] = Sn[c];
        Dp[c] = Dn[c];
      }
      sxp0 = sxn0;
      sxp1 = sxn1;
    }
  };
  double cur[RY], nxt[RY];
  double red = 0.0;
#pragma unroll
  for (int k = 0; k < RY; ++k) nxt[k] = 0.0;
  for (int pi = 0; pi < kRing; ++pi) issue(pi);
  if (BULK || tmi) {
    mbar_wait(&fullb[0], 0);
    mbar_wait(&fullb[1], 0);
  } else {
    cp_async_wait_s<kRing - 2>();     // planes 0 and 1 (levels z0 - 1, z0) have landed
  }
  __syncthreads();
  if (act) {
    readcol(0, Alo);
    readcol(1, Ahi);
    double scratch[RY];
#pragma unroll
    for (int k = 0; k < RY; ++k) scratch[k] = 0.0;
    if (FACT) vertices_f(0, scratch, nxt); else vertices(0, scratch, nxt);
  }
  __syncthreads();                    // planes 0 and 1 have been read by every thread
  for (int zz = 0; zz < TZ; ++zz) {
    const int z = z0 + zz;
    if (BULK || tmi) mbar_wait(&fullb[(zz + 2) % kRing], ((zz + 2) / kRing) & 1);
    else cp_async_wait_s<kRing - 3>();   // plane zz + 2 (level z + 1) has landed
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
      if (FACT) vertices_f(zz + 1, cur, nxt); else vertices(zz + 1, cur, nxt);   // vertex level z = plane zz + 1
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
  if (!BULK) cp_async_wait_s<0>();
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
    return e ? std::atoi(e) : 4;   // factored form: RY 4 (2 CTAs/SM, 128 registers, no spill)
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
  static const bool fact = [] {
    const char* e = std::getenv("FGD_ST_FACT");
    return e ? std::atoi(e) != 0 : true;
  }();
  // plane staging (FGD_ST_STAGE): 2 = tensor-map TMA boxes (default where it applies), 1 = 1-D bulk
  // copies per row (measured slower: 2.73 vs 1.73 ms at 512^3), 0 = per-thread cp.async
  const int stage_env = [] {                      // read per call (the tests switch it)
    const char* e = std::getenv("FGD_ST_STAGE");
    if (!e && std::getenv("FGD_ST_BULK")) return (int)SG_BULK;
    return e ? std::atoi(e) : (int)SG_TENSOR;
  }();
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const double* src_a = (mode == ST_APPLY) ? a : zin;
  const bool aligned = s.Nx % 16 == 0 && al16(src_a) && (mode == ST_APPLY || al16(pold)) && al16(c->phase);
  int stage = SG_CP;
  if (stage_env == SG_BULK && fact && aligned &&
      (!s.dist || (al16(s.a_lo) && al16(s.a_hi) && al16(s.p_lo) && al16(s.p_hi) && al16(s.ph_lo))))
    stage = SG_BULK;
  // tensor maps: full 32 x (8 RY) tiles of a single-slab cell with at least one interior tile
  StencilMaps tm{};
  if (stage_env == SG_TENSOR && fact && aligned && !s.dist && s.TX == SBX && WY == SBY && s.Nx >= 3 * SBX &&
      s.Ny >= 3 * s.TY) {
    const bool ok = tma_encode_3d(&tm.a, src_a, 8, s.Nx, s.Ny, s.Nz, s.TX + 4, s.TY + 2) &&
                    tma_encode_3d(&tm.p, mode == ST_PCG ? pold : src_a, 8, s.Nx, s.Ny, s.Nz, s.TX + 4, s.TY + 2) &&
                    tma_encode_3d(&tm.ph, c->phase, 1, s.Nx, s.Ny, s.Nz, s.TX + 16, s.TY + 1);
    if (ok) stage = SG_TENSOR;
  }
#define STL(RYV, FV, SV)                                                                                          \
  {                                                                                                               \
    const size_t smem = stencil_smem<RYV>(mode == ST_PCG ? 2 : 1, SV);                                           \
    if (mode == ST_APPLY) {                                                                                       \
      auto kf = k_stencil<ST_APPLY, RYV, FV, SV>;                                                                 \
      e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                      \
      if (e == cudaSuccess)                                                                                       \
        e = launch_pdl(kf, grid, block, smem, c->stream, s, a, (const double*)nullptr, (double*)nullptr, q,      \
                       (const uint8_t*)c->phase, c->sc, c->partials, rop, rslot, tm);                            \
    } else {                                                                                                      \
      auto kf = k_stencil<ST_PCG, RYV, FV, SV>;                                                                   \
      e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                      \
      if (e == cudaSuccess)                                                                                       \
        e = launch_pdl(kf, grid, block, smem, c->stream, s, zin, pold, pout, q, (const uint8_t*)c->phase, c->sc, \
                       c->partials, rop, rslot, tm);                                                              \
    }                                                                                                             \
  }
  if (stage == SG_TENSOR) {
    if (RY == 4) STL(4, true, SG_TENSOR) else if (RY == 2) STL(2, true, SG_TENSOR) else STL(1, true, SG_TENSOR)
  } else if (stage == SG_BULK) {
    if (RY == 4) STL(4, true, SG_BULK) else if (RY == 2) STL(2, true, SG_BULK) else STL(1, true, SG_BULK)
  } else if (fact) {
    if (RY == 4) STL(4, true, SG_CP) else if (RY == 2) STL(2, true, SG_CP) else STL(1, true, SG_CP)
  } else {
    if (RY == 4) STL(4, false, SG_CP) else if (RY == 2) STL(2, false, SG_CP) else STL(1, false, SG_CP)
  }
#undef STL
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_stencil: ") + cudaGetErrorString(e));
  return FGD_OK;
}

}  // namespace fgd
