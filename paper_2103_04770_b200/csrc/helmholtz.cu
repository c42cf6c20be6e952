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
  int Nx, Ny, Nz, TX, TY, TZ;
  size_t nvox;
  double ih[3];          // 1 / (4 h_j)
  double lut[kMaxPhases];  // l^2 per phase
};

enum StencilMode : int { ST_APPLY = 0, ST_PCG = 1 };

// periodic wrap for power-of-two extents (i >= -n)
__device__ __forceinline__ int wrapi(int i, int n) { return (i + n) & (n - 1); }

template <int MODE>
__global__ void __launch_bounds__(256) k_stencil(SArgs s, const double* __restrict__ ain, const double* __restrict__ pold,
                                                  double* __restrict__ pout, double* __restrict__ q,
                                                  const uint8_t* __restrict__ phase, DevScalars* sc, double* partials,
                                                  int red_op) {
  extern __shared__ double shm[];
  const int TX = s.TX, TY = s.TY, TZ = s.TZ;
  const int AX = TX + 2, AY = TY + 2, AZ = TZ + 2;
  const int FX = TX + 1, FY = TY + 1, FZ = TZ + 1;
  const int NA = AX * AY * AZ, NF = FX * FY * FZ;
  double* sa = shm;
  double* sf = shm + NA;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, z0 = blockIdx.z * TZ;
  const double beta = (MODE == ST_PCG) ? sc->beta : 0.0;
  for (int i = threadIdx.x; i < NA; i += blockDim.x) {
    const int ax = i % AX, ay = (i / AX) % AY, az = i / (AX * AY);
    const int gx = wrapi(x0 - 1 + ax, s.Nx), gy = wrapi(y0 - 1 + ay, s.Ny), gz = wrapi(z0 - 1 + az, s.Nz);
    const size_t g = ((size_t)gz * s.Ny + gy) * s.Nx + gx;
    double v = ain[g];
    if (MODE == ST_PCG) v = fma(beta, pold[g], v);
    sa[i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NF; i += blockDim.x) {
    const int fx = i % FX, fy = (i / FX) % FY, fz = i / (FX * FY);
    const int gx = wrapi(x0 - 1 + fx, s.Nx), gy = wrapi(y0 - 1 + fy, s.Ny), gz = wrapi(z0 - 1 + fz, s.Nz);
    const double l2 = s.lut[phase[((size_t)gz * s.Ny + gy) * s.Nx + gx]];
    const double* b = sa + (fz * AY + fy) * AX + fx;
    const double a000 = b[0], a100 = b[1], a010 = b[AX], a110 = b[AX + 1];
    const double a001 = b[AX * AY], a101 = b[AX * AY + 1], a011 = b[AX * AY + AX], a111 = b[AX * AY + AX + 1];
    const double gxv = ((a100 - a000) + (a110 - a010) + (a101 - a001) + (a111 - a011)) * s.ih[0];
    const double gyv = ((a010 - a000) + (a110 - a100) + (a011 - a001) + (a111 - a101)) * s.ih[1];
    const double gzv = ((a001 - a000) + (a101 - a100) + (a011 - a010) + (a111 - a110)) * s.ih[2];
    sf[i] = l2 * gxv;
    sf[NF + i] = l2 * gyv;
    sf[2 * NF + i] = l2 * gzv;
  }
  __syncthreads();
  double red[1] = {0.0};
  for (int i = threadIdx.x; i < TX * TY * TZ; i += blockDim.x) {
    const int ox = i % TX, oy = (i / TX) % TY, oz = i / (TX * TY);
    const double ac = sa[((oz + 1) * AY + oy + 1) * AX + ox + 1];
    // f at x - v, v in {0,1}^3: f-tile index (o + 1 - v)
    const int f111 = (oz * FY + oy) * FX + ox;  // v = (1,1,1)
    const double* fx_ = sf + f111;
    const double* fy_ = sf + NF + f111;
    const double* fz_ = sf + 2 * NF + f111;
    const int dX = 1, dY = FX, dZ = FX * FY;
    // v = (vx,vy,vz) -> offset (1-vx)dX + (1-vy)dY + (1-vz)dZ ; sign s_j(v) = +1 if v_j = 1
    // D_x^T: sum over v of s_x(v) f_x(x - v) = [f(vx=1) - f(vx=0)] summed over vy, vz
    const double tx = (fx_[0] - fx_[dX]) + (fx_[dY] - fx_[dY + dX]) + (fx_[dZ] - fx_[dZ + dX]) +
                      (fx_[dZ + dY] - fx_[dZ + dY + dX]);
    const double ty = (fy_[0] - fy_[dY]) + (fy_[dX] - fy_[dX + dY]) + (fy_[dZ] - fy_[dZ + dY]) +
                      (fy_[dZ + dX] - fy_[dZ + dX + dY]);
    const double tz = (fz_[0] - fz_[dZ]) + (fz_[dX] - fz_[dX + dZ]) + (fz_[dY] - fz_[dY + dZ]) +
                      (fz_[dY + dX] - fz_[dY + dX + dZ]);
    const double out = ac + tx * s.ih[0] + ty * s.ih[1] + tz * s.ih[2];
    const size_t g = ((size_t)(z0 + oz) * s.Ny + y0 + oy) * s.Nx + x0 + ox;
    q[g] = out;
    if (MODE == ST_PCG) {
      pout[g] = ac;
      red[0] = fma(ac, out, red[0]);
    }
  }
  if (MODE == ST_PCG) reduce_finalize<1>(red, partials, sc, red_op, 0);
}

double mean_ell2(const fgd_ctx* c, int field) {
  double s = 0.0;
  for (int q = 0; q < c->nphases; ++q) s += (double)c->phase_count[q] * c->ell[field][q] * c->ell[field][q];
  return s / (double)c->nvox;
}

fgd_status launch_stencil(fgd_ctx* c, int field, int mode, const double* a, const double* zin, const double* pold,
                          double* pout, double* q, int red_op) {
  SArgs s{};
  s.Nx = c->n[0];
  s.Ny = c->n[1];
  s.Nz = c->n[2];
  s.TX = std::min(32, s.Nx);
  s.TY = std::min(8, s.Ny);
  s.TZ = std::min(4, s.Nz);
  s.nvox = c->nvox;
  for (int j = 0; j < 3; ++j) s.ih[j] = 0.25 / c->h[j];
  for (int p = 0; p < kMaxPhases; ++p) s.lut[p] = (p < c->nphases) ? c->ell[field][p] * c->ell[field][p] : 0.0;
  dim3 grid(s.Nx / s.TX, s.Ny / s.TY, s.Nz / s.TZ);
  const size_t smem = sizeof(double) * ((size_t)(s.TX + 2) * (s.TY + 2) * (s.TZ + 2) +
                                        3 * (size_t)(s.TX + 1) * (s.TY + 1) * (s.TZ + 1));
  if (mode == ST_PCG) {
    fgd_status st = ensure_partials(c, (size_t)grid.x * grid.y * grid.z);
    if (st != FGD_OK) return st;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_stencil<ST_APPLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(k_stencil<ST_PCG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set = true;
  }
  c->launches++;
  KTimer kt(c, KC_STENCIL);
  if (mode == ST_APPLY)
    k_stencil<ST_APPLY><<<grid, 256, smem, c->stream>>>(s, a, nullptr, nullptr, q, c->phase, c->sc, c->partials, red_op);
  else
    k_stencil<ST_PCG><<<grid, 256, smem, c->stream>>>(s, zin, pold, pout, q, c->phase, c->sc, c->partials, red_op);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_stencil: ") + cudaGetErrorString(e));
  return FGD_OK;
}

}  // namespace fgd
