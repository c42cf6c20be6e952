// Deterministic grid reductions: warp shuffles -> block -> per-CTA partials -> the last CTA
// sums the partials in a fixed order and finalises the Krylov scalars on the device.
#pragma once
#include "fgd_internal.cuh"

namespace fgd {

__device__ __forceinline__ int lin_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
__device__ __forceinline__ int block_threads() { return blockDim.x * blockDim.y * blockDim.z; }

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sred) {
  const int tid = lin_tid();
  const int lane = tid & 31, warp = tid >> 5;
  const int nw = (block_threads() + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) sred[warp * NV + i] = v[i];
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += sred[w * NV + i];
      v[i] = s;
    }
  }
}

__device__ __forceinline__ void finalize(DevScalars* sc, int op, int slot, const double* t, int nv) {
  switch (op) {
    case RED_STORE:
      for (int i = 0; i < nv; ++i) sc->red[slot + i] = t[i];
      break;
    case RED_MECH_INIT:
      sc->rr = t[0];
      sc->bb = t[0];
      sc->beta = 0.0;
      sc->alpha = 0.0;
      sc->tol2 *= t[0];   // the host stored tol^2
      sc->done = 0;
      sc->iters = 0;
      break;
    case RED_MECH_PQ:
    case RED_HELM_PQ:
      sc->pq = t[0];
      sc->alpha = sc->rr / t[0];
      break;
    case RED_MECH_RR:
      sc->beta = t[0] / sc->rr;
      sc->rr = t[0];
      sc->iters += 1;
      if (t[0] < sc->tol2) sc->done = 1;
      break;
    case RED_HELM_RZ:
      sc->beta = t[0] / sc->rr;
      sc->rr = t[0];
      break;
    case RED_HELM_INIT:
      sc->rr = t[0];
      sc->beta = 0.0;
      break;
    case RED_HELM_RN:
      sc->rn2 = t[0];
      sc->iters += 1;
      if (t[0] < sc->tol2) sc->done = 1;
      break;
    case RED_BB:
      sc->bb = t[0];
      sc->tol2 *= t[0];   // the host stored tol^2
      sc->done = 0;
      sc->iters = 0;
      break;
    default:
      break;
  }
}

// Every thread of every CTA must call this (uniform control flow).
template <int NV>
__device__ __forceinline__ void reduce_finalize(double (&v)[NV], double* partials, DevScalars* sc, int op,
                                                int slot) {
  __shared__ double sred[32 * NV];
  __shared__ int am_last;
  const unsigned nblk = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int tid = lin_tid();
  block_sum<NV>(v, sred);
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[(size_t)bid * NV + i] = v[i];
    __threadfence();
    const unsigned prev = atomicAdd(&sc->counter[0], 1u);
    am_last = (prev == nblk - 1);
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    double t[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) t[i] = 0.0;
    for (unsigned b = tid; b < nblk; b += block_threads()) {
#pragma unroll
      for (int i = 0; i < NV; ++i) t[i] += __ldcg(&partials[(size_t)b * NV + i]);
    }
    block_sum<NV>(t, sred);
    if (tid == 0) {
      finalize(sc, op, slot, t, NV);
      sc->counter[0] = 0;
      __threadfence();
    }
  }
}

}  // namespace fgd
