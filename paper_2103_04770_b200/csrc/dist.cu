// Slab decomposition across GPUs: one process per GPU, z-slabs in real space,
// y-slabs in the z pass.  The data-path collectives are
//   * the two transposes of every 3D FFT round trip (block all-to-all of the slab layout of
//     pipes.cu: S[r][s] -> R[s][r]), as grouped ncclSend/ncclRecv on the context stream;
//   * the one-plane z-halo exchange of the Helmholtz stencil (periodic neighbours);
//   * allreduce of the Krylov dot products, macro averages and error norms (<= 14 doubles per
//     sync point) and an allreduce-max of the staggered strain error.
// With FGD_EMULATE_SLABS=P on a single GPU the same slab layout is used for all P slabs in one
// address space and the all-to-all is a set of device-to-device block copies -- one kernel over
// all ranks' data, which validates the transposition layout without a second GPU.
#include <nccl.h>

#include <cstdlib>
#include <cstring>

#include "reduce.cuh"

namespace fgd {

#define FGD_NCCL(ctx, call)                                                                    \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      return set_err(ctx, FGD_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));       \
  } while (0)

static ncclComm_t comm_of(const fgd_ctx* c) { return reinterpret_cast<ncclComm_t>(c->comm); }

fgd_status dist_init(fgd_ctx* c, const fgd_dist* d) {
  c->rank = 0;
  c->nranks = 1;
  c->P = 1;
  if (d && d->nranks > 1) {
    if (!d->nccl_id) return set_err(c, FGD_EINVAL, "nranks > 1 needs nccl_id (fgd_nccl_id on rank 0, broadcast)");
    if (d->rank < 0 || d->rank >= d->nranks) return set_err(c, FGD_EINVAL, "rank out of range");
    c->rank = d->rank;
    c->nranks = d->nranks;
    c->P = d->nranks;
    ncclUniqueId id;
    std::memcpy(&id, d->nccl_id, sizeof(id));
    ncclComm_t comm;
    FGD_NCCL(c, ncclCommInitRank(&comm, d->nranks, id, d->rank));
    c->comm = comm;
  } else if (const char* e = std::getenv("FGD_EMULATE_SLABS")) {
    const int p = std::atoi(e);
    if (p > 1) c->P = p;
  }
  const int P = c->P;
  if ((P & (P - 1)) != 0 || c->n[2] % P != 0 || c->n[1] % P != 0 || c->n[2] / P < 1 || c->n[1] / P < 1)
    return set_err(c, FGD_EINVAL, "slab count must be a power of two dividing N2 and N3");
  c->nz_l = c->nranks > 1 ? c->n[2] / c->nranks : c->n[2];
  c->z0 = c->rank * c->nz_l;
  return FGD_OK;
}

void dist_destroy(fgd_ctx* c) {
  if (c->comm) ncclCommDestroy(comm_of(c));
  c->comm = nullptr;
}

// S (specB) <-> R (specC).  Block (r, s) of S, size ncomp*Hx*nys*nzs complex, goes to block
// (s, r) of R.  fwd: S -> R (before the z pass); !fwd: R -> S (after it).
fgd_status exchange(fgd_ctx* c, int ncomp, bool fwd) {
  if (c->P == 1) return FGD_OK;
  const int P = c->P;
  const size_t blk = (size_t)ncomp * c->Hx * (c->n[1] / P) * (c->n[2] / P);
  double2* src = fwd ? c->specB : c->specC;
  double2* dst = fwd ? c->specC : c->specB;
  KTimer kt(c, KC_COMM);
  if (c->nranks == 1) {
    // emulated: every (r, s) block is local; S[r][s] -> R[s][r] (the map is an involution)
    for (int r = 0; r < P; ++r)
      for (int s = 0; s < P; ++s)
        FGD_CUDA(c, cudaMemcpyAsync(dst + (size_t)(s * P + r) * blk, src + (size_t)(r * P + s) * blk,
                                    blk * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    return FGD_OK;
  }
  FGD_NCCL(c, ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    FGD_NCCL(c, ncclSend(src + (size_t)p * blk, 2 * blk, ncclDouble, p, comm_of(c), c->stream));
    FGD_NCCL(c, ncclRecv(dst + (size_t)p * blk, 2 * blk, ncclDouble, p, comm_of(c), c->stream));
  }
  FGD_NCCL(c, ncclGroupEnd());
  return FGD_OK;
}

fgd_status allreduce_sum(fgd_ctx* c, double* dev, int count) {
  if (c->nranks == 1) return FGD_OK;
  KTimer kt(c, KC_COMM);
  FGD_NCCL(c, ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, comm_of(c), c->stream));
  return FGD_OK;
}

fgd_status allreduce_max_u64(fgd_ctx* c, unsigned long long* dev) {
  if (c->nranks == 1) return FGD_OK;
  KTimer kt(c, KC_COMM);
  FGD_NCCL(c, ncclAllReduce(dev, dev, 1, ncclUint64, ncclMax, comm_of(c), c->stream));
  return FGD_OK;
}

__global__ void k_finalize(DevScalars* sc, int op, int slot) {
  double t = sc->red[slot];
  finalize(sc, op, 0, &t, 1);
}

// For nranks > 1 a reducing kernel stores its LOCAL sum in red[kRedSlot]; the global sum is
// formed by an allreduce and the Krylov scalars are finalised by a one-thread kernel.
int red_op_for(const fgd_ctx* c, int op) { return (c->nranks > 1 && op != RED_NONE && op != RED_STORE) ? RED_STORE : op; }
int red_slot_for(const fgd_ctx* c, int op, int slot) {
  return (c->nranks > 1 && op != RED_NONE && op != RED_STORE) ? kDistSlot : slot;
}
fgd_status post_reduce(fgd_ctx* c, int op) {
  if (c->nranks == 1 || op == RED_NONE || op == RED_STORE) return FGD_OK;
  if (allreduce_sum(c, &c->sc->red[kDistSlot], 1) != FGD_OK) return FGD_ENCCL;
  c->launches++;
  k_finalize<<<1, 1, 0, c->stream>>>(c->sc, op, kDistSlot);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("k_finalize: ") + cudaGetErrorString(e));
  return FGD_OK;
}

// One-plane periodic z-halo of a rank-local field (nranks > 1): lo <- plane z0-1, hi <- plane z0+nz.
fgd_status halo_exchange(fgd_ctx* c, const void* field, size_t plane_bytes, void* lo, void* hi) {
  if (c->nranks == 1) return FGD_OK;
  const int up = (c->rank + 1) % c->nranks, dn = (c->rank + c->nranks - 1) % c->nranks;
  const char* f = static_cast<const char*>(field);
  const char* last = f + (size_t)(c->nz_l - 1) * plane_bytes;
  KTimer kt(c, KC_COMM);
  FGD_NCCL(c, ncclGroupStart());
  // order matters when up == dn (P = 2): first the plane sent up / received from below
  FGD_NCCL(c, ncclSend(last, plane_bytes, ncclChar, up, comm_of(c), c->stream));
  FGD_NCCL(c, ncclSend(f, plane_bytes, ncclChar, dn, comm_of(c), c->stream));
  FGD_NCCL(c, ncclRecv(lo, plane_bytes, ncclChar, dn, comm_of(c), c->stream));
  FGD_NCCL(c, ncclRecv(hi, plane_bytes, ncclChar, up, comm_of(c), c->stream));
  FGD_NCCL(c, ncclGroupEnd());
  return FGD_OK;
}

}  // namespace fgd

extern "C" fgd_status fgd_nccl_id(unsigned char* out) {
  if (!out) return FGD_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FGD_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return FGD_OK;
}
