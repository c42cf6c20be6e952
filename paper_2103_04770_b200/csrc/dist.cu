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
//
// Loopback transport (validation of the multi-rank code on ONE GPU): P contexts of one process,
// driven by P host threads, join an in-process group through an id from fgd_loopback_id().  Every
// collective is then stream-ordered device-to-device copies between the ranks' buffers, ordered by
// CUDA events and host barriers (no kernel ever waits on another rank's kernel):
//   publish: rank r records `ready_r` on its stream, posts its buffer pointer, host barrier,
//            then makes its stream wait for every ready_s;
//   move:    rank r copies what it receives from the peers' posted buffers (the same blocks NCCL
//            would deliver);
//   finish:  rank r records `done_r`, host barrier, its stream waits for every done_s (so no rank
//            overwrites a posted buffer before all peers have read it).
// Allreduces copy all P contributions into a per-rank stage and sum them in rank order in one
// kernel (identical result on every rank).  Every nranks > 1 branch of the library (slab layout
// with ky offsets, rank-0 zero frequency, z-halos, distributed finalise, max-ERR on bit patterns)
// runs unchanged; only the byte movement differs from NCCL.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "reduce.cuh"

namespace fgd {

#define TRYD(x)                   \
  do {                            \
    fgd_status s_ = (x);          \
    if (s_ != FGD_OK) return s_;  \
  } while (0)

#define FGD_NCCL(ctx, call)                                                                    \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      return set_err(ctx, FGD_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));       \
  } while (0)

static ncclComm_t comm_of(const fgd_ctx* c) { return reinterpret_cast<ncclComm_t>(c->comm); }

// ---- loopback group ---------------------------------------------------------------------------
static const char kLoopMagic[8] = {'F', 'G', 'D', 'L', 'O', 'O', 'P', 0};
constexpr int kLoopStage = 64;   // doubles per rank in an allreduce stage

struct LoopGroup {
  int P = 0;
  int members = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<const void*> ptr;
  std::vector<cudaEvent_t> ready, done;
  std::string key;
  // generation barrier with a timeout (a rank that left on an error must not hang the others forever)
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    const unsigned long long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; });
  }
};
static std::mutex g_loop_m;
static std::map<std::string, LoopGroup*> g_loops;

struct LoopRank {
  LoopGroup* g = nullptr;
  double* stage = nullptr;   // [P][kLoopStage]
};
static LoopRank* loop_of(const fgd_ctx* c) { return reinterpret_cast<LoopRank*>(c->loop); }

static fgd_status loop_join(fgd_ctx* c, const unsigned char* id) {
  const std::string key(reinterpret_cast<const char*>(id) + 8, 24);
  LoopGroup* g = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_loop_m);
    auto it = g_loops.find(key);
    if (it == g_loops.end()) {
      g = new LoopGroup();
      g->P = c->nranks;
      g->key = key;
      g->ptr.assign(c->nranks, nullptr);
      g->ready.assign(c->nranks, nullptr);
      g->done.assign(c->nranks, nullptr);
      g_loops[key] = g;
    } else {
      g = it->second;
    }
    if (g->P != c->nranks) return set_err(c, FGD_EINVAL, "loopback group: nranks differs between ranks");
    if (g->ready[c->rank]) return set_err(c, FGD_EINVAL, "loopback group: rank joined twice");
    if (cudaEventCreateWithFlags(&g->ready[c->rank], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done[c->rank], cudaEventDisableTiming) != cudaSuccess)
      return set_err(c, FGD_ECUDA, "loopback events");
    g->members++;
  }
  LoopRank* lr = new LoopRank();
  lr->g = g;
  c->loop = lr;
  if (cudaMalloc((void**)&lr->stage, (size_t)c->nranks * kLoopStage * sizeof(double)) != cudaSuccess)
    return set_err(c, FGD_ENOMEM, "loopback stage");
  // every rank has its events before anyone records into them
  if (!g->barrier()) return set_err(c, FGD_ENCCL, "loopback group: not all ranks joined within 300 s");
  return FGD_OK;
}

static void loop_leave(fgd_ctx* c) {
  LoopRank* lr = loop_of(c);
  if (!lr) return;
  LoopGroup* g = lr->g;
  // collective: a peer may still be issuing its stream waits on our events of the last collective
  g->barrier();
  if (lr->stage) cudaFree(lr->stage);
  {
    std::lock_guard<std::mutex> lk(g_loop_m);
    if (g->ready[c->rank]) cudaEventDestroy(g->ready[c->rank]);
    if (g->done[c->rank]) cudaEventDestroy(g->done[c->rank]);
    g->ready[c->rank] = g->done[c->rank] = nullptr;
    if (--g->members == 0) {
      g_loops.erase(g->key);
      delete g;
    }
  }
  delete lr;
  c->loop = nullptr;
}

static fgd_status loop_publish(fgd_ctx* c, const void* p, cudaStream_t st) {
  LoopGroup* g = loop_of(c)->g;
  g->ptr[c->rank] = p;
  FGD_CUDA(c, cudaEventRecord(g->ready[c->rank], st));
  if (!g->barrier()) return set_err(c, FGD_ENCCL, "loopback barrier timeout (publish)");
  for (int s = 0; s < g->P; ++s) FGD_CUDA(c, cudaStreamWaitEvent(st, g->ready[s], 0));
  return FGD_OK;
}
static fgd_status loop_publish(fgd_ctx* c, const void* p) { return loop_publish(c, p, c->stream); }

static fgd_status loop_finish(fgd_ctx* c, cudaStream_t st) {
  LoopGroup* g = loop_of(c)->g;
  FGD_CUDA(c, cudaEventRecord(g->done[c->rank], st));
  if (!g->barrier()) return set_err(c, FGD_ENCCL, "loopback barrier timeout (finish)");
  for (int s = 0; s < g->P; ++s) FGD_CUDA(c, cudaStreamWaitEvent(st, g->done[s], 0));
  return FGD_OK;
}
static fgd_status loop_finish(fgd_ctx* c) { return loop_finish(c, c->stream); }

// dev[i] = sum_s stage[s][i] (rank order), or the max of the 64-bit patterns
__global__ void k_loop_sum(double* dev, const double* stage, int P, int count) {
  const int i = threadIdx.x;
  if (i >= count) return;
  double t = 0.0;
  for (int s = 0; s < P; ++s) t += stage[s * kLoopStage + i];
  dev[i] = t;
}
__global__ void k_loop_max(unsigned long long* dev, const double* stage, int P) {
  unsigned long long m = 0;
  for (int s = 0; s < P; ++s) m = max(m, reinterpret_cast<const unsigned long long*>(stage)[s * kLoopStage]);
  *dev = m;
}

static fgd_status loop_allreduce(fgd_ctx* c, void* dev, int count, bool max_u64) {
  if (count > kLoopStage) return set_err(c, FGD_EINVAL, "loopback allreduce: count > 64");
  LoopRank* lr = loop_of(c);
  TRYD(loop_publish(c, dev));
  for (int s = 0; s < lr->g->P; ++s)
    FGD_CUDA(c, cudaMemcpyAsync(lr->stage + (size_t)s * kLoopStage, lr->g->ptr[s], (size_t)count * 8,
                                cudaMemcpyDeviceToDevice, c->stream));
  TRYD(loop_finish(c));
  c->launches++;
  if (max_u64)
    k_loop_max<<<1, 1, 0, c->stream>>>(static_cast<unsigned long long*>(dev), lr->stage, lr->g->P);
  else
    k_loop_sum<<<1, kLoopStage, 0, c->stream>>>(static_cast<double*>(dev), lr->stage, lr->g->P, count);
  FGD_CUDA(c, cudaGetLastError());
  return FGD_OK;
}

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
    if (std::memcmp(d->nccl_id, kLoopMagic, 8) == 0) {
      if (d->nranks > 64) return set_err(c, FGD_EINVAL, "loopback: at most 64 ranks");
      TRYD(loop_join(c, d->nccl_id));
      goto slabs;
    }
    ncclUniqueId id;
    std::memcpy(&id, d->nccl_id, sizeof(id));
    ncclComm_t comm;
    FGD_NCCL(c, ncclCommInitRank(&comm, d->nranks, id, d->rank));
    c->comm = comm;
  } else if (const char* e = std::getenv("FGD_EMULATE_SLABS")) {
    const int p = std::atoi(e);
    if (p > 1) c->P = p;
  }
slabs:
  const int P = c->P;
  if ((P & (P - 1)) != 0 || c->n[2] % P != 0 || c->n[1] % P != 0 || c->n[2] / P < 1 || c->n[1] / P < 1)
    return set_err(c, FGD_EINVAL, "slab count must be a power of two dividing N2 and N3");
  c->nz_l = c->nranks > 1 ? c->n[2] / c->nranks : c->n[2];
  c->z0 = c->rank * c->nz_l;
  return FGD_OK;
}

void dist_destroy(fgd_ctx* c) {
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  for (cudaEvent_t e : c->ov_ev) cudaEventDestroy(e);
  c->ov_ev.clear();
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  c->comm_stream = nullptr;
  for (void* q : c->peer_ipc) cudaIpcCloseMemHandle(q);
  c->peer_ipc.clear();
  if (c->bar_buf) cudaFree(c->bar_buf);
  c->bar_buf = nullptr;
  loop_leave(c);
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
  if (c->loop) {
    TRYD(loop_publish(c, src));
    for (int p = 0; p < P; ++p)
      FGD_CUDA(c, cudaMemcpyAsync(dst + (size_t)p * blk, static_cast<const double2*>(loop_of(c)->g->ptr[p]) +
                                                             (size_t)c->rank * blk,
                                  blk * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    return loop_finish(c);
  }
  FGD_NCCL(c, ncclGroupStart());
  for (int p = 0; p < P; ++p) {
    FGD_NCCL(c, ncclSend(src + (size_t)p * blk, 2 * blk, ncclDouble, p, comm_of(c), c->stream));
    FGD_NCCL(c, ncclRecv(dst + (size_t)p * blk, 2 * blk, ncclDouble, p, comm_of(c), c->stream));
  }
  FGD_NCCL(c, ncclGroupEnd());
  return FGD_OK;
}

// One kx chunk [kxa, kxb) of the transpose, on stream st: for every peer p and component cc the
// contiguous run of (kxb - kxa) * nys * nzs complex values at kx = kxa of block p (nranks > 1 only).
static fgd_status exchange_chunk(fgd_ctx* c, int ncomp, bool fwd, int kxa, int kxb, cudaStream_t st) {
  const int P = c->P;
  kxb = std::min(kxb, c->Hx);
  if (kxb <= kxa) return FGD_OK;
  const size_t nn = (size_t)(c->n[1] / P) * (c->n[2] / P);
  const size_t blk = (size_t)ncomp * c->Hx * nn;
  const size_t cnt = (size_t)(kxb - kxa) * nn;
  double2* src = fwd ? c->specB : c->specC;
  double2* dst = fwd ? c->specC : c->specB;
  if (c->loop) {
    TRYD(loop_publish(c, src, st));
    for (int p = 0; p < P; ++p) {
      const double2* peer = static_cast<const double2*>(loop_of(c)->g->ptr[p]) + (size_t)c->rank * blk;
      for (int cc = 0; cc < ncomp; ++cc) {
        const size_t off = ((size_t)cc * c->Hx + kxa) * nn;
        FGD_CUDA(c, cudaMemcpyAsync(dst + (size_t)p * blk + off, peer + off, cnt * sizeof(double2),
                                    cudaMemcpyDeviceToDevice, st));
      }
    }
    return loop_finish(c, st);
  }
  FGD_NCCL(c, ncclGroupStart());
  for (int p = 0; p < P; ++p)
    for (int cc = 0; cc < ncomp; ++cc) {
      const size_t off = (size_t)p * blk + ((size_t)cc * c->Hx + kxa) * nn;
      FGD_NCCL(c, ncclSend(src + off, 2 * cnt, ncclDouble, p, comm_of(c), st));
      FGD_NCCL(c, ncclRecv(dst + off, 2 * cnt, ncclDouble, p, comm_of(c), st));
    }
  FGD_NCCL(c, ncclGroupEnd());
  return FGD_OK;
}

// ---- peer-store transposes -------------------------------------------------
// FGD_PEER=1 (opt-in; nranks in [2, kMaxPeers], one NVLink domain): the y-forward pass stores its output
// straight into the z-pass buffers R of the destination ranks and the y-inverse pass loads from them
// (YArgs::peer), so the two transposes of a round trip disappear into the passes; what remains are two
// stream-ordered rank barriers (after the y-forward stores, after the z pass).  The peers' buffers are
// mapped once: loopback ranks share the address space; NCCL ranks allgather cudaIpcMemHandles of their
// specC allocations and open them (same node, P2P capable -- the 8 x B200 NVSwitch box).  Measured
// alternative to the ncclSend/ncclRecv transposes; unmeasured here (one GPU per call).
bool peer_mode(fgd_ctx* c) {
  const char* e = std::getenv("FGD_PEER");   // read per call (the tests switch it)
  return e && std::atoi(e) != 0 && c->nranks > 1 && c->nranks <= kMaxPeers;
}

static fgd_status peer_setup(fgd_ctx* c) {
  if (c->peer_ready) return FGD_OK;
  const int P = c->nranks;
  if (!c->bar_buf) {
    FGD_CUDA(c, cudaMalloc((void**)&c->bar_buf, 64));
    FGD_CUDA(c, cudaMemsetAsync(c->bar_buf, 0, 64, c->stream));
  }
  if (c->loop) {
    TRYD(loop_publish(c, c->specC));
    for (int s = 0; s < P; ++s) c->peerC[s] = static_cast<double2*>(const_cast<void*>(loop_of(c)->g->ptr[s]));
    TRYD(loop_finish(c));
  } else {
    cudaIpcMemHandle_t mine;
    FGD_CUDA(c, cudaIpcGetMemHandle(&mine, c->specC));
    unsigned char* dh = nullptr;
    FGD_CUDA(c, cudaMalloc((void**)&dh, (size_t)(P + 1) * sizeof(mine)));
    FGD_CUDA(c, cudaMemcpyAsync(dh + (size_t)P * sizeof(mine), &mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
    FGD_NCCL(c, ncclAllGather(dh + (size_t)P * sizeof(mine), dh, sizeof(mine), ncclChar, comm_of(c), c->stream));
    std::vector<cudaIpcMemHandle_t> all(P);
    FGD_CUDA(c, cudaMemcpyAsync(all.data(), dh, (size_t)P * sizeof(mine), cudaMemcpyDeviceToHost, c->stream));
    FGD_CUDA(c, cudaStreamSynchronize(c->stream));
    cudaFree(dh);
    for (int s = 0; s < P; ++s) {
      if (s == c->rank) {
        c->peerC[s] = c->specC;
        continue;
      }
      void* q = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&q, all[s], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return set_err(c, FGD_ECUDA, std::string("peer-store transposes: cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
      c->peer_ipc.push_back(q);
      c->peerC[s] = static_cast<double2*>(q);
    }
  }
  c->peer_ready = true;
  return FGD_OK;
}

// every rank's earlier work on its stream completes before any rank's later work starts
static fgd_status rank_barrier(fgd_ctx* c) {
  KTimer kt(c, KC_COMM);
  if (c->loop) {
    TRYD(loop_publish(c, nullptr));
    return loop_finish(c);
  }
  FGD_NCCL(c, ncclAllReduce(c->bar_buf, c->bar_buf, 1, ncclDouble, ncclSum, comm_of(c), c->stream));
  return FGD_OK;
}

// Number of kx chunks of the overlapped round trip (nranks > 1): FGD_OVERLAP (default 4; 1 = the
// monolithic transpose), at most HxA / 4.
static int overlap_chunks(const fgd_ctx* c) {
  const char* e = std::getenv("FGD_OVERLAP");   // read per call (the tests switch it)
  const int k = e ? std::atoi(e) : 4;
  return std::max(1, std::min(k, c->HxA / 4));
}

// y-forward, transpose, z pass (projection or preconditioner), transpose back, y-inverse of the
// spectra in specA/specB: the y/z half of every operator apply.  With nranks > 1 the kx range is
// cut into K chunks (multiples of 4 columns) and pipelined over two streams:
//   compute: y(0) .. y(K-1) | z(0) .. z(K-1) | yinv(0) .. yinv(K-1)
//   comm:          a2a(0) .. a2a(K-1) | a2a'(0) .. a2a'(K-1)
// chunk i's transpose runs while the compute stream works on chunk i+1, each compute step waiting
// only for its own chunk's transpose (events).  The persistent kernels of the overlapped phase
// leave kCommSMs SMs free for the communication kernels.
constexpr int kCommSMs = 8;
fgd_status yz_round_trip(fgd_ctx* c, int ncomp, int zmode, double scale, const double* shift, double mean_ell2) {
  if (peer_mode(c)) {
    // R[s][r] on rank s is written by rank r's y-forward and read back by rank r's y-inverse only, and
    // rank s's z pass runs between the two barriers: no other ordering is needed across round trips
    TRYD(peer_setup(c));
    struct On {
      fgd_ctx* c;
      explicit On(fgd_ctx* cc) : c(cc) { c->peer_on = true; }
      ~On() { c->peer_on = false; }
    } on(c);
    TRYD(pipe_y(c, ncomp, false));
    TRYD(rank_barrier(c));
    TRYD(pipe_z(c, ncomp, zmode, scale, shift, mean_ell2));
    TRYD(rank_barrier(c));
    return pipe_y(c, ncomp, true);
  }
  // One GPU, large grids: the y passes are bound by the strided side of their transpose and the z
  // pass by the FP64 pipe, so they can share the SMs: the kx range is cut into K chunks, the z pass of
  // chunk i runs on a second stream next to the y-forward of chunk i + 1 / the y-inverse of chunk
  // i - 1, every persistent grid capped so that CTAs of both kernels are resident together
  // (FGD_YZ_OVERLAP=K, FGD_YZ_SPLIT="ry,rz": SMs' worth of CTAs the y / z grids leave free).
  if (c->nranks == 1 && c->P == 1 && c->nvox > ((size_t)1 << 21)) {
    const char* eo = std::getenv("FGD_YZ_OVERLAP");
    const int Ko = eo ? std::min(std::atoi(eo), c->HxA / 4) : 0;
    if (Ko > 1) {
      int ry = 74, rz = 74;
      if (const char* es = std::getenv("FGD_YZ_SPLIT")) std::sscanf(es, "%d,%d", &ry, &rz);
      if (!c->comm_stream) FGD_CUDA(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
      while ((int)c->ov_ev.size() < 2 * Ko + 1) {
        cudaEvent_t e;
        FGD_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ov_ev.push_back(e);
      }
      cudaEvent_t* ey = c->ov_ev.data();
      cudaEvent_t* ez = ey + Ko;
      std::vector<int> kb(Ko + 1);
      const int n4 = c->HxA / 4;
      for (int i = 0; i <= Ko; ++i) kb[i] = 4 * (int)((long long)i * n4 / Ko);
      cudaStream_t s1 = c->stream, s2 = c->comm_stream;
      struct Restore {
        fgd_ctx* c;
        cudaStream_t s;
        ~Restore() {
          c->stream = s;
          c->sm_reserve = 0;
        }
      } restore{c, s1};
      // s2 starts after everything queued on s1 so far (the x pass that produced the spectra)
      FGD_CUDA(c, cudaEventRecord(c->ov_ev[2 * Ko], s1));
      FGD_CUDA(c, cudaStreamWaitEvent(s2, c->ov_ev[2 * Ko], 0));
      c->sm_reserve = ry;
      for (int i = 0; i < Ko; ++i) {
        TRYD(pipe_y(c, ncomp, false, kb[i], kb[i + 1]));
        FGD_CUDA(c, cudaEventRecord(ey[i], s1));
      }
      c->stream = s2;
      c->sm_reserve = rz;
      for (int i = 0; i < Ko; ++i) {
        FGD_CUDA(c, cudaStreamWaitEvent(s2, ey[i], 0));
        TRYD(pipe_z(c, ncomp, zmode, scale, shift, mean_ell2, kb[i], kb[i + 1]));
        FGD_CUDA(c, cudaEventRecord(ez[i], s2));
      }
      c->stream = s1;
      c->sm_reserve = ry;
      for (int i = 0; i < Ko; ++i) {
        FGD_CUDA(c, cudaStreamWaitEvent(s1, ez[i], 0));
        TRYD(pipe_y(c, ncomp, true, kb[i], kb[i + 1]));
      }
      return FGD_OK;
    }
  }
  const int K = c->nranks > 1 ? overlap_chunks(c) : 1;
  if (K <= 1) {
    TRYD(pipe_y(c, ncomp, false));
    TRYD(exchange(c, ncomp, true));
    TRYD(pipe_z(c, ncomp, zmode, scale, shift, mean_ell2));
    TRYD(exchange(c, ncomp, false));
    return pipe_y(c, ncomp, true);
  }
  if (!c->comm_stream) {
    FGD_CUDA(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  }
  while ((int)c->ov_ev.size() < 4 * K) {
    cudaEvent_t e;
    FGD_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ov_ev.push_back(e);
  }
  cudaEvent_t* ey = c->ov_ev.data();
  cudaEvent_t *ea = ey + K, *ez = ey + 2 * K, *eb = ey + 3 * K;
  std::vector<int> kb(K + 1);
  const int n4 = c->HxA / 4;
  for (int i = 0; i <= K; ++i) kb[i] = 4 * (int)((long long)i * n4 / K);
  struct Reserve {
    fgd_ctx* c;
    explicit Reserve(fgd_ctx* cc) : c(cc) { c->sm_reserve = kCommSMs; }
    ~Reserve() { c->sm_reserve = 0; }
  } reserve(c);
  cudaStream_t cs = c->comm_stream;
  for (int i = 0; i < K; ++i) {
    TRYD(pipe_y(c, ncomp, false, kb[i], kb[i + 1]));
    FGD_CUDA(c, cudaEventRecord(ey[i], c->stream));
  }
  for (int i = 0; i < K; ++i) {
    FGD_CUDA(c, cudaStreamWaitEvent(cs, ey[i], 0));
    TRYD(exchange_chunk(c, ncomp, true, kb[i], kb[i + 1], cs));
    FGD_CUDA(c, cudaEventRecord(ea[i], cs));
  }
  for (int i = 0; i < K; ++i) {
    FGD_CUDA(c, cudaStreamWaitEvent(c->stream, ea[i], 0));
    TRYD(pipe_z(c, ncomp, zmode, scale, shift, mean_ell2, kb[i], kb[i + 1]));
    FGD_CUDA(c, cudaEventRecord(ez[i], c->stream));
  }
  for (int i = 0; i < K; ++i) {
    FGD_CUDA(c, cudaStreamWaitEvent(cs, ez[i], 0));
    TRYD(exchange_chunk(c, ncomp, false, kb[i], kb[i + 1], cs));
    FGD_CUDA(c, cudaEventRecord(eb[i], cs));
  }
  for (int i = 0; i < K; ++i) {
    FGD_CUDA(c, cudaStreamWaitEvent(c->stream, eb[i], 0));
    TRYD(pipe_y(c, ncomp, true, kb[i], kb[i + 1]));
  }
  return FGD_OK;
}

fgd_status allreduce_sum(fgd_ctx* c, double* dev, int count) {
  if (c->nranks == 1) return FGD_OK;
  KTimer kt(c, KC_COMM);
  if (c->loop) return loop_allreduce(c, dev, count, false);
  FGD_NCCL(c, ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, comm_of(c), c->stream));
  return FGD_OK;
}

fgd_status allreduce_max_u64(fgd_ctx* c, unsigned long long* dev) {
  if (c->nranks == 1) return FGD_OK;
  KTimer kt(c, KC_COMM);
  if (c->loop) return loop_allreduce(c, dev, 1, true);
  FGD_NCCL(c, ncclAllReduce(dev, dev, 1, ncclUint64, ncclMax, comm_of(c), c->stream));
  return FGD_OK;
}

// guard: the Krylov loop's convergence guard (nullptr outside a batched loop); once the device flag
// is set, the reducing kernels of the remaining launched iterations skip, the allreduce then sums
// stale partials, and the finalise must skip too (else it would count and apply a phantom iteration)
__global__ void k_finalize(DevScalars* sc, const DevScalars* guard, int op, int slot) {
  if (guard_done(guard)) return;
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
  k_finalize<<<1, 1, 0, c->stream>>>(c->sc, c->guard ? c->sc : nullptr, op, kDistSlot);
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
  if (c->loop) {
    TRYD(loop_publish(c, field));
    const LoopGroup* g = loop_of(c)->g;
    FGD_CUDA(c, cudaMemcpyAsync(lo, static_cast<const char*>(g->ptr[dn]) + (size_t)(c->nz_l - 1) * plane_bytes,
                                plane_bytes, cudaMemcpyDeviceToDevice, c->stream));
    FGD_CUDA(c, cudaMemcpyAsync(hi, g->ptr[up], plane_bytes, cudaMemcpyDeviceToDevice, c->stream));
    return loop_finish(c);
  }
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

extern "C" fgd_status fgd_loopback_id(unsigned char* out) {
  if (!out) return FGD_EINVAL;
  static std::mutex m;
  static unsigned long long counter = 0;
  std::memset(out, 0, 128);
  std::memcpy(out, fgd::kLoopMagic, 8);
  unsigned long long k[3];
  {
    std::lock_guard<std::mutex> lk(m);
    k[0] = ++counter;
  }
  k[1] = (unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count();
  k[2] = (unsigned long long)(uintptr_t)&counter;
  std::memcpy(out + 8, k, 24);
  return FGD_OK;
}

extern "C" fgd_status fgd_nccl_id(unsigned char* out) {
  if (!out) return FGD_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FGD_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return FGD_OK;
}
