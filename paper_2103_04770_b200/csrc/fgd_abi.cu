// libfgd C ABI (include/fgd.h): context, data setting, operator applies, Krylov solvers,
// Newton and the Algorithm 1 staggered increment.  Host orchestration only: every step of the
// hot path runs in the kernels of passes.cu / helmholtz.cu / constitutive.cu; the Krylov
// scalars live on the device and the host reads one or two doubles per iteration to decide
// convergence.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>

#include "fgd_internal.cuh"

namespace fgd {

fgd_status set_err(fgd_ctx* c, fgd_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

static int next_event(fgd_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    c->ev_pool.push_back(e);
  }
  return (int)c->ev_used++;
}

KTimer::KTimer(fgd_ctx* cc, int k) : c(cc), cls(k) {
  if (!c->timing) return;
  e0 = next_event(c);
  if (e0 >= 0) cudaEventRecord(c->ev_pool[e0], c->stream);
}

KTimer::~KTimer() {
  if (e0 < 0) return;
  const int e1 = next_event(c);
  if (e1 < 0) return;
  cudaEventRecord(c->ev_pool[e1], c->stream);
  c->ev_rec.push_back({cls, {e0, e1}});
}

static bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

template <typename T>
static fgd_status dalloc(fgd_ctx* c, T** p, size_t count) {
  if (*p) return FGD_OK;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T) + 16);
  if (e != cudaSuccess) {
    *p = nullptr;
    cudaGetLastError();
    return set_err(c, FGD_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return FGD_OK;
}

fgd_status ensure_spectral(fgd_ctx* c) {
  const size_t nc = (size_t)c->spec_comps;
  fgd_status s = dalloc(c, &c->specA, nc * c->nspecA);
  if (s != FGD_OK) return s;
  if (c->P > 1) {
    s = dalloc(c, &c->specC, nc * c->nspec);
    if (s != FGD_OK) return s;
  }
  return dalloc(c, &c->specB, nc * c->nspec);
}

fgd_status ensure_partials(fgd_ctx* c, size_t nblocks) {
  const size_t need = nblocks * 16;
  if (need <= c->partials_cap) return FGD_OK;
  if (c->partials) {
    cudaStreamSynchronize(c->stream);
    cudaFree(c->partials);
    c->partials = nullptr;
  }
  fgd_status s = dalloc(c, &c->partials, need);
  if (s != FGD_OK) return s;
  c->partials_cap = need;
  return FGD_OK;
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Host/device argument staging.  in(): returns a device pointer holding `count` doubles of p.
struct Stage {
  fgd_ctx* c;
  std::vector<void*> bufs;
  explicit Stage(fgd_ctx* cc) : c(cc) {}
  ~Stage() {
    for (void* b : bufs) cudaFreeAsync(b, c->stream);
  }
  template <typename T>
  fgd_status in(const T* p, size_t count, const T** out) {
    if (!p || is_device_ptr(p)) {
      *out = p;
      return FGD_OK;
    }
    void* d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, count * sizeof(T) + 16, c->stream);
    if (e != cudaSuccess) return set_err(c, FGD_ENOMEM, std::string("staging: ") + cudaGetErrorString(e));
    bufs.push_back(d);
    e = h2d(d, p, count * sizeof(T));
    if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("H2D: ") + cudaGetErrorString(e));
    *out = (const T*)d;
    return FGD_OK;
  }
  // Large host->device copies are split in two halves on two streams (the context stream and an
  // auxiliary one ordered by events), so that two copy engines share the PCIe link.
  cudaError_t h2d(void* d, const void* p, size_t bytes) {
    if (bytes < ((size_t)64 << 20)) return cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, c->stream);
    cudaError_t e = cudaSuccess;
    if (!c->aux) {
      e = cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->aux_ev[0], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->aux_ev[1], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    const size_t h = (bytes / 2 + 255) & ~(size_t)255;
    if ((e = cudaEventRecord(c->aux_ev[0], c->stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(c->aux, c->aux_ev[0], 0)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync((char*)d + h, (const char*)p + h, bytes - h, cudaMemcpyHostToDevice, c->aux)) != cudaSuccess)
      return e;
    if ((e = cudaEventRecord(c->aux_ev[1], c->aux)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(d, p, h, cudaMemcpyHostToDevice, c->stream)) != cudaSuccess) return e;
    return cudaStreamWaitEvent(c->stream, c->aux_ev[1], 0);
  }
  // out(): device destination for a result that must end in p (copied back by finish()).
  struct Pending {
    void* host;
    const void* dev;
    size_t bytes;
  };
  std::vector<Pending> pend;
  template <typename T>
  fgd_status out(T* p, size_t count, T** dst) {
    if (!p || is_device_ptr(p)) {
      *dst = p;
      return FGD_OK;
    }
    void* d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, count * sizeof(T) + 16, c->stream);
    if (e != cudaSuccess) return set_err(c, FGD_ENOMEM, std::string("staging: ") + cudaGetErrorString(e));
    bufs.push_back(d);
    pend.push_back({(void*)p, d, count * sizeof(T)});
    *dst = (T*)d;
    return FGD_OK;
  }
  fgd_status finish() {
    for (auto& q : pend) {
      cudaError_t e = cudaMemcpyAsync(q.host, q.dev, q.bytes, cudaMemcpyDeviceToHost, c->stream);
      if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("D2H: ") + cudaGetErrorString(e));
    }
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return set_err(c, FGD_ECUDA, std::string("sync: ") + cudaGetErrorString(e));
    return FGD_OK;
  }
};

static fgd_status sync_read(fgd_ctx* c, const void* dev, size_t bytes, void* host) {
  FGD_CUDA(c, cudaMemcpyAsync(c->pinned, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
  FGD_CUDA(c, cudaStreamSynchronize(c->stream));
  std::memcpy(host, c->pinned, bytes);
  return FGD_OK;
}

#define TRY(x)                         \
  do {                                 \
    fgd_status s_ = (x);               \
    if (s_ != FGD_OK) return s_;       \
  } while (0)

// twiddle tables e^{-2 pi i m/N} for N = 1..512 (long double, exact at quarter turns)
static fgd_status build_tables(fgd_ctx* c) {
  std::vector<double2> h;
  size_t off[11];
  for (int l = 0; l <= 9; ++l) {
    const int N = 1 << l;
    off[l] = h.size();
    for (int m = 0; m < N; ++m) {
      double re, im;
      if ((4 * m) % N == 0) {
        const int qd = (4 * m / N) % 4;
        const double cs[4] = {1, 0, -1, 0}, sn[4] = {0, 1, 0, -1};
        re = cs[qd];
        im = -sn[qd];
      } else {
        const long double ang = 2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)N;
        re = (double)cosl(ang);
        im = (double)(-sinl(ang));
      }
      h.push_back(make_double2(re, im));
    }
  }
  TRY(dalloc(c, &c->tw_all, h.size()));
  FGD_CUDA(c, cudaMemcpy(c->tw_all, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  for (int l = 0; l <= 9; ++l) c->tabs.tw[l] = c->tw_all + off[l];
  c->tabs.tw[10] = nullptr;
  return FGD_OK;
}

static double inv_nvox(const fgd_ctx* c) { return 1.0 / (double)c->nvox_g; }

// a reducing launch: (op, slot) as the kernel must see them, then the distributed finalisation
#define RED(op) red_op_for(c, op), red_slot_for(c, op, 0)
#define RED_S(op, slot) red_op_for(c, op), red_slot_for(c, op, slot)

// ---- composite operators (all enqueued on c->stream) -----------------------------------------
// y = G*(C : x)
static fgd_status op_projected_tangent(fgd_ctx* c, const double* x, double* y) {
  TRY(ensure_spectral(c));
  TRY(launch_xfwd(c, 6, XF_TANGENT, x, nullptr, nullptr, c->compact ? c->Cc : c->C, RED_NONE, 0));
  TRY(yz_round_trip(c, 6, Z_PROJECT, inv_nvox(c), nullptr, 0.0));
  return launch_xinv(c, 6, XI_STORE, y, nullptr, nullptr, nullptr, RED_NONE, 0);
}

// y = scale * G*(tau - S); optional reduction of y.y into op/slot
static fgd_status op_projection(fgd_ctx* c, const double* tau, const double* S, double scale, double* y, int red_op,
                                int red_slot) {
  TRY(ensure_spectral(c));
  double shift[6] = {0, 0, 0, 0, 0, 0};
  if (S)
    for (int i = 0; i < 6; ++i) shift[i] = S[i] * (double)c->nvox_g;
  TRY(launch_xfwd(c, 6, XF_PLAIN, tau, nullptr, nullptr, nullptr, RED_NONE, 0));
  TRY(yz_round_trip(c, 6, Z_PROJECT, scale * inv_nvox(c), shift, 0.0));
  if (red_op == RED_NONE) return launch_xinv(c, 6, XI_STORE, y, nullptr, nullptr, nullptr, RED_NONE, 0);
  TRY(launch_xinv(c, 6, XI_STORE_RR, y, nullptr, nullptr, nullptr, red_op_for(c, red_op), red_slot_for(c, red_op, red_slot)));
  if (red_op == RED_STORE) return allreduce_sum(c, &c->sc->red[red_slot], 1);
  return post_reduce(c, red_op);
}

// z = F^-1 M F r ; if r_for_dot != null: reduce r.z with red_op
static fgd_status op_precond(fgd_ctx* c, int field, const double* r, double* z, int red_op) {
  TRY(ensure_spectral(c));
  TRY(launch_xfwd(c, 1, XF_PLAIN, r, nullptr, nullptr, nullptr, RED_NONE, 0));
  TRY(launch_precond_yz(c, inv_nvox(c), mean_ell2(c, field)));
  if (red_op == RED_NONE) return launch_xinv(c, 1, XI_STORE, z, nullptr, nullptr, nullptr, RED_NONE, 0);
  TRY(launch_xinv(c, 1, XI_HELM_Z, z, nullptr, nullptr, r, RED(red_op)));
  return post_reduce(c, red_op);
}

static fgd_status ensure_helm(fgd_ctx* c) {
  for (int i = 0; i < 6; ++i) TRY(dalloc(c, &c->hb[i], c->nvox));
  return FGD_OK;
}
static fgd_status ensure_cg(fgd_ctx* c) {
  TRY(dalloc(c, &c->cg_x, 6 * c->nvox));
  TRY(dalloc(c, &c->cg_r, 6 * c->nvox));
  return dalloc(c, &c->cg_p, 6 * c->nvox);
}
static fgd_status ensure_state(fgd_ctx* c) {
  const size_t n = c->nvox;
  const size_t J = std::max(1, c->nfields);
  if (c->st_eps) return FGD_OK;
  TRY(dalloc(c, &c->st_eps, 6 * n));
  TRY(dalloc(c, &c->st_epsp, 6 * n));
  TRY(dalloc(c, &c->st_ep, n));
  TRY(dalloc(c, &c->st_hist, n));
  TRY(dalloc(c, &c->st_abar, J * n));
  TRY(dalloc(c, &c->w_eps, 6 * n));
  TRY(dalloc(c, &c->w_eps_prev, 6 * n));
  TRY(dalloc(c, &c->w_sig, 6 * n));
  TRY(dalloc(c, &c->w_alpha, J * n));
  TRY(dalloc(c, &c->w_abar, J * n));
  TRY(dalloc(c, &c->w_D, J * n));
  TRY(dalloc(c, &c->cm_epsp, 6 * n));
  TRY(dalloc(c, &c->cm_ep, n));
  TRY(dalloc(c, &c->cm_hist, n));
  TRY(dalloc(c, &c->w_b, 6 * n));
  TRY(dalloc(c, &c->w_de, 6 * n));
  TRY(dalloc(c, &c->Cc, 9 * n));
  FGD_CUDA(c, cudaMemsetAsync(c->st_eps, 0, 6 * n * 8, c->stream));
  FGD_CUDA(c, cudaMemsetAsync(c->st_epsp, 0, 6 * n * 8, c->stream));
  FGD_CUDA(c, cudaMemsetAsync(c->st_ep, 0, n * 8, c->stream));
  FGD_CUDA(c, cudaMemsetAsync(c->st_hist, 0, n * 8, c->stream));
  FGD_CUDA(c, cudaMemsetAsync(c->st_abar, 0, J * n * 8, c->stream));
  FGD_CUDA(c, cudaMemsetAsync(c->w_abar, 0, J * n * 8, c->stream));
  FGD_CUDA(c, cudaMemcpyAsync(c->w_eps, c->st_eps, 6 * n * 8, cudaMemcpyDeviceToDevice, c->stream));
  return FGD_OK;
}

// Algorithm 2 in real space (equivalent to the Fourier-space PCG: F is unitary up to N).
// Krylov loops with tol > 0 on one GPU launch iterations in growing batches (4, 8, .. 32) and
// read the device convergence flag once per batch; the hot kernels skip themselves once the
// finalise of the monitored norm has set it (guard_done), so the returned iterate and iteration
// count are those of the converged iteration.  With nranks > 1 the same holds on every rank (the
// flag is finalised from allreduced sums, identical on all ranks, so all ranks take the same
// host decisions); batches stop at 8 there, because the collectives of skipped iterations still
// move their (unused) bytes.
struct GuardScope {
  fgd_ctx* c;
  GuardScope(fgd_ctx* cc, bool on) : c(cc) { c->guard = on; }
  ~GuardScope() { c->guard = false; }
};

// Launch-bound small grids: a block of `reps` standard Krylov iterations is captured once per solve
// into a CUDA graph (on a private capture stream) and replayed on the context stream, one graph
// launch per block instead of ~8 kernel launches per iteration.  Used on one GPU for grids of at
// most 2^21 voxels and with per-launch timing off; the captured pointers are context buffers.
struct KGraph {
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;   // kernels per replay (launch accounting)
  ~KGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

static bool use_graphs(const fgd_ctx* c) {
  static const bool off = std::getenv("FGD_NO_GRAPHS") != nullptr;
  return !off && c->nranks == 1 && !c->timing && c->nvox <= ((size_t)1 << 21);
}

// Captures `reps` calls of body(); on any failure the capture is dropped (g->exec stays null, the
// CUDA error state is cleared) and the caller keeps launching kernels directly.
template <typename F>
static void capture_graph(fgd_ctx* c, int reps, F body, KGraph* g) {
  if (!c->cap && cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess) {
    (void)cudaGetLastError();
    c->cap = nullptr;
    return;
  }
  cudaStream_t saved = c->stream;
  const long long l0 = c->launches;
  const std::string err0 = c->err;
  c->stream = c->cap;
  cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
  fgd_status st = FGD_OK;
  for (int k = 0; k < reps && st == FGD_OK && e == cudaSuccess; ++k) st = body();
  cudaGraph_t graph = nullptr;
  if (e == cudaSuccess) e = cudaStreamEndCapture(c->stream, &graph);
  c->stream = saved;
  g->launches = c->launches - l0;
  c->launches = l0;
  if (st == FGD_OK && e == cudaSuccess && graph) e = cudaGraphInstantiate(&g->exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (st != FGD_OK || e != cudaSuccess) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    g->exec = nullptr;
    (void)cudaGetLastError();
    c->err = err0;
  }
}

static fgd_status replay_graph(fgd_ctx* c, const KGraph& g) {
  c->launches += g.launches;
  FGD_CUDA(c, cudaGraphLaunch(g.exec, c->stream));
  return FGD_OK;
}

// x0 (may be null = 0): initial guess (warm start).  The stopping test stays relative to
// ||b|| (Algorithm 2); an initial residual already below it returns x0 after 0 iterations.
static fgd_status pcg_helmholtz(fgd_ctx* c, int field, const double* b, double* x_out, double tol, int maxit,
                                int* iters, double* relres, const double* x0 = nullptr) {
  TRY(ensure_helm(c));
  TRY(ensure_spectral(c));
  const size_t n = c->nvox;
  double* x = c->hb[0];
  double* r = c->hb[1];
  double* z = c->hb[2];
  double* P[2] = {c->hb[3], c->hb[4]};
  double* q = c->hb[5];
  FGD_CUDA(c, cudaMemsetAsync(P[0], 0, n * 8, c->stream));
  if (x0) {
    // x = x0, r = b - L x0 (the stencil writes L x0 into q)
    if (x0 != x) FGD_CUDA(c, cudaMemcpyAsync(x, x0, n * 8, cudaMemcpyDeviceToDevice, c->stream));
    TRY(launch_stencil(c, field, 0, x, nullptr, nullptr, nullptr, q, RED_NONE));
    FGD_CUDA(c, cudaMemcpyAsync(r, b, n * 8, cudaMemcpyDeviceToDevice, c->stream));
    TRY(launch_axpy(c, n, r, q, -1.0));
  } else {
    FGD_CUDA(c, cudaMemsetAsync(x, 0, n * 8, c->stream));
    FGD_CUDA(c, cudaMemcpyAsync(r, b, n * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  const bool batched = tol > 0.0;
  const int max_batch = c->nranks > 1 ? 8 : 32;
  TRY(launch_guard_init(c, tol > 0.0 ? tol * tol : 0.0));
  TRY(launch_dot(c, n, b, b, RED(RED_BB)));
  TRY(post_reduce(c, RED_BB));
  double bb = 0.0;
  TRY(sync_read(c, &c->sc->bb, 8, &bb));
  int it = 0;
  double rel = 0.0;
  bool start = bb > 0.0;
  if (start && x0) {
    TRY(launch_dot(c, n, r, r, RED_S(RED_STORE, 9)));
    TRY(allreduce_sum(c, &c->sc->red[9], 1));
    double rr0 = 0.0;
    TRY(sync_read(c, &c->sc->red[9], 8, &rr0));
    rel = std::sqrt(rr0 / bb);
    if (tol > 0.0 && rel < tol) start = false;   // the guess already solves the system
  }
  if (start) {
    TRY(op_precond(c, field, r, z, RED_HELM_INIT));
    int cur = 0;
    rel = 1.0;
    GuardScope gs(c, batched);
    int launched = 0, batch = 4;
    bool done = false;
    // batched mode: one PCG iteration (stencil, update, preconditioner, inverse pass); P[] alternates,
    // so a captured block has an even number of iterations
    auto iteration = [&]() -> fgd_status {
      TRY(launch_stencil(c, field, 1, nullptr, z, P[cur], P[cur ^ 1], q, RED_HELM_PQ));
      TRY(post_reduce(c, RED_HELM_PQ));
      cur ^= 1;
      TRY(launch_xfwd_io(c, 1, XF_HELM_UPDATE, P[cur], q, x, r, nullptr, RED(RED_HELM_RN)));
      TRY(post_reduce(c, RED_HELM_RN));
      TRY(launch_precond_yz(c, inv_nvox(c), mean_ell2(c, field)));
      TRY(launch_xinv(c, 1, XI_HELM_Z, z, nullptr, nullptr, r, RED(RED_HELM_RZ)));
      TRY(post_reduce(c, RED_HELM_RZ));
      return FGD_OK;
    };
    constexpr int kG = 4;
    KGraph graph;
    int gcur = 0;
    const bool graphs = batched && use_graphs(c) && maxit > 2 * kG;
    while (batched && launched < maxit && !done) {
      const int nb = std::min(batch, maxit - launched);
      int k = 0;
      if (graphs && !graph.exec && nb >= kG) {
        gcur = cur;
        capture_graph(c, kG, iteration, &graph);
        cur = gcur;   // the capture only recorded the launches
      }
      for (; graph.exec && cur == gcur && k + kG <= nb; k += kG, launched += kG) TRY(replay_graph(c, graph));
      for (; k < nb; ++k, ++launched) TRY(iteration());
      int flags[2];   // done, iters
      TRY(sync_read(c, &c->sc->done, sizeof(flags), flags));
      done = flags[0] != 0;
      batch = std::min(2 * batch, max_batch);
    }
    while (!batched && launched < maxit && !done) {
      const int nb = 1;
      for (int k = 0; k < nb; ++k, ++launched) {
        TRY(launch_stencil(c, field, 1, nullptr, z, P[cur], P[cur ^ 1], q, RED_HELM_PQ));
        TRY(post_reduce(c, RED_HELM_PQ));
        cur ^= 1;
        TRY(launch_xfwd_io(c, 1, XF_HELM_UPDATE, P[cur], q, x, r, nullptr, RED(RED_HELM_RN)));
        TRY(post_reduce(c, RED_HELM_RN));
        if (!batched && tol > 0.0) {
          double rn2;
          TRY(sync_read(c, &c->sc->rn2, 8, &rn2));
          if (std::sqrt(rn2 / bb) < tol) {
            done = true;
            ++launched;
            break;
          }
        }
        TRY(launch_precond_yz(c, inv_nvox(c), mean_ell2(c, field)));
        TRY(launch_xinv(c, 1, XI_HELM_Z, z, nullptr, nullptr, r, RED(RED_HELM_RZ)));
        TRY(post_reduce(c, RED_HELM_RZ));
      }
      if (batched) {
        int flags[2];   // done, iters
        TRY(sync_read(c, &c->sc->done, sizeof(flags), flags));
        done = flags[0] != 0;
        batch = std::min(2 * batch, max_batch);
      }
    }
    if (batched) {
      int flags[2];
      TRY(sync_read(c, &c->sc->done, sizeof(flags), flags));
      it = flags[1];
    } else {
      it = launched;
    }
    double rn2;
    TRY(sync_read(c, &c->sc->rn2, 8, &rn2));
    rel = std::sqrt(rn2 / bb);
  }
  if (x_out) FGD_CUDA(c, cudaMemcpyAsync(x_out, x, n * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (iters) *iters = it;
  if (relres) *relres = rel;
  if (tol > 0.0 && bb > 0.0 && rel >= tol) return set_err(c, FGD_ENOCONV, "Helmholtz PCG did not converge");
  return FGD_OK;
}

// Mechanical CG on G*(C : de) = b, de_0 = 0.  p.q = p.Cp for p in range(G*).
static fgd_status cg_mech(fgd_ctx* c, const double* b, double* x_out, double tol, int maxit, int* iters,
                          double* relres) {
  TRY(ensure_cg(c));
  TRY(ensure_spectral(c));
  const size_t n6 = 6 * c->nvox;
  // r_0 = b is never copied: the first tangent pass reads b as r (p_1 = b, x_1 = 0, no memsets)
  // and the first inverse pass writes r_1 = b - alpha q into cg_r.
  if (((uintptr_t)b & 15) != 0) {
    FGD_CUDA(c, cudaMemcpyAsync(c->cg_r, b, n6 * 8, cudaMemcpyDeviceToDevice, c->stream));
    b = c->cg_r;
  }
  const bool batched = tol > 0.0;
  const int max_batch = c->nranks > 1 ? 8 : 32;
  TRY(launch_guard_init(c, tol > 0.0 ? tol * tol : 0.0));
  TRY(launch_dot(c, n6, b, b, RED(RED_MECH_INIT)));
  TRY(post_reduce(c, RED_MECH_INIT));
  double bb = 0.0;
  TRY(sync_read(c, &c->sc->bb, 8, &bb));
  int it = 0;
  double rel = 0.0;
  if (bb > 0.0) {
    rel = 1.0;
    GuardScope gs(c, batched);
    int launched = 0, batch = 4;
    bool done = false;
    auto iteration = [&](bool first) -> fgd_status {
      TRY(launch_xfwd_io(c, 6, XF_TANGENT_CG, first ? b : c->cg_r, nullptr, c->cg_p, c->cg_x,
                         c->compact ? c->Cc : c->C, RED(RED_MECH_PQ), first ? 1 : 0));
      TRY(yz_round_trip(c, 6, Z_PROJECT, inv_nvox(c), nullptr, 0.0));
      TRY(post_reduce(c, RED_MECH_PQ));
      TRY(launch_xinv(c, 6, XI_MECH_CG, nullptr, nullptr, c->cg_r, first ? b : c->cg_r, RED(RED_MECH_RR)));
      TRY(post_reduce(c, RED_MECH_RR));
      return FGD_OK;
    };
    constexpr int kG = 4;   // iterations per graph replay
    KGraph graph;
    const bool graphs = batched && use_graphs(c) && maxit > 2 * kG;
    while (launched < maxit && !done) {
      const int nb = batched ? std::min(batch, maxit - launched) : 1;
      int k = 0;
      if (launched == 0) {
        TRY(iteration(true));
        ++k;
        ++launched;
      }
      if (graphs && !graph.exec && nb - k >= kG) capture_graph(c, kG, [&]() { return iteration(false); }, &graph);
      for (; graph.exec && k + kG <= nb; k += kG, launched += kG) TRY(replay_graph(c, graph));
      for (; k < nb; ++k, ++launched) TRY(iteration(false));
      if (batched) {
        int flags[2];   // done, iters
        TRY(sync_read(c, &c->sc->done, sizeof(flags), flags));
        done = flags[0] != 0;
        batch = std::min(2 * batch, max_batch);
      } else if (tol > 0.0) {
        double rr;
        TRY(sync_read(c, &c->sc->rr, 8, &rr));
        done = std::sqrt(rr / bb) < tol;
      }
    }
    if (batched) {
      int flags[2];
      TRY(sync_read(c, &c->sc->done, sizeof(flags), flags));
      it = flags[1];
    } else {
      it = launched;
    }
    double rr;
    TRY(sync_read(c, &c->sc->rr, 8, &rr));
    rel = std::sqrt(rr / bb);
    if (it > 0) TRY(launch_axpy_alpha(c, n6, c->cg_x, c->cg_p));   // x += alpha_last p_last
  }
  if (it == 0) FGD_CUDA(c, cudaMemsetAsync(c->cg_x, 0, n6 * 8, c->stream));   // b = 0 or maxit = 0
  if (x_out) FGD_CUDA(c, cudaMemcpyAsync(x_out, c->cg_x, n6 * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (iters) *iters = it;
  if (relres) *relres = rel;
  if (tol > 0.0 && bb > 0.0 && rel >= tol) return set_err(c, FGD_ENOCONV, "mechanical CG did not converge");
  return FGD_OK;
}

static fgd_status check_ready(fgd_ctx* c, bool need_phase, bool need_nonlocal, bool need_mat) {
  if (!c) return FGD_EINVAL;
  if (need_phase && !c->phase) return set_err(c, FGD_ESTATE, "fgd_set_phases has not been called");
  if (need_nonlocal && !c->nonlocal_set) return set_err(c, FGD_ESTATE, "fgd_set_nonlocal has not been called");
  if (need_mat) {
    for (int q = 0; q < c->nphases; ++q)
      if (!c->mat_set[q]) return set_err(c, FGD_ESTATE, "material of phase " + std::to_string(q) + " not set");
  }
  return FGD_OK;
}

}  // namespace fgd

using namespace fgd;

extern "C" {

fgd_status fgd_create(const fgd_grid* g, const fgd_dist* d, fgd_ctx** out) {
  if (!g || !out) return FGD_EINVAL;
  *out = nullptr;
  fgd_ctx* c = new fgd_ctx();
  auto fail = [&](fgd_status s, const std::string& m) {
    fprintf(stderr, "fgd_create: %s\n", m.c_str());
    fgd_destroy(c);
    return s;
  };
  if (g->dims != 2 && g->dims != 3) return fail(FGD_EINVAL, "dims must be 2 or 3");
  for (int i = 0; i < 3; ++i) {
    c->n[i] = g->n[i];
    c->L[i] = g->L[i];
  }
  if (g->dims == 2) c->n[2] = 1;
  for (int i = 0; i < 2; ++i)
    if (!is_pow2(c->n[i]) || c->n[i] < 4 || c->n[i] > kMaxN) return fail(FGD_EINVAL, "N1, N2 must be powers of two in [4, 512]");
  if (!is_pow2(c->n[2]) || c->n[2] > kMaxN) return fail(FGD_EINVAL, "N3 must be 1 or a power of two <= 512");
  if (c->n[2] == 1 && g->dims == 3) return fail(FGD_EINVAL, "dims = 3 needs N3 >= 2");
  for (int i = 0; i < 3; ++i) {
    if (!(c->L[i] > 0.0)) {
      if (i == 2 && c->n[2] == 1) c->L[2] = c->L[0] / c->n[0];
      else return fail(FGD_EINVAL, "L_i must be > 0");
    }
    c->h[i] = c->L[i] / c->n[i];
  }
  if (g->scheme != 0 && g->scheme != 1) return fail(FGD_EINVAL, "scheme must be 0 or 1");
  c->scheme = g->scheme;
  c->dims = g->dims;
  c->Hx = c->n[0] / 2 + 1;
  if (d) {
    c->device = d->device;
    c->stream = (cudaStream_t)d->stream;
  }
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(FGD_ECUDA, "cudaSetDevice failed");
  if (dist_init(c, d) != FGD_OK) return fail(FGD_EINVAL, c->err);
  c->nvox_g = (size_t)c->n[0] * c->n[1] * c->n[2];
  c->nvox = (size_t)c->n[0] * c->n[1] * c->nz_l;
  c->nspec = (size_t)c->Hx * c->n[1] * c->nz_l;
  c->HxA = (c->Hx + 3) & ~3;
  c->nspecA = (size_t)c->HxA * c->n[1] * c->nz_l;
  // stream == NULL is the legacy default stream (it orders against every other blocking stream,
  // e.g. PyTorch's default stream, so inputs produced there are complete before our kernels run)
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (build_tables(c) != FGD_OK) return fail(FGD_ECUDA, c->err);
  if (dalloc(c, &c->sc, 1) != FGD_OK) return fail(FGD_ENOMEM, c->err);
  if (cudaMemset(c->sc, 0, sizeof(DevScalars)) != cudaSuccess) return fail(FGD_ECUDA, "memset");
  if (cudaMallocHost((void**)&c->pinned, 4096) != cudaSuccess) return fail(FGD_ENOMEM, "cudaMallocHost");
  if (ensure_partials(c, 148 * 64) != FGD_OK) return fail(FGD_ENOMEM, c->err);
  *out = c;
  return FGD_OK;
}

void fgd_destroy(fgd_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  void* bufs[] = {c->tw_all, c->phase, c->C, c->Cc, c->specA, c->specB, c->cg_x, c->cg_r, c->cg_p, c->sc, c->partials,
                  c->st_eps, c->st_epsp, c->st_ep, c->st_hist, c->st_abar, c->w_eps, c->w_eps_prev, c->w_sig,
                  c->w_alpha, c->w_abar, c->w_D, c->cm_epsp, c->cm_ep, c->cm_hist, c->w_b, c->w_de};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (int i = 0; i < 6; ++i)
    if (c->hb[i]) cudaFree(c->hb[i]);
  if (c->hg) cudaFree(c->hg);
  for (fgd_helm_sub& h : c->hsub) {
    if (h.stream) cudaStreamSynchronize(h.stream);
    void* hbufs[] = {h.hb[0], h.hb[1], h.hb[2], h.hb[3], h.hb[4], h.hb[5], h.specA, h.specB, h.specC, h.sc, h.partials};
    for (void* b : hbufs)
      if (b) cudaFree(b);
    if (h.pinned) cudaFreeHost(h.pinned);
    if (h.ev) cudaEventDestroy(h.ev);
    if (h.cap) cudaStreamDestroy(h.cap);
    if (h.stream) cudaStreamDestroy(h.stream);
  }
  if (c->hsub_ev) cudaEventDestroy(c->hsub_ev);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->cap) cudaStreamDestroy(c->cap);
  for (cudaEvent_t e : c->aux_ev)
    if (e) cudaEventDestroy(e);
  dist_destroy(c);
  if (c->specC) cudaFree(c->specC);
  if (c->halo) cudaFree(c->halo);
  if (c->phase_halo) cudaFree(c->phase_halo);
  delete c;
}

const char* fgd_last_error(const fgd_ctx* c) { return c ? c->err.c_str() : "null context"; }

fgd_status fgd_local_extent(const fgd_ctx* c, int* z0, int* nz) {
  if (!c) return FGD_EINVAL;
  if (z0) *z0 = c->z0;
  if (nz) *nz = c->nz_l;
  return FGD_OK;
}

unsigned long long fgd_launch_count(const fgd_ctx* c) { return c ? c->launches : 0ull; }

fgd_status fgd_set_phases(fgd_ctx* c, const uint8_t* phase, int nphases) {
  if (!c || !phase) return set_err(c, FGD_EINVAL, "null argument");
  if (nphases < 1 || nphases > kMaxPhases) return set_err(c, FGD_EINVAL, "nphases must be in [1, 16]");
  TRY(dalloc(c, &c->phase, c->nvox));
  if (is_device_ptr(phase))
    FGD_CUDA(c, cudaMemcpyAsync(c->phase, phase, c->nvox, cudaMemcpyDeviceToDevice, c->stream));
  else
    FGD_CUDA(c, cudaMemcpyAsync(c->phase, phase, c->nvox, cudaMemcpyHostToDevice, c->stream));
  unsigned long long* cnt = nullptr;
  int* bad = nullptr;
  FGD_CUDA(c, cudaMallocAsync((void**)&cnt, 8 * kMaxPhases + 16, c->stream));
  FGD_CUDA(c, cudaMemsetAsync(cnt, 0, 8 * kMaxPhases + 16, c->stream));
  bad = (int*)(cnt + kMaxPhases);
  TRY(launch_phase_count(c, c->phase, cnt, nphases, bad));
  unsigned long long h[kMaxPhases + 2];
  FGD_CUDA(c, cudaMemcpyAsync(h, cnt, 8 * kMaxPhases + 16, cudaMemcpyDeviceToHost, c->stream));
  FGD_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFreeAsync(cnt, c->stream);
  if (*(int*)(h + kMaxPhases)) return set_err(c, FGD_EINVAL, "phase id >= nphases");
  c->nphases = nphases;
  c->phase_count.assign(h, h + nphases);
  if (c->nranks > 1) {
    // global phase counts (for <l^2>) and the one-plane phase halo of the Helmholtz stencil
    for (int q = 0; q < nphases; ++q) c->pinned[256 + q] = (double)h[q];
    FGD_CUDA(c, cudaMemcpyAsync(&c->sc->red[0], c->pinned + 256, 8 * nphases, cudaMemcpyHostToDevice, c->stream));
    TRY(allreduce_sum(c, &c->sc->red[0], nphases));
    double tot[kMaxPhases];
    TRY(sync_read(c, &c->sc->red[0], 8 * nphases, tot));
    for (int q = 0; q < nphases; ++q) c->phase_count[q] = (long long)(tot[q] + 0.5);
    const size_t plane = (size_t)c->n[0] * c->n[1];
    TRY(dalloc(c, &c->phase_halo, 2 * plane));
    TRY(halo_exchange(c, c->phase, plane, c->phase_halo, c->phase_halo + plane));
    FGD_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  return FGD_OK;
}

fgd_status fgd_set_material(fgd_ctx* c, int phase, const fgd_material* m) {
  if (!c || !m) return set_err(c, FGD_EINVAL, "null argument");
  if (phase < 0 || phase >= kMaxPhases) return set_err(c, FGD_EINVAL, "phase out of range");
  if (m->model < 0 || m->model > 3) return set_err(c, FGD_EINVAL, "unknown material model");
  if (!(m->E > 0.0) || !(m->nu > -1.0 && m->nu < 0.5)) return set_err(c, FGD_EINVAL, "E > 0 and -1 < nu < 0.5 required");
  if (m->model == 1 && !(m->eps_r > m->eps_c)) return set_err(c, FGD_EINVAL, "eps_r must exceed eps_c");
  if (m->model == 2 && !(m->kappa_f > m->kappa0)) return set_err(c, FGD_EINVAL, "kappa_f must exceed kappa0");
  if (m->model == 3) {
    const bool ok = m->sigma_y > 0.0 && m->q1 > 0.0 && m->q3 > 0.0 && m->q1 * m->q1 >= m->q3 && m->f_c > 0.0 &&
                    m->f_f > m->f_c && m->s_n > 0.0 && m->n_hard > 0.0 && m->n_hard < 1.0 && m->fstar_max > 0.0 &&
                    m->fstar_max < (m->q1 + std::sqrt(m->q1 * m->q1 - m->q3)) / m->q3;
    if (!ok)
      return set_err(c, FGD_EINVAL,
                     "GTN needs sigma_y, q1, q3, s_n > 0, q1^2 >= q3, 0 < f_c < f_f, 0 < n_hard < 1, "
                     "0 < fstar_max < f_V*");
  }
  c->mat[phase] = Material{m->model, m->E, m->nu, m->sigma_y, m->H, m->eps_c, m->eps_r, m->d_max, m->kappa0,
                           m->kappa_f, m->q1, m->q2, m->q3, m->f_c, m->f_f, m->f_n, m->eps_n, m->s_n, m->n_hard,
                           m->fstar_max};
  c->mat_set[phase] = true;
  return FGD_OK;
}

fgd_status fgd_set_nonlocal(fgd_ctx* c, int nfields, const double* ell, const int* source_phase) {
  if (!c) return FGD_EINVAL;
  if (!c->phase) return set_err(c, FGD_ESTATE, "fgd_set_phases must precede fgd_set_nonlocal");
  if (nfields < 0 || nfields > kMaxFields) return set_err(c, FGD_EINVAL, "nfields must be in [0, 4]");
  if (nfields > 0 && (!ell || !source_phase)) return set_err(c, FGD_EINVAL, "null argument");
  if (c->st_eps && nfields != c->nfields) return set_err(c, FGD_ESTATE, "nfields cannot change after the state exists");
  for (int j = 0; j < nfields; ++j) {
    if (source_phase[j] < 0 || source_phase[j] >= c->nphases) return set_err(c, FGD_EINVAL, "source_phase out of range");
    for (int q = 0; q < c->nphases; ++q) {
      if (!(ell[j * c->nphases + q] >= 0.0)) return set_err(c, FGD_EINVAL, "ell must be >= 0");
      c->ell[j][q] = ell[j * c->nphases + q];
    }
    c->source_phase[j] = source_phase[j];
  }
  c->nfields = nfields;
  c->nonlocal_set = true;
  return FGD_OK;
}

fgd_status fgd_set_control(fgd_ctx* c, const int* mask) {
  if (!c || !mask) return set_err(c, FGD_EINVAL, "null argument");
  for (int i = 0; i < 6; ++i) c->stress_mask[i] = mask[i] ? 1 : 0;
  c->control_set = true;
  return FGD_OK;
}

fgd_status fgd_set_tangent(fgd_ctx* c, const double* C) {
  if (!c || !C) return set_err(c, FGD_EINVAL, "null argument");
  TRY(dalloc(c, &c->C, 21 * c->nvox));
  if (is_device_ptr(C))
    FGD_CUDA(c, cudaMemcpyAsync(c->C, C, 21 * c->nvox * 8, cudaMemcpyDeviceToDevice, c->stream));
  else
    FGD_CUDA(c, cudaMemcpyAsync(c->C, C, 21 * c->nvox * 8, cudaMemcpyHostToDevice, c->stream));
  FGD_CUDA(c, cudaStreamSynchronize(c->stream));
  c->tangent_set = true;
  c->compact = 0;
  return FGD_OK;
}

fgd_status fgd_apply_projected_tangent(fgd_ctx* c, const double* x, double* y) {
  if (!c || !x || !y) return set_err(c, FGD_EINVAL, "null argument");
  if (!c->tangent_set) return set_err(c, FGD_ESTATE, "no tangent (fgd_set_tangent or fgd_constitutive)");
  Stage st(c);
  const double* dx;
  double* dy;
  TRY(st.in(x, 6 * c->nvox, &dx));
  TRY(st.out(y, 6 * c->nvox, &dy));
  TRY(op_projected_tangent(c, dx, dy));
  return st.finish();
}

fgd_status fgd_apply_projection(fgd_ctx* c, const double* tau, const double* S, double* y) {
  if (!c || !tau || !y) return set_err(c, FGD_EINVAL, "null argument");
  Stage st(c);
  const double* dt;
  double* dy;
  TRY(st.in(tau, 6 * c->nvox, &dt));
  TRY(st.out(y, 6 * c->nvox, &dy));
  TRY(op_projection(c, dt, S, 1.0, dy, RED_NONE, 0));
  return st.finish();
}

static fgd_status check_field(fgd_ctx* c, int field) {
  TRY(check_ready(c, true, true, false));
  if (field < 0 || field >= c->nfields) return set_err(c, FGD_EINVAL, "field out of range");
  return FGD_OK;
}

fgd_status fgd_apply_helmholtz(fgd_ctx* c, int field, const double* a, double* y) {
  if (!c || !a || !y) return set_err(c, FGD_EINVAL, "null argument");
  TRY(check_field(c, field));
  Stage st(c);
  const double* da;
  double* dy;
  TRY(st.in(a, c->nvox, &da));
  TRY(st.out(y, c->nvox, &dy));
  TRY(launch_stencil(c, field, 0, da, nullptr, nullptr, nullptr, dy, RED_NONE));
  return st.finish();
}

fgd_status fgd_apply_helmholtz_precond(fgd_ctx* c, int field, const double* r, double* z) {
  if (!c || !r || !z) return set_err(c, FGD_EINVAL, "null argument");
  TRY(check_ready(c, true, true, false));
  if (field < 0 || field >= c->nfields) return set_err(c, FGD_EINVAL, "field out of range");
  Stage st(c);
  const double* dr;
  double* dz;
  TRY(st.in(r, c->nvox, &dr));
  TRY(st.out(z, c->nvox, &dz));
  TRY(op_precond(c, field, dr, dz, RED_NONE));
  return st.finish();
}

// NEXT#3 -- the J Helmholtz problems of a staggered iteration are independent ("computed
// independently"): solve them SIDE BY SIDE.  Field 0 runs on the context, every field
// j >= 1 on a copy of the context that owns its stream, Krylov scalars, work vectors and
// one-component spectrum buffers (fgd_helm_sub), each driven by its own host thread (the batched
// loops read their convergence flag from the host).  Every solve executes exactly the kernels,
// grids and reduction orders of pcg_helmholtz, so the results are bitwise those of J consecutive
// solves.  On the launch-latency-bound grids (<= 2^21 voxels) the two dependent kernel chains
// overlap; on HBM-bound grids the solves stay consecutive (persistent grids already fill the GPU).
// FGD_HELM_CONC = 0 / 1 forces the choice.  One GPU only: the communicator is not shared by threads.
static bool helm_concurrent(const fgd_ctx* c, int J) {
  const char* e = std::getenv("FGD_HELM_CONC");   // read per call: tests toggle it
  if (J < 2 || c->nranks != 1 || c->timing) return false;
  if (e) return std::atoi(e) != 0;
  return c->nvox <= ((size_t)1 << 21);
}

static fgd_status helm_sub_init(fgd_ctx* c, fgd_helm_sub* h) {
  if (h->stream) return FGD_OK;
  FGD_CUDA(c, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  FGD_CUDA(c, cudaEventCreateWithFlags(&h->ev, cudaEventDisableTiming));
  TRY(dalloc(c, &h->sc, 1));
  FGD_CUDA(c, cudaMemsetAsync(h->sc, 0, sizeof(DevScalars), h->stream));
  FGD_CUDA(c, cudaMallocHost((void**)&h->pinned, 4096));
  return FGD_OK;
}

// src, x0 (may be null), out: J fields one after another on the device.  st[j], iters[j], relres[j]
// per field; returns the first hard error (anything but FGD_ENOCONV), else FGD_OK.
static fgd_status helm_solve_all(fgd_ctx* c, int J, const double* src, const double* x0, double* out, double tol,
                                 int maxit, fgd_status* st, int* iters, double* relres) {
  const size_t n = c->nvox;
  auto solve = [&](fgd_ctx* cc, int j) {
    st[j] = pcg_helmholtz(cc, j, src + (size_t)j * n, out + (size_t)j * n, tol, maxit, &iters[j], &relres[j],
                          x0 ? x0 + (size_t)j * n : nullptr);
  };
  if (!helm_concurrent(c, J)) {
    for (int j = 0; j < J; ++j) {
      solve(c, j);
      if (st[j] != FGD_OK && st[j] != FGD_ENOCONV) return st[j];
      // a failed field stops the sequence like the staggered loop always did
      if (st[j] == FGD_ENOCONV) {
        for (int k = j + 1; k < J; ++k) st[k] = FGD_ENOCONV, iters[k] = 0, relres[k] = 0.0;
        break;
      }
    }
    return FGD_OK;
  }
  TRY(ensure_helm(c));
  TRY(ensure_spectral(c));
  if ((int)c->hsub.size() < J - 1) c->hsub.resize(J - 1);
  if (!c->hsub_ev) FGD_CUDA(c, cudaEventCreateWithFlags(&c->hsub_ev, cudaEventDisableTiming));
  for (int j = 1; j < J; ++j) TRY(helm_sub_init(c, &c->hsub[j - 1]));
  FGD_CUDA(c, cudaEventRecord(c->hsub_ev, c->stream));
  std::vector<fgd_ctx> copies;
  copies.reserve(J - 1);
  for (int j = 1; j < J; ++j) {
    fgd_helm_sub& h = c->hsub[j - 1];
    FGD_CUDA(c, cudaStreamWaitEvent(h.stream, c->hsub_ev, 0));
    copies.push_back(*c);
    fgd_ctx& s = copies.back();
    s.stream = h.stream;
    s.cap = h.cap;
    s.own_stream = false;
    for (int i = 0; i < 6; ++i) s.hb[i] = h.hb[i];
    s.specA = h.specA;
    s.specB = h.specB;
    s.specC = h.specC;
    s.spec_comps = 1;
    s.sc = h.sc;
    s.partials = h.partials;
    s.partials_cap = h.partials_cap;
    s.pinned = h.pinned;
    s.hsub.clear();
    s.ev_pool.clear();
    s.ev_rec.clear();
    s.ov_ev.clear();
    s.guard = false;
    s.launches = 0;
    s.err.clear();
  }
  std::vector<std::thread> th;
  auto run = [&](int j) {
    fgd_ctx* s = &copies[j - 1];
    if (cudaSetDevice(s->device) != cudaSuccess) {
      st[j] = set_err(s, FGD_ECUDA, "cudaSetDevice failed");
      return;
    }
    solve(s, j);
    cudaEventRecord(c->hsub[j - 1].ev, s->stream);
  };
  std::vector<int> inline_fields;   // no thread available: solved on this thread after field 0
  for (int j = 1; j < J; ++j) {
    try {
      th.emplace_back(run, j);
    } catch (...) {
      inline_fields.push_back(j);
    }
  }
  solve(c, 0);
  for (int j : inline_fields) run(j);
  for (auto& t : th) t.join();
  fgd_status hard = (st[0] != FGD_OK && st[0] != FGD_ENOCONV) ? st[0] : FGD_OK;
  for (int j = 1; j < J; ++j) {
    fgd_helm_sub& h = c->hsub[j - 1];
    fgd_ctx& s = copies[j - 1];
    // keep what the copy allocated (work vectors, spectra, partial sums, capture stream)
    h.cap = s.cap;
    for (int i = 0; i < 6; ++i) h.hb[i] = s.hb[i];
    h.specA = s.specA;
    h.specB = s.specB;
    h.specC = s.specC;
    h.partials = s.partials;
    h.partials_cap = s.partials_cap;
    c->launches += s.launches;
    cudaStreamWaitEvent(c->stream, h.ev, 0);
    if (st[j] != FGD_OK && (st[j] != FGD_ENOCONV || st[0] == FGD_OK) && hard == FGD_OK) {
      c->err = s.err;
      if (st[j] != FGD_ENOCONV) hard = st[j];
    }
  }
  return hard;
}

fgd_status fgd_solve_helmholtz(fgd_ctx* c, int field, const double* src, double* abar, double tol, int maxit,
                               int* iters, double* relres) {
  if (!c) return FGD_EINVAL;
  TRY(check_field(c, field));
  if (maxit < 0) return set_err(c, FGD_EINVAL, "maxit < 0");
  Stage st(c);
  const double* ds = nullptr;
  if (src) {
    TRY(st.in(src, c->nvox, &ds));
  } else {
    if (!c->have_sigma) return set_err(c, FGD_ESTATE, "src == NULL needs a previous fgd_constitutive");
    ds = c->w_alpha + (size_t)field * c->nvox;
  }
  double* dout = nullptr;
  if (abar) {
    TRY(st.out(abar, c->nvox, &dout));
  } else {
    TRY(ensure_state(c));
    dout = c->w_abar + (size_t)field * c->nvox;
  }
  fgd_status s = pcg_helmholtz(c, field, ds, dout, tol, maxit, iters, relres);
  fgd_status f = st.finish();
  return s != FGD_OK ? s : f;
}

fgd_status fgd_solve_helmholtz_from(fgd_ctx* c, int field, const double* src, const double* x0, double* abar,
                                    double tol, int maxit, int* iters, double* relres) {
  if (!c) return FGD_EINVAL;
  TRY(check_field(c, field));
  if (maxit < 0) return set_err(c, FGD_EINVAL, "maxit < 0");
  if (!src || !abar) return set_err(c, FGD_EINVAL, "null argument");
  Stage st(c);
  const double *ds = nullptr, *dx0 = nullptr;
  TRY(st.in(src, c->nvox, &ds));
  if (x0) TRY(st.in(x0, c->nvox, &dx0));
  double* dout = nullptr;
  TRY(st.out(abar, c->nvox, &dout));
  fgd_status s = pcg_helmholtz(c, field, ds, dout, tol, maxit, iters, relres, dx0);
  fgd_status f = st.finish();
  return s != FGD_OK ? s : f;
}

fgd_status fgd_solve_helmholtz_all(fgd_ctx* c, const double* src, const double* x0, double* abar, double tol,
                                   int maxit, int* iters, double* relres) {
  if (!c) return FGD_EINVAL;
  if (!c->nonlocal_set || c->nfields < 1) return set_err(c, FGD_ESTATE, "no non-local fields set");
  if (maxit < 0) return set_err(c, FGD_EINVAL, "maxit < 0");
  if (!src || !abar) return set_err(c, FGD_EINVAL, "null argument");
  const int J = c->nfields;
  Stage st(c);
  const double *ds = nullptr, *dx0 = nullptr;
  TRY(st.in(src, (size_t)J * c->nvox, &ds));
  if (x0) TRY(st.in(x0, (size_t)J * c->nvox, &dx0));
  double* dout = nullptr;
  TRY(st.out(abar, (size_t)J * c->nvox, &dout));
  fgd_status hs[kMaxFields];
  int hit[kMaxFields] = {};
  double hrel[kMaxFields] = {};
  fgd_status s = helm_solve_all(c, J, ds, dx0, dout, tol, maxit, hs, hit, hrel);
  for (int j = 0; j < J; ++j) {
    if (iters) iters[j] = hit[j];
    if (relres) relres[j] = hrel[j];
    if (s == FGD_OK && hs[j] != FGD_OK) s = hs[j];
  }
  fgd_status f = st.finish();
  return s != FGD_OK ? s : f;
}

fgd_status fgd_solve_tangent_cg(fgd_ctx* c, const double* b, double* de, double tol, int maxit, int* iters,
                                double* relres) {
  if (!c) return FGD_EINVAL;
  if (!c->tangent_set) return set_err(c, FGD_ESTATE, "no tangent");
  if (maxit < 0) return set_err(c, FGD_EINVAL, "maxit < 0");
  Stage st(c);
  const double* db = nullptr;
  if (b) {
    TRY(st.in(b, 6 * c->nvox, &db));
  } else {
    if (!c->have_residual) return set_err(c, FGD_ESTATE, "b == NULL needs a previous fgd_mech_residual");
    db = c->w_b;
  }
  double* dx = nullptr;
  if (de) {
    TRY(st.out(de, 6 * c->nvox, &dx));
  } else {
    TRY(ensure_state(c));
    dx = c->w_de;
  }
  fgd_status s = cg_mech(c, db, dx, tol, maxit, iters, relres);
  fgd_status f = st.finish();
  return s != FGD_OK ? s : f;
}

fgd_status fgd_constitutive(fgd_ctx* c, const double* eps, double* sigma_out, double* macro) {
  if (!c) return FGD_EINVAL;
  TRY(check_ready(c, true, true, true));
  TRY(ensure_state(c));
  Stage st(c);
  const double* de = c->w_eps;
  if (eps) {
    TRY(st.in(eps, 6 * c->nvox, &de));
    if (de != c->w_eps)
      FGD_CUDA(c, cudaMemcpyAsync(c->w_eps, de, 6 * c->nvox * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  TRY(launch_constitutive(c, c->w_eps));
  const bool gtn = has_gtn(c);   // red[6]: GTN return mappings that did not converge
  TRY(allreduce_sum(c, &c->sc->red[0], gtn ? 7 : 6));
  c->tangent_set = true;
  c->compact = 1;
  c->have_sigma = true;
  if (sigma_out) {
    double* ds;
    TRY(st.out(sigma_out, 6 * c->nvox, &ds));
    FGD_CUDA(c, cudaMemcpyAsync(ds, c->w_sig, 6 * c->nvox * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  double m[7] = {0, 0, 0, 0, 0, 0, 0};
  TRY(sync_read(c, c->sc->red, gtn ? 56 : 48, m));
  for (int i = 0; i < 6; ++i) c->last_macro[i] = m[i] / (double)c->nvox_g;
  if (macro)
    for (int i = 0; i < 6; ++i) macro[i] = c->last_macro[i];
  if (m[6] > 0.0) {
    st.finish();
    return set_err(c, FGD_ENOCONV, std::to_string((long long)m[6]) + " GTN return mappings did not converge");
  }
  return st.finish();
}

fgd_status fgd_mech_residual(fgd_ctx* c, const double* S_target, double* b_out, double* rms) {
  if (!c) return FGD_EINVAL;
  if (!c->have_sigma) return set_err(c, FGD_ESTATE, "fgd_mech_residual needs a previous fgd_constitutive");
  double S[6] = {0, 0, 0, 0, 0, 0};
  if (S_target)
    for (int i = 0; i < 6; ++i) S[i] = S_target[i] * c->stress_mask[i];
  TRY(op_projection(c, c->w_sig, S, -1.0, c->w_b, RED_STORE, 8));
  c->have_residual = true;
  double ss;
  TRY(sync_read(c, &c->sc->red[8], 8, &ss));
  if (rms) *rms = std::sqrt(ss / (double)c->nvox_g);
  if (b_out) {
    Stage st(c);
    double* db;
    TRY(st.out(b_out, 6 * c->nvox, &db));
    FGD_CUDA(c, cudaMemcpyAsync(db, c->w_b, 6 * c->nvox * 8, cudaMemcpyDeviceToDevice, c->stream));
    return st.finish();
  }
  return FGD_OK;
}

// staggered-error ingredients over all ranks (sums of red[16..29], max of the strain change)
static fgd_status err_reduce(fgd_ctx* c, const double* eps, const double* eps_prev, const double* anew,
                             const double* aold) {
  FGD_CUDA(c, cudaMemsetAsync(&c->sc->maxbits, 0, 8, c->stream));
  TRY(launch_err(c, eps, eps_prev, anew, aold, &c->sc->maxbits));
  TRY(allreduce_sum(c, &c->sc->red[16], 14));
  return allreduce_max_u64(c, &c->sc->maxbits);
}

constexpr int kMaxBacktrack = 5;   // R-LS: at most 5 halvings of a Newton step

// FGD_TRACE=1: one stderr line per Newton iteration and per staggered iteration (diagnostics)
static bool trace_on() {
  static const bool on = std::getenv("FGD_TRACE") != nullptr;
  return on;
}

static double sigma_ref(const fgd_ctx* c) {
  double s = 0.0, e = 0.0;
  for (int q = 0; q < c->nphases; ++q) {
    s = std::max(s, (c->mat[q].model == 1 || c->mat[q].model == 3) ? c->mat[q].sigma_y : 0.0);
    e = std::max(e, c->mat[q].E);
  }
  return s > 0.0 ? s : e * 1e-3;
}

fgd_status fgd_solve_increment(fgd_ctx* c, const fgd_increment* inc, fgd_report* rep) {
  if (!c || !inc) return set_err(c, FGD_EINVAL, "null argument");
  TRY(check_ready(c, true, true, true));
  TRY(ensure_state(c));
  const size_t n = c->nvox;
  const double ng = (double)c->nvox_g;
  const int J = c->nfields;
  // 1. eps^(0) = eps_n + dE on strain-controlled comps; abar^(0) = abar_n  (A-22)
  double mean_n[6];
  {
    // <eps_n> : use the err kernel's sums with eps_prev = eps
    FGD_CUDA(c, cudaMemsetAsync(&c->sc->maxbits, 0, 8, c->stream));
    TRY(err_reduce(c, c->st_eps, c->st_eps, c->st_abar, c->st_abar));
    double red[6];
    TRY(sync_read(c, &c->sc->red[16], 48, red));
    for (int i = 0; i < 6; ++i) mean_n[i] = red[i] / ng;
  }
  double dE[6];
  for (int i = 0; i < 6; ++i) dE[i] = c->stress_mask[i] ? 0.0 : inc->E_target[i] - mean_n[i];
  std::memcpy(c->pinned + 64, dE, 48);
  FGD_CUDA(c, cudaMemcpyAsync(&c->sc->red[40], c->pinned + 64, 48, cudaMemcpyHostToDevice, c->stream));
  TRY(launch_init_iterate(c, c->st_eps, c->w_eps, &c->sc->red[40]));
  if (J > 0) FGD_CUDA(c, cudaMemcpyAsync(c->w_abar, c->st_abar, (size_t)J * n * 8, cudaMemcpyDeviceToDevice, c->stream));
  double S[6];
  for (int i = 0; i < 6; ++i) S[i] = inc->S_target[i] * c->stress_mask[i];
  const double sref = sigma_ref(c);
  int newton_total = 0, cg_total = 0, helm_total = 0, k = 0;
  double err = INFINITY, err_min = INFINITY;
  int stalled = 0;
  bool converged = false;
  double macro[6] = {0, 0, 0, 0, 0, 0};
  std::string why = "increment did not converge";
  // every exit fills rep with the work done so far (failed attempts included)
  auto fill_rep = [&]() {
    if (!rep) return;
    for (int i = 0; i < 6; ++i) rep->macro_stress[i] = macro[i];
    rep->err = err;
    rep->stag_it = k + (converged ? 1 : 0);
    rep->newton_it = newton_total;
    rep->cg_it = cg_total;
    rep->helm_it = helm_total;
  };
  // a hard (non-convergence-unrelated) error: report and return it
  auto hard = [&](fgd_status s) {
    fill_rep();
    return s;
  };
#define TRY_INC(x)                  \
  do {                              \
    fgd_status s_ = (x);            \
    if (s_ != FGD_OK) return hard(s_); \
  } while (0)
  for (k = 0; k < inc->max_stag; ++k) {
    FGD_CUDA(c, cudaMemcpyAsync(c->w_eps_prev, c->w_eps, 6 * n * 8, cudaMemcpyDeviceToDevice, c->stream));
    bool newton_ok = false;
    double rms_prev = INFINITY, lam = 1.0;
    int nback = 0;
    bool have_step = false;
    for (int r = 0; r <= inc->max_newton; ++r) {
      const fgd_status cs = fgd_constitutive(c, nullptr, nullptr, macro);
      if (cs == FGD_ENOCONV) {   // a GTN return mapping failed: roll back, the caller cuts back
        why = "GTN return mapping failed in increment";
        break;
      }
      if (cs != FGD_OK) return hard(cs);
      double rms;
      TRY_INC(fgd_mech_residual(c, S, nullptr, &rms));
      const double nm = std::sqrt(macro[0] * macro[0] + macro[1] * macro[1] + macro[2] * macro[2] + macro[3] * macro[3] +
                                  macro[4] * macro[4] + macro[5] * macro[5]);
      if (rms < inc->tol_newton * std::max(nm, 1e-6 * sref)) {
        newton_ok = true;
        break;
      }
      // R-LS: a Newton step that does not lower the residual RMS is halved (at most 5 times),
      // re-evaluating sigma and the residual at eps_r + lam de (no new linear solve)
      if (inc->line_search && have_step && rms >= rms_prev && nback < kMaxBacktrack) {
        lam *= 0.5;
        ++nback;
        if (trace_on() && c->rank == 0) fprintf(stderr, "fgd trace: stag %d newton %d backtrack lam %.4g\n", k, r, lam);
        TRY_INC(launch_axpy(c, 6 * n, c->w_eps, c->w_de, -lam));
        continue;
      }
      if (r == inc->max_newton) {
        why = "Newton did not converge in increment";
        break;
      }
      rms_prev = rms;
      lam = 1.0;
      nback = 0;
      have_step = true;
      int it = 0;
      double cg_rel = 0.0;
      fgd_status s = cg_mech(c, c->w_b, c->w_de, inc->tol_cg, inc->max_cg, &it, &cg_rel);
      cg_total += it;
      if (trace_on() && c->rank == 0)
        fprintf(stderr, "fgd trace: stag %d newton %d rms/|S| %.3e cg %d relres %.2e\n", k, r,
                rms / std::max(nm, 1e-6 * sref), it, cg_rel);
      if (s != FGD_OK && s != FGD_ENOCONV) return hard(s);
      ++newton_total;
      TRY_INC(launch_axpy(c, 6 * n, c->w_eps, c->w_de, 1.0));
    }
    if (!newton_ok) break;
    // Helmholtz solves with the converged sources (A-28)
    bool helm_ok = true;
    {
      // the J solves write abar^(k+1) into w_D (kept there until ERR is known), side by side on
      // launch-bound grids (helm_solve_all)
      fgd_status hs[kMaxFields];
      int hit[kMaxFields] = {};
      double hrel[kMaxFields] = {};
      fgd_status s = helm_solve_all(c, J, c->w_alpha, inc->warm_start ? c->w_abar : nullptr, c->w_D, inc->tol_helm,
                                    inc->max_helm, hs, hit, hrel);
      if (s != FGD_OK) return hard(s);
      for (int j = 0; j < J; ++j) {
        helm_total += hit[j];
        if (hs[j] == FGD_ENOCONV) {
          why = "Helmholtz PCG did not converge in increment";
          helm_ok = false;
        }
      }
    }
    if (!helm_ok) break;
    // ERR (A-02)
    FGD_CUDA(c, cudaMemsetAsync(&c->sc->maxbits, 0, 8, c->stream));
    TRY_INC(err_reduce(c, c->w_eps, c->w_eps_prev, c->w_D, c->w_abar));
    double red[14];
    unsigned long long mb;
    TRY_INC(sync_read(c, &c->sc->red[16], 8 * 14, red));
    TRY_INC(sync_read(c, &c->sc->maxbits, 8, &mb));
    double mx;
    std::memcpy(&mx, &mb, 8);
    double den = 0.0;
    for (int i = 0; i < 6; ++i) den += (red[i] / ng) * (red[i] / ng);
    den = std::sqrt(den);
    err = den > 1e-12 ? mx / den : mx;
    for (int j = 0; j < J; ++j) {
      const double dn = std::sqrt(red[7 + 2 * j]), nm = std::sqrt(red[6 + 2 * j]);
      err = std::max(err, dn > 1e-12 ? nm / dn : nm);
    }
    if (trace_on() && c->rank == 0) fprintf(stderr, "fgd trace: stag %d ERR %.3e\n", k, err);
    if (err < inc->tol_stag) {   // w_abar = abar^(k) (frozen in the mechanics), w_D = abar^(k+1)
      converged = true;
      break;
    }
    // stag_stall > 0 (off for Algorithm 1 as printed): give up once ERR has not improved on its
    // running minimum for that many consecutive iterations -- a staggered loop that unfreezes new
    // damage in every iteration (the step is too large); the caller cuts back (A-34) without
    // paying max_stag iterations first
    if (err < err_min) {
      err_min = err;
      stalled = 0;
    } else if (inc->stag_stall > 0 && ++stalled >= inc->stag_stall) {
      why = "staggered iteration stalled (ERR not improving)";
      break;
    }
    if (J > 0) FGD_CUDA(c, cudaMemcpyAsync(c->w_abar, c->w_D, (size_t)J * n * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
#undef TRY_INC
  fill_rep();
  if (!converged) {
    // rollback: committed state untouched; reset the iterate
    FGD_CUDA(c, cudaMemcpyAsync(c->w_eps, c->st_eps, 6 * n * 8, cudaMemcpyDeviceToDevice, c->stream));
    if (J > 0) FGD_CUDA(c, cudaMemcpyAsync(c->w_abar, c->st_abar, (size_t)J * n * 8, cudaMemcpyDeviceToDevice, c->stream));
    FGD_CUDA(c, cudaStreamSynchronize(c->stream));
    return set_err(c, FGD_ENOCONV, why);
  }
  // 3. commit (A-16, A-30): eps^p, eps_p recomputed at the converged strain with the fields the last
  // mechanics was frozen at; history from the accepted abar^(k+1)
  TRY(launch_commit(c, c->w_eps, J > 0 ? c->w_D : c->w_abar, c->cm_epsp, c->cm_ep, c->cm_hist));
  if (J > 0) FGD_CUDA(c, cudaMemcpyAsync(c->w_abar, c->w_D, (size_t)J * n * 8, cudaMemcpyDeviceToDevice, c->stream));
  std::swap(c->st_epsp, c->cm_epsp);
  std::swap(c->st_ep, c->cm_ep);
  std::swap(c->st_hist, c->cm_hist);
  FGD_CUDA(c, cudaMemcpyAsync(c->st_eps, c->w_eps, 6 * n * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (J > 0) FGD_CUDA(c, cudaMemcpyAsync(c->st_abar, c->w_abar, (size_t)J * n * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (rep) {
    FGD_CUDA(c, cudaMemsetAsync(&c->sc->maxbits, 0, 8, c->stream));
    TRY(err_reduce(c, c->st_eps, c->st_eps, c->st_abar, c->st_abar));
    double red[6];
    TRY(sync_read(c, &c->sc->red[16], 48, red));
    for (int i = 0; i < 6; ++i) rep->macro_strain[i] = red[i] / ng;
  }
  FGD_CUDA(c, cudaStreamSynchronize(c->stream));
  return FGD_OK;
}

fgd_status fgd_get_field(fgd_ctx* c, int which, double* out) {
  if (!c || !out) return set_err(c, FGD_EINVAL, "null argument");
  TRY(ensure_state(c));
  const size_t n = c->nvox;
  const double* src = nullptr;
  size_t cnt = n;
  if (which == FGD_FIELD_STRESS) src = c->w_sig, cnt = 6 * n;
  else if (which == FGD_FIELD_STRAIN) src = c->st_eps, cnt = 6 * n;
  else if (which == FGD_FIELD_EPS_P) src = c->st_epsp, cnt = 6 * n;
  else if (which == FGD_FIELD_EQPS) src = c->st_ep;
  else if (which == FGD_FIELD_HIST) src = c->st_hist;
  else if (which == FGD_FIELD_TANGENT) {
    if (c->compact) {
      TRY(dalloc(c, &c->C, 21 * n));
      TRY(launch_expand_tangent(c, c->Cc, c->C));
    }
    src = c->C, cnt = 21 * n;
  }
  else if (which == FGD_FIELD_ITERATE) src = c->w_eps, cnt = 6 * n;
  else if (which >= FGD_FIELD_NONLOCAL && which < FGD_FIELD_NONLOCAL + c->nfields)
    src = c->w_abar + (size_t)(which - FGD_FIELD_NONLOCAL) * n;
  else if (which >= FGD_FIELD_SOURCE && which < FGD_FIELD_SOURCE + c->nfields)
    src = c->w_alpha + (size_t)(which - FGD_FIELD_SOURCE) * n;
  else if (which >= FGD_FIELD_NONLOCAL_ITERATE && which < FGD_FIELD_NONLOCAL_ITERATE + c->nfields)
    src = c->w_abar + (size_t)(which - FGD_FIELD_NONLOCAL_ITERATE) * n;
  else return set_err(c, FGD_EINVAL, "unknown field");
  Stage st(c);
  double* d;
  TRY(st.out(out, cnt, &d));
  FGD_CUDA(c, cudaMemcpyAsync(d, src, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
  return st.finish();
}

fgd_status fgd_set_field(fgd_ctx* c, int which, const double* in) {
  if (!c || !in) return set_err(c, FGD_EINVAL, "null argument");
  if (!c->nonlocal_set) return set_err(c, FGD_ESTATE, "fgd_set_nonlocal must precede fgd_set_field");
  TRY(ensure_state(c));
  const size_t n = c->nvox;
  double* dst[2] = {nullptr, nullptr};
  size_t cnt = n;
  if (which == FGD_FIELD_STRAIN) dst[0] = c->st_eps, dst[1] = c->w_eps, cnt = 6 * n;
  else if (which == FGD_FIELD_EPS_P) dst[0] = c->st_epsp, cnt = 6 * n;
  else if (which == FGD_FIELD_EQPS) dst[0] = c->st_ep;
  else if (which == FGD_FIELD_HIST) dst[0] = c->st_hist;
  else if (which == FGD_FIELD_ITERATE) dst[0] = c->w_eps, cnt = 6 * n;
  else if (which >= FGD_FIELD_NONLOCAL && which < FGD_FIELD_NONLOCAL + c->nfields)
    dst[0] = c->st_abar + (size_t)(which - FGD_FIELD_NONLOCAL) * n, dst[1] = c->w_abar + (size_t)(which - FGD_FIELD_NONLOCAL) * n;
  else if (which >= FGD_FIELD_NONLOCAL_ITERATE && which < FGD_FIELD_NONLOCAL_ITERATE + c->nfields)
    dst[0] = c->w_abar + (size_t)(which - FGD_FIELD_NONLOCAL_ITERATE) * n;
  else return set_err(c, FGD_EINVAL, "unknown or read-only field");
  Stage st(c);
  const double* d;
  TRY(st.in(in, cnt, &d));
  for (double* t : dst)
    if (t) FGD_CUDA(c, cudaMemcpyAsync(t, d, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
  return st.finish();
}

static fgd_status flush_timing(fgd_ctx* c) {
  if (c->ev_rec.empty()) return FGD_OK;
  FGD_CUDA(c, cudaStreamSynchronize(c->stream));
  for (auto& r : c->ev_rec) {
    float ms = 0.f;
    FGD_CUDA(c, cudaEventElapsedTime(&ms, c->ev_pool[r.second.first], c->ev_pool[r.second.second]));
    c->kt_ms[r.first] += ms;
    c->kt_cnt[r.first] += 1;
  }
  c->ev_rec.clear();
  c->ev_used = 0;
  return FGD_OK;
}

fgd_status fgd_set_timing(fgd_ctx* c, int enable) {
  if (!c) return FGD_EINVAL;
  if (enable) {
    TRY(flush_timing(c));
    for (int i = 0; i < FGD_NUM_KCLASS; ++i) {
      c->kt_ms[i] = 0.0;
      c->kt_cnt[i] = 0;
    }
  }
  c->timing = enable != 0;
  return FGD_OK;
}

fgd_status fgd_kernel_times(fgd_ctx* c, double* ms, unsigned long long* count, int n) {
  if (!c) return FGD_EINVAL;
  TRY(flush_timing(c));
  for (int i = 0; i < n && i < FGD_NUM_KCLASS; ++i) {
    if (ms) ms[i] = c->kt_ms[i];
    if (count) count[i] = c->kt_cnt[i];
  }
  return FGD_OK;
}

fgd_status fgd_macro_stress(fgd_ctx* c, double out[6]) {
  if (!c || !out) return set_err(c, FGD_EINVAL, "null argument");
  for (int i = 0; i < 6; ++i) out[i] = c->last_macro[i];
  return FGD_OK;
}

}  // extern "C"
