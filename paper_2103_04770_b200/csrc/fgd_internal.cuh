// Internal declarations of libfgd (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

// Race hunting without compute-sanitizer (closed on this pool): a build with -DFGD_JITTER
// (build.py --jitter -> libfgd_jitter.so) makes every warp leaving a CTA barrier (__syncthreads,
// named barriers, warp syncs of the FFT exchanges) sleep a pseudo-random 0-4 us with probability
// 1/4.  Accesses that are not ordered by a barrier then interleave very differently from the
// production build, so tests/test_gpu_race.py compares both builds bit for bit.
#ifdef FGD_JITTER
__device__ __forceinline__ void fgd_jitter() {
  unsigned t = (unsigned)clock64() ^ ((threadIdx.x >> 5) * 2654435761u) ^ (blockIdx.x * 40503u);
  t ^= t >> 13;
  t *= 0x5bd1e995u;
  t ^= t >> 15;
  if ((t & 3u) == 0u) __nanosleep(t & 4095u);
}
__device__ __forceinline__ void fgd_syncthreads_jitter() {
  __syncthreads();
  fgd_jitter();
}
#define __syncthreads() fgd_syncthreads_jitter()
#define FGD_JIT() fgd_jitter()
#else
#define FGD_JIT() \
  do {            \
  } while (0)
#endif

#include "../../include/fgd.h"
#include "fft.cuh"

namespace fgd {

// Persistent grids are sized SMs x occupancy, so the per-CTA partial sums of a reduction (and
// therefore the last bits of the Krylov scalars) depend on the kernel's register / shared-memory
// footprint.  FGD_GRID_CAP=n caps every persistent grid at n CTAs (validation only: two builds
// with different footprints then reduce in the same order, tests/test_gpu_race.py).
inline int grid_cap(int g) {
  static const int cap = [] {
    const char* e = std::getenv("FGD_GRID_CAP");
    return e ? std::atoi(e) : 0;
  }();
  return cap > 0 && g > cap ? cap : g;
}

constexpr int kMaxPhases = 16;
constexpr int kMaxFields = 4;
constexpr int kMaxPeers = 8;     // ranks of the peer-store transposes (one NVLink domain)
constexpr int kMaxN = 512;
constexpr int kRedSlots = 48;            // doubles per reduction record
constexpr int kDistSlot = 47;            // local partial of a finalising reduction (nranks > 1)

// Device-resident Krylov / reduction scalars.  Written by the "last CTA" of a reducing kernel.
// Programmatic dependent launch (sm_90+): the hot-path kernels are launched with
// programmaticStreamSerialization, call pdl_trigger() first thing (so the NEXT kernel's CTAs may be
// scheduled onto SMs as this grid drains and run their prologue -- shared-memory tables, barrier
// init) and pdl_wait() before their first access to global data written by earlier work on the
// stream.  griddepcontrol.wait returns once the prerequisite grid has completed and its memory
// operations are visible; kernels launched without the attribute are unaffected.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Measured on the 256^3 sweep: with the attribute on, the early-resident dependent CTAs made the
// step 3.8 % SLOWER (42.7 vs 41.1 ms), so it is off; the device-side calls are then no-ops.
constexpr bool kUsePdl = false;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = kUsePdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

struct DevScalars;
// Device-side convergence guard of the Krylov loops: with tol > 0 the host launches iterations in
// batches and reads the flag once per batch; every kernel of an iteration returns immediately
// (uniformly, before any shared-memory work) once the finalise of the monitored reduction has
// set sc->done, so the iterate is exactly the one of the converged iteration.
__device__ __forceinline__ bool guard_done(const DevScalars* g);

struct DevScalars {
  double rr;        // mech: r.r        | helm: r.z
  double pq;        // mech: p.C p      | helm: p.L p
  double alpha;
  double beta;
  double bb;        // |b|^2 (stopping reference)
  double rn2;       // helm: r.r after the update
  double tol2;      // convergence threshold on the monitored square norm (tol^2 |b|^2)
  int done;         // set by the finalise once the monitored norm is below tol2
  int iters;        // Krylov iterations completed (device count)
  double red[kRedSlots];   // generic reduction results
  unsigned int counter[8];
  unsigned long long maxbits;
};

// Every hot kernel tests guard_done() BEFORE pdl_wait(): correct only while PDL is off (with PDL a
// dependent grid could read a stale done = 0 and run while later kernels of its iteration skip).
// Move the test after pdl_wait() before enabling kUsePdl.
static_assert(!kUsePdl, "guard_done() is read before pdl_wait(); see the note above");
__device__ __forceinline__ bool guard_done(const DevScalars* g) {
  return g != nullptr && *(volatile const int*)&g->done != 0;
}

enum RedOp : int {
  RED_NONE = 0,
  RED_STORE = 1,          // red[0..nv) = sums
  RED_MECH_INIT = 2,      // rr = bb = s0, beta = 0
  RED_MECH_PQ = 3,        // pq = s0, alpha = rr / pq
  RED_MECH_RR = 4,        // beta = s0 / rr, rr = s0
  RED_HELM_INIT = 5,      // rr(=r.z) = s0, beta = 0
  RED_HELM_PQ = 6,        // pq = s0, alpha = rr / pq
  RED_HELM_RN = 7,        // rn2 = s0
  RED_HELM_RZ = 8,        // beta = s0 / rr, rr = s0
  RED_BB = 9,             // bb = s0
};

struct Material {
  int model;
  double E, nu, sigma_y, H, eps_c, eps_r, d_max, kappa0, kappa_f;
  double q1, q2, q3, f_c, f_f, f_n, eps_n, s_n, n_hard, fstar_max;   // GTN (model 3)
};

struct ConstTables {
  const double2* tw[11];   // tw[log2 N] : e^{-2 pi i m / N}, m in [0, N)
};

}  // namespace fgd

// Layout A of the x-pass half spectra: A[c][z][kx / kKB][y][kx % kKB] (HxA = Hx rounded up to 4
// kx slots, the padding never read).  A y-pass tile of kKB kx reads kKB * Ny * 16 B contiguous per
// plane; an x-pass tile of kXR rows writes runs of kXR * kKB * 16 B.
constexpr int kKB = 2;   // kx block of layout A
constexpr int kXR = 2;   // rows per tile of the bulk-copy tangent x pass (k_xtan)
__host__ __device__ __forceinline__ size_t aidx(int HxA, int Ny, int Nz, int c, int z, int y, int kx) {
  return (((size_t)(c * Nz + z) * (HxA / kKB) + kx / kKB) * Ny + y) * kKB + (kx & (kKB - 1));
}

// Resources of one concurrently solved non-local field j >= 1 (NEXT#3, helm_solve_all): its own
// stream, Krylov scalars, work vectors and one-component spectrum buffers, so that the J independent
// Helmholtz solves of a staggered iteration run side by side on the GPU.
struct fgd_helm_sub {
  cudaStream_t stream = nullptr, cap = nullptr;
  cudaEvent_t ev = nullptr;
  double* hb[6] = {};
  double2 *specA = nullptr, *specB = nullptr, *specC = nullptr;
  fgd::DevScalars* sc = nullptr;
  double* partials = nullptr;
  size_t partials_cap = 0;
  double* pinned = nullptr;
};

struct fgd_ctx {
  int dims = 3;
  int n[3] = {1, 1, 1};        // Nx, Ny, Nz
  double L[3] = {1, 1, 1};
  double h[3] = {1, 1, 1};
  int scheme = 1;
  size_t nvox = 0;             // LOCAL voxels (this rank's z-slab)
  size_t nvox_g = 0;           // global voxels
  int nz_l = 1;                // local z planes
  int z0 = 0;                  // first global z plane of this rank
  int rank = 0, nranks = 1;    // processes (one GPU each)
  int P = 1;                   // slab count of the transposed-spectrum layout (nranks, or emulated)
  void* comm = nullptr;        // ncclComm_t
  void* loop = nullptr;        // loopback transport rank (dist.cu), instead of NCCL
  cudaStream_t comm_stream = nullptr;   // transposes of the overlapped y/z round trip (nranks > 1)
  std::vector<cudaEvent_t> ov_ev;       // chunk events of the overlapped round trip
  int sm_reserve = 0;          // SMs the persistent kernels leave free (overlapped communication)
  double2* specC = nullptr;    // z-pass buffer when P > 1
  // peer-store transposes (NEXT#4, FGD_PEER=1): every rank's specC in this process's address space
  bool peer_on = false, peer_ready = false;
  double2* peerC[fgd::kMaxPeers] = {};
  std::vector<void*> peer_ipc;          // mappings opened with cudaIpcOpenMemHandle (NCCL transport)
  double* bar_buf = nullptr;            // dummy of the allreduce used as a stream-ordered rank barrier
  double* halo = nullptr;      // stencil halo planes (nranks > 1): [field 0 lo, hi][field 1 lo, hi]
  uint8_t* phase_halo = nullptr;
  int Hx = 1;
  int HxA = 1;                 // kx stride of the x-pass spectrum layout A[c][z][y][kx] (Hx rounded up to 4)
  size_t nspec = 0;            // Hx * Ny * Nz complex per component
  size_t nspecA = 0;           // HxA * Ny * Nz
  int device = 0;
  cudaStream_t stream = nullptr;
  bool guard = false;                   // Krylov loop in flight: hot kernels skip once sc->done
  cudaStream_t aux = nullptr;           // second copy stream for split host<->device staging
  cudaStream_t cap = nullptr;           // stream used to capture Krylov iterations into CUDA graphs
  cudaEvent_t aux_ev[2] = {nullptr, nullptr};
  bool own_stream = false;
  std::string err;
  unsigned long long launches = 0;

  // tables
  double2* tw_all = nullptr;
  fgd::ConstTables tabs{};

  // geometry / materials
  uint8_t* phase = nullptr;
  int nphases = 0;
  std::vector<long long> phase_count;
  fgd::Material mat[fgd::kMaxPhases]{};
  bool mat_set[fgd::kMaxPhases]{};
  int nfields = 0;
  double ell[fgd::kMaxFields][fgd::kMaxPhases]{};
  int source_phase[fgd::kMaxFields]{};
  bool nonlocal_set = false;
  int stress_mask[6] = {0, 0, 0, 0, 0, 0};
  bool control_set = false;

  // device buffers (lazily allocated)
  double* C = nullptr;         // 21 * nvox packed tangent (fgd_set_tangent)
  double* Cc = nullptr;        // 9 * nvox compact tangent [n, ca, cb, cc] (fgd_constitutive)
  int compact = 0;             // 1: the CG uses Cc, 0: C
  bool tangent_set = false;
  double2* specA = nullptr;    // 6 * nspecA, layout A (see aidx)
  double2* specB = nullptr;    // 6 * nspec
  double* cg_x = nullptr;      // 6 * nvox
  double* cg_r = nullptr;
  double* cg_p = nullptr;
  double* hb[6] = {};          // helmholtz work vectors: x r z p0 p1 q
  int spec_comps = 6;          // components the spectrum buffers hold (1 in a concurrent-field copy)
  std::vector<fgd_helm_sub> hsub;   // concurrent solves of the fields j >= 1
  cudaEvent_t hsub_ev = nullptr;
  double* hg = nullptr;        // 3 * nvox: gradient field of the Fourier-form Helmholtz operator
  fgd::DevScalars* sc = nullptr;
  double* partials = nullptr;  // per-CTA partial sums
  size_t partials_cap = 0;
  double* pinned = nullptr;    // host pinned scalars

  // solver state (increment)
  double* st_eps = nullptr;    // 6 * nvox committed strain
  double* st_epsp = nullptr;   // 6 * nvox
  double* st_ep = nullptr;     // nvox
  double* st_hist = nullptr;   // nvox
  double* st_abar = nullptr;   // J * nvox
  double* w_eps = nullptr;     // 6 * nvox current iterate
  double* w_eps_prev = nullptr;
  double* w_sig = nullptr;     // 6 * nvox
  double* w_alpha = nullptr;   // J * nvox
  double* w_abar = nullptr;    // J * nvox
  double* w_D = nullptr;       // nvox frozen damage
  double* cm_epsp = nullptr;   // commit scratch (swapped with st_*)
  double* cm_ep = nullptr;
  double* cm_hist = nullptr;
  double* w_b = nullptr;       // 6 * nvox Newton residual
  double* w_de = nullptr;      // 6 * nvox Newton correction
  bool have_sigma = false;
  bool have_residual = false;
  double last_macro[6] = {0, 0, 0, 0, 0, 0};

  // per-kernel-class event timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<int, int>>> ev_rec;   // class, (start, end) event indices
  size_t ev_used = 0;
  double kt_ms[FGD_NUM_KCLASS] = {};
  unsigned long long kt_cnt[FGD_NUM_KCLASS] = {};
};

namespace fgd {

// error helpers
fgd_status set_err(fgd_ctx* c, fgd_status s, const std::string& m);
#define FGD_CUDA(ctx, call)                                                                   \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return ::fgd::set_err(ctx, FGD_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// scoped event timer around one kernel launch (no-op unless ctx->timing)
enum KClass : int { KC_XFWD6 = 0, KC_YFWD6, KC_Z6, KC_YINV6, KC_XINV6, KC_XFWD1, KC_YFWD1, KC_Z1, KC_YINV1, KC_XINV1,
                    KC_STENCIL, KC_CONST, KC_OTHER, KC_COMM, KC_XFWD6_CG };
struct KTimer {
  fgd_ctx* c;
  int cls, e0 = -1;
  KTimer(fgd_ctx* cc, int k);
  ~KTimer();
};

// launchers (passes.cu)
fgd_status launch_xfwd(fgd_ctx* c, int ncomp, int mode, const double* in0, const double* in1, double* out0,
                       const double* Cp, int red_op, int red_slot);
fgd_status launch_xfwd_io(fgd_ctx* c, int ncomp, int mode, const double* in0, const double* in1, double* out0,
                          double* io1, const double* Cp, int red_op, int red_slot, int first = 0);
fgd_status launch_yfwd(fgd_ctx* c, int ncomp);
fgd_status launch_z(fgd_ctx* c, int ncomp, int mode, double scale, const double* dc_shift, double mean_ell2);
fgd_status launch_yinv(fgd_ctx* c, int ncomp);
fgd_status launch_xinv(fgd_ctx* c, int ncomp, int mode, double* out0, double* io1, double* io2,
                       const double* in1, int red_op, int red_slot);
fgd_status ensure_spectral(fgd_ctx* c);
// pipes.cu (persistent cp.async pipelines)
fgd_status pipe_y(fgd_ctx* c, int ncomp, bool inv, int kxa = 0, int kxb = -1);
fgd_status pipe_z(fgd_ctx* c, int ncomp, int mode, double scale, const double* dc_shift, double mean_ell2, int kxa = 0,
                  int kxb = -1);
fgd_status pipe_xinv(fgd_ctx* c, int ncomp, int mode, double* out0, double* io1, double* io2, const double* in1,
                     int red_op, int red_slot);
fgd_status pipe_xfwd_plain(fgd_ctx* c, int ncomp, const double* in0);
fgd_status launch_precond_yz(fgd_ctx* c, double scale, double mean_ell2);
fgd_status ensure_partials(fgd_ctx* c, size_t nblocks);

// dist.cu
fgd_status dist_init(fgd_ctx* c, const fgd_dist* d);
void dist_destroy(fgd_ctx* c);
fgd_status exchange(fgd_ctx* c, int ncomp, bool fwd);
bool peer_mode(fgd_ctx* c);   // peer-store transposes requested and possible (nranks in [2, kMaxPeers])
fgd_status yz_round_trip(fgd_ctx* c, int ncomp, int zmode, double scale, const double* shift, double mean_ell2);
fgd_status allreduce_sum(fgd_ctx* c, double* dev, int count);
fgd_status allreduce_max_u64(fgd_ctx* c, unsigned long long* dev);
int red_op_for(const fgd_ctx* c, int op);
int red_slot_for(const fgd_ctx* c, int op, int slot);
fgd_status post_reduce(fgd_ctx* c, int op);
fgd_status halo_exchange(fgd_ctx* c, const void* field, size_t plane_bytes, void* lo, void* hi);

// helmholtz.cu
fgd_status launch_stencil(fgd_ctx* c, int field, int mode, const double* a, const double* zin,
                          const double* pold, double* pout, double* q, int red_op);
// Fourier form of the Helmholtz operator (continuous scheme, any scheme): y = a + F^-1 sum_j
// conj(k_j) F(l^2 F^-1(k_j F a)); with zin/pold: a = zin + beta pold is formed first and written to
// pout, and p.y is reduced with red_op (the PCG step, like launch_stencil's ST_PCG)
fgd_status helm_fourier(fgd_ctx* c, int field, const double* a, const double* zin, const double* pold, double* pout,
                        double* y, int red_op);
double mean_ell2(const fgd_ctx* c, int field);

// constitutive.cu
fgd_status launch_constitutive(fgd_ctx* c, const double* eps);
fgd_status launch_commit(fgd_ctx* c, const double* eps, const double* abar_new, double* epsp_out, double* ep_out,
                         double* hist_out);
bool has_gtn(const fgd_ctx* c);
fgd_status launch_err(fgd_ctx* c, const double* eps, const double* eps_prev, const double* abar_new,
                      const double* abar_old, unsigned long long* maxbits);
fgd_status launch_dot(fgd_ctx* c, size_t n, const double* a, const double* b, int op, int slot);
fgd_status launch_axpy(fgd_ctx* c, size_t n, double* y, const double* x, double s);
fgd_status launch_axpy_alpha(fgd_ctx* c, size_t n, double* y, const double* x);   // y += sc->alpha x
fgd_status launch_guard_init(fgd_ctx* c, double tol2);   // sc->tol2 = tol^2, done = iters = 0
fgd_status launch_init_iterate(fgd_ctx* c, const double* eps_n, double* eps, const double* dE6_dev);
fgd_status launch_phase_count(fgd_ctx* c, const uint8_t* ph, unsigned long long* cnt, int nph, int* bad);
fgd_status launch_expand_tangent(fgd_ctx* c, const double* Cc, double* Cp);

// x-pass modes
enum XFwdMode : int {
  XF_PLAIN = 0,        // tau_c = in0[c]
  XF_TANGENT = 1,      // tau = C : in0
  XF_TANGENT_CG = 2,   // x(io1) += alpha p(out0) [previous step]; p = r(in0) + beta p; tau = C p; write p, x;
                       // reduce p.tau
  XF_HELM_UPDATE = 3,  // x(out0) += alpha p(in0); r(io) -= alpha q(in1); tau = r ; reduce r.r
  XF_PLAIN_RED = 4,    // tau_c = in0[c]; reduce sum_c tau_c (means)
};
enum ZMode : int {
  Z_PROJECT = 0,   // 6 comps: Galerkin projection G^*(xi)
  Z_PRECOND = 1,   // 1 comp: scale / (1 + <l^2> |k|^2)
  Z_GRAD = 2,      // 3 comps (three copies of a^): comp j *= scale k_j          (Fourier-form Helmholtz)
  Z_DIV = 3,       // 3 comps: comp 0 = scale sum_j conj(k_j) g^_j, comps 1, 2 = 0
};
enum XInvMode : int {
  XI_STORE = 0,        // out0 = q
  XI_MECH_CG = 1,      // r(io2) = r_old(in1) - alpha q ; reduce r.r  (x is updated one step late, in
                       // XF_TANGENT_CG; in1 = b on the first step, = io2 afterwards)
  XI_HELM_Z = 2,       // z(out0) = q ; reduce r(in3).q
  XI_STORE_RR = 3,     // out0 = q ; reduce q.q
};

}  // namespace fgd
