// Shared-memory FP64 line FFTs for sm_100a (Stockham auto-sort, radix 2/4/8 butterflies in
// registers, one warp or a sub-warp group per line).
//
// Convention: forward F(u)(k) = sum_n u(n) e^{-2 pi i k n / N} (unnormalised),
// inverse with +i and no scaling here (the 1/N of F^-1 is folded into the spectral multiply).
//
// A line of N complex doubles lives in shared memory with one 16 B pad slot every 8 elements
// (PAD) to break the stride-8 bank pattern of the first Stockham passes, and an odd line stride
// so that "same index, consecutive lines" accesses are conflict free.  Each line is owned by
// TPL = N / E threads (E = 8 elements per thread per pass); passes are separated by
// __syncwarp() when a line sits in one warp, by a named barrier per line otherwise (N = 512).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fgd {

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }
// Two plan families: W = false (8 points per thread; radix-8/4 passes, more threads per line) and
// W = true ("wide": 16 points per thread for N = 128/256 with radix-16 passes -- two shared-memory
// exchanges instead of three, for the shared-memory-bound C2C passes).
__host__ __device__ constexpr int fft_E(int N, bool W = false) { return N < 8 ? N : ((W && (N == 128 || N == 256)) ? 16 : 8); }
__host__ __device__ constexpr int fft_TPL(int N, bool W = false) { return N / fft_E(N, W); }
__host__ __device__ constexpr int fft_npass(int N, bool W = false) {
  return N <= 1 ? 0 : (N <= 8 ? 1 : (N <= 64 ? 2 : ((W && N <= 256) ? 2 : 3)));
}
// W = false: 2:{2} 4:{4} 8:{8} 16:{4,4} 32:{8,4} 64:{8,8} 128:{8,4,4} 256:{8,8,4} 512:{8,8,8}
// W = true : as above except 128:{8,16} 256:{16,16}
__host__ __device__ constexpr int fft_radix(int N, int p, bool W = false) {
  return N <= 8 ? N
       : N == 16 ? 4
       : N == 32 ? (p == 0 ? 8 : 4)
       : N == 64 ? 8
       : N == 128 ? (W ? (p == 0 ? 8 : 16) : (p == 0 ? 8 : 4))
       : N == 256 ? (W ? 16 : (p < 2 ? 8 : 4))
       : 8;
}
__host__ __device__ constexpr int fft_ns(int N, int p, bool W = false) {
  return p == 0 ? 1 : fft_ns(N, p - 1, W) * fft_radix(N, p - 1, W);
}
// Per-pass twiddle tables: pass p with stride NS > 1 stores w^{r k}, r = 1..P-1, k = 0..NS-1, at
// offset tw_off(N, p) + (r - 1) NS + k, so that the threads of a warp (consecutive k) read
// consecutive 16 B words (no bank conflicts) -- w = e^{-2 pi i / (NS P)}.
__host__ __device__ constexpr int tw_off(int N, int p, bool W = false) {
  return p == 0 ? 0
                : tw_off(N, p - 1, W) +
                      (fft_ns(N, p - 1, W) > 1 ? (fft_radix(N, p - 1, W) - 1) * fft_ns(N, p - 1, W) : 0);
}
__host__ __device__ constexpr int tw_total(int N, bool W = false) { return N <= 1 ? 0 : tw_off(N, fft_npass(N, W), W); }
__host__ __device__ constexpr int pad_len(int N) { return N + (N >> 3); }
__device__ __forceinline__ int PAD(int i) { return i + (i >> 3); }
// Slot of element i of line l.  The padded layout PAD keeps every address an immediate offset
// from one base register per thread (cheap in registers; an XOR swizzle was measured to double
// the register demand of the unrolled passes); `l` is kept in the signature so that the layout
// can change in one place.
__device__ __forceinline__ int SWZ(int, int i) { return PAD(i); }
// shared-memory stride (complex slots) of a C2C line of N points / of an x line (M points plus
// the Nyquist slot): odd, so that consecutive lines start in different 16 B bank groups.
__host__ __device__ constexpr int cline(int N) { return pad_len(N) | 1; }
__host__ __device__ constexpr int xline(int M) { return (pad_len(M) + 1) | 1; }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conjg(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV> __device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <int P, bool INV> __device__ __forceinline__ void dft(double2* v);

template <> __device__ __forceinline__ void dft<1, false>(double2*) {}
template <> __device__ __forceinline__ void dft<1, true>(double2*) {}

template <int P, bool INV> __device__ __forceinline__ void dft2(double2* v) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
template <> __device__ __forceinline__ void dft<2, false>(double2* v) { dft2<2, false>(v); }
template <> __device__ __forceinline__ void dft<2, true>(double2* v) { dft2<2, true>(v); }

template <bool INV> __device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  double2 t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = mul_mi<INV>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}
template <> __device__ __forceinline__ void dft<4, false>(double2* v) { dft4<false>(v[0], v[1], v[2], v[3]); }
template <> __device__ __forceinline__ void dft<4, true>(double2* v) { dft4<true>(v[0], v[1], v[2], v[3]); }

template <bool INV> __device__ __forceinline__ void dft8(double2* v) {
  constexpr double c = 0.70710678118654752440;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  // w = e^{-i pi/4} (forward) / e^{+i pi/4} (inverse)
  double2 w1o1 = INV ? make_double2(c * (o1.x - o1.y), c * (o1.x + o1.y))
                     : make_double2(c * (o1.x + o1.y), c * (o1.y - o1.x));
  double2 w2o2 = mul_mi<INV>(o2);
  double2 w3o3 = INV ? make_double2(-c * (o3.x + o3.y), c * (o3.x - o3.y))
                     : make_double2(c * (o3.y - o3.x), -c * (o3.x + o3.y));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, w1o1);
  v[5] = csub(e1, w1o1);
  v[2] = cadd(e2, w2o2);
  v[6] = csub(e2, w2o2);
  v[3] = cadd(e3, w3o3);
  v[7] = csub(e3, w3o3);
}
template <> __device__ __forceinline__ void dft<8, false>(double2* v) { dft8<false>(v); }
template <> __device__ __forceinline__ void dft<8, true>(double2* v) { dft8<true>(v); }

// radix-16 as 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2; DFT4 over n1, twiddle W16^{n2 k1}, DFT4 over n2
template <bool INV> __device__ __forceinline__ double2 w16(double2 a, int e) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
  // a * W16^e, W16 = e^{-i pi/8} (forward) / e^{+i pi/8} (inverse); e in {1,2,3,4,6,9}
  double2 w;
  switch (e) {
    case 1: w = make_double2(c1, -s1); break;
    case 2: w = make_double2(h, -h); break;
    case 3: w = make_double2(s1, -c1); break;
    case 4: w = make_double2(0.0, -1.0); break;
    case 6: w = make_double2(-h, -h); break;
    default: w = make_double2(-c1, s1); break;   // 9
  }
  if (INV) w.y = -w.y;
  return cmul(a, w);
}
template <bool INV> __device__ __forceinline__ void dft16(double2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);   // v[4 k1 + n2] = y[n2][k1]
  v[5] = w16<INV>(v[5], 1);
  v[6] = w16<INV>(v[6], 2);
  v[7] = w16<INV>(v[7], 3);
  v[9] = w16<INV>(v[9], 2);
  v[10] = mul_mi<INV>(v[10]);
  v[11] = w16<INV>(v[11], 6);
  v[13] = w16<INV>(v[13], 3);
  v[14] = w16<INV>(v[14], 6);
  v[15] = w16<INV>(v[15], 9);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);  // X[k1+4k2] at v[4k1+k2]
  double2 t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[4 * k1 + k2];
}
template <> __device__ __forceinline__ void dft<16, false>(double2* v) { dft16<false>(v); }
template <> __device__ __forceinline__ void dft<16, true>(double2* v) { dft16<true>(v); }

// cos(pi e / 16) for any integer e (compile-time constant after unrolling)
__host__ __device__ constexpr double cos_pi16(int e) {
  constexpr double C[9] = {1.0,
                           0.98078528040323044912618223613424,
                           0.92387953251128675612818318939679,
                           0.83146961230254523707878837761791,
                           0.70710678118654752440084436210485,
                           0.55557023301960222474283081394853,
                           0.38268343236508977172845998403040,
                           0.19509032201612826784828486847702,
                           0.0};
  e &= 31;
  return e <= 8 ? C[e] : (e <= 16 ? -C[16 - e] : (e <= 24 ? -C[e - 16] : C[32 - e]));
}
// a * W32^e, W32 = e^{-2 pi i / 32} (forward) / e^{+2 pi i / 32} (inverse)
template <bool INV> __device__ __forceinline__ double2 w32(double2 a, int e) {
  if ((e & 31) == 8) return mul_mi<INV>(a);
  const double c = cos_pi16(e), s = cos_pi16(8 - e);   // sin(pi e / 16) = cos(pi (8 - e) / 16)
  return cmul(a, make_double2(c, INV ? s : -s));
}
// radix-32 as 4 x 8: n = n2 + 8 n1 (n1 < 4, n2 < 8), k = k1 + 4 k2 (k1 < 4, k2 < 8):
// DFT4 over n1, twiddle W32^{n2 k1}, DFT8 over n2, reorder to natural order (free after unrolling)
// First stage (DFT4 over n1 and the W32 twiddles, in place): afterwards dft8(v + 8 k1) leaves
// X[k1 + 4 k2] at v[8 k1 + k2] -- callers that consume the outputs group by group (storing each
// group at once, to keep the register footprint down) call the two stages themselves.
template <bool INV> __device__ __forceinline__ void dft32_stage1(double2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2) dft4<INV>(v[n2], v[8 + n2], v[16 + n2], v[24 + n2]);   // v[n2 + 8 k1] = Y[n2][k1]
#pragma unroll
  for (int k1 = 1; k1 < 4; ++k1)
#pragma unroll
    for (int n2 = 1; n2 < 8; ++n2) v[n2 + 8 * k1] = w32<INV>(v[n2 + 8 * k1], n2 * k1);
}
template <bool INV> __device__ __forceinline__ void dft32(double2* v) {
  dft32_stage1<INV>(v);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft8<INV>(v + 8 * k1);                                  // v[8 k1 + k2] = X[k1 + 4 k2]
  double2 t[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) t[i] = v[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) v[k1 + 4 * k2] = t[8 * k1 + k2];
}

// Twiddle load from the shared-memory table through a volatile asm.  Keeps the compiler
// from hoisting every twiddle of every pass out of a persistent tile loop into registers.
__device__ __forceinline__ double2 ld_tw(const double2* p) {
  double2 w;
  const unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y) : "r"(s));
  return w;
}

// One Stockham pass of radix P over a line of N (padded, in shared memory).  Thread t in
// [0, TPL) owns E/P butterflies j = t + b*TPL.  tw = table e^{-2 pi i m / N}, m in [0, N).
// Synchronise the TPL threads that own a line: a warp (or part of one) -> __syncwarp; two or
// more warps (N = 512: TPL = 64) -> a named barrier per line slot.
template <int TPL>
__device__ __forceinline__ void line_sync(int bar) {
  if constexpr (TPL <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(TPL) : "memory");
  }
  FGD_JIT();
}

template <int N, int P, int NS, bool INV, bool W, int PASS>
__device__ __forceinline__ void stockham_pass(double2* line, int l, int t, bool active, const double2* tw, int bar) {
  constexpr int E = fft_E(N, W);
  constexpr int TPL = fft_TPL(N, W);
  constexpr int NB = E / P;          // butterflies per thread
  constexpr int NP = N / P;          // butterflies per line
  // Loads and arithmetic are unconditional (an inactive group reads a valid line and discards
  // the result); only the stores are predicated.  Keeping v[] out of divergent regions stops
  // the compiler from spilling it around the reconvergence point.
  double2 v[E];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + b * TPL;
#pragma unroll
    for (int r = 0; r < P; ++r)
      v[b * P + r] = (NP % 8 == 0) ? line[SWZ(l, j) + r * (NP / 8 * 9)] : line[SWZ(l, j + r * NP)];
  }
  line_sync<TPL>(bar);
  {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = t + b * TPL;
      const int k = j % NS;
      if (NS > 1) {
        constexpr int OFF = tw_off(N, PASS, W);
#pragma unroll
        for (int r = 1; r < P; ++r) {
          double2 w = ld_tw(tw + OFF + (r - 1) * NS + k);
          if (INV) w.y = -w.y;
          v[b * P + r] = cmul(v[b * P + r], w);
        }
      }
      dft<P, INV>(&v[b * P]);
      const int base = (j / NS) * NS * P + k;
      if (active) {
#pragma unroll
        for (int r = 0; r < P; ++r) {
          // PAD(base + r NS) as one base register + immediate: NS % 8 == 0 -> 9 NS/8 per step;
          // NS == 1 -> base is a multiple of P, so PAD(base + r) = PAD(base) + r + r/8 for P >= 8
          // and PAD(base) + r for P < 8 ([base, base + P) does not cross a multiple of 8)
          const int o = (NS % 8 == 0) ? SWZ(l, base) + r * (NS / 8 * 9)
                      : (NS == 1) ? SWZ(l, base) + r + (r >> 3) : SWZ(l, base + r * NS);
          line[o] = v[b * P + r];
        }
      }
    }
  }
  line_sync<TPL>(bar);
}

template <int N, int PASS, int NS, bool INV, bool W>
__device__ __forceinline__ void fft_passes(double2* line, int l, int t, bool active, const double2* tw, int bar) {
  if constexpr (PASS < fft_npass(N, W)) {
    constexpr int P = fft_radix(N, PASS, W);
    stockham_pass<N, P, NS, INV, W, PASS>(line, l, t, active, tw, bar);
    fft_passes<N, PASS + 1, NS * P, INV, W>(line, l, t, active, tw, bar);
  }
}

// Copy a table of n entries into shared memory (all threads; caller syncs).
__device__ __forceinline__ void load_table(double2* dst, const double2* __restrict__ src, int n) {
  const int nt = blockDim.x * blockDim.y * blockDim.z;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  for (int i = tid; i < n; i += nt) dst[i] = __ldg(&src[i]);
}

// Build the per-pass twiddle tables of an N-point FFT (tw_total(N) entries) in shared memory from
// the global table e^{-2 pi i m / N} (all threads; caller syncs).
template <int N, bool W = false, int PASS = 0>
__device__ __forceinline__ void build_pass_tables(double2* dst, const double2* __restrict__ twN) {
  if constexpr (PASS < fft_npass(N, W)) {
    constexpr int NS = fft_ns(N, PASS, W), P = fft_radix(N, PASS, W);
    if constexpr (NS > 1) {
      constexpr int STEP = N / (NS * P), OFF = tw_off(N, PASS, W);
      const int nt = blockDim.x * blockDim.y * blockDim.z;
      const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
      for (int i = tid; i < (P - 1) * NS; i += nt) {
        const int r = 1 + i / NS, k = i % NS;
        dst[OFF + i] = __ldg(&twN[r * k * STEP]);
      }
    }
    build_pass_tables<N, W, PASS + 1>(dst, twN);
  }
}

// FFT all `nl` lines (stride ldl elements) of a CTA's shared buffer.  Every thread of the CTA
// must call this (warp-synchronous inside); lines are distributed TPL threads per line.
template <int N, bool INV, bool W = false>
__device__ __forceinline__ void fft_lines(double2* buf, int nl, int ldl, const double2* tw) {
  if constexpr (N > 1) {
    constexpr int TPL = fft_TPL(N, W);
    const int lines_per_round = blockDim.x / TPL;
    const int slot = threadIdx.x / TPL;
    const int t = threadIdx.x % TPL;
    for (int base = 0; base < nl; base += lines_per_round) {
      const int l = base + slot;
      const bool active = l < nl;
      fft_passes<N, 0, 1, INV, W>(buf + (size_t)(active ? l : 0) * ldl, active ? l : 0, t, active, tw, 1 + slot);
    }
  }
}


// ---------------------------------------------------------------------------------------------
// Register FFTs of one 128- or 256-point line held in shared memory (natural padded order SWZ in
// and out), for the x passes.  M = 16 x T (T = 8 or 16 threads per line, all in one warp, 16
// points per thread): thread tt loads z[tt + T j], DFT16 over j, twiddle W_M^{tt k2}, one exchange
// (rows of T + 1 slots), DFT_T over n1 for k2 = tt (+ 8 when T = 8: two DFT8), written back in
// natural order.  Two shared-memory accesses per point for the exchange instead of two per radix
// pass.  twR[(k2 - 1) T + tt] = W_M^{tt k2}; the inverse uses the conjugates.
template <int M>
__host__ __device__ constexpr bool fft_reg_ok() { return M == 128 || M == 256; }
template <int M>
__host__ __device__ constexpr int fft_reg_tpl() { return M / 16; }

template <int M>
__device__ __forceinline__ void fft_reg_tables(double2* twR, const double2* __restrict__ twM) {
  constexpr int T = M / 16;
  const int nt = blockDim.x * blockDim.y * blockDim.z;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  for (int k = tid; k < 15 * T; k += nt) twR[k] = __ldg(&twM[(k % T) * (1 + k / T)]);
}

template <int M, bool INV>
__device__ __forceinline__ void fft_reg_inplace(double2* ln, int l, int tt, const double2* twR) {
  constexpr int T = M / 16;
  constexpr int RP = T + 1;   // exchange row pitch
  double2 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = ln[SWZ(l, tt + T * j)];
  dft16<INV>(v);
#pragma unroll
  for (int k2 = 1; k2 < 16; ++k2) {
    double2 w = ld_tw(twR + (k2 - 1) * T + tt);
    if (INV) w.y = -w.y;
    v[k2] = cmul(v[k2], w);
  }
  __syncwarp();
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) ln[k2 * RP + tt] = v[k2];
  __syncwarp();
  if constexpr (T == 16) {
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) v[n1] = ln[tt * RP + n1];
    dft16<INV>(v);
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) ln[SWZ(l, tt + 16 * k1)] = v[k1];
  } else {
    double2 u0[8], u1[8];
#pragma unroll
    for (int n1 = 0; n1 < 8; ++n1) {
      u0[n1] = ln[tt * RP + n1];
      u1[n1] = ln[(tt + 8) * RP + n1];
    }
    dft<8, INV>(u0);
    dft<8, INV>(u1);
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
      ln[SWZ(l, tt + 16 * k1)] = u0[k1];
      ln[SWZ(l, tt + 8 + 16 * k1)] = u1[k1];
    }
  }
}


}  // namespace fgd
