/* fgd.h -- C ABI of libfgd: the data-parallel hot path of the staggered FFT solver for
 * implicit-gradient ductile damage of Magri, Lucarini, Lemoine, Adam, Segurado,
 * "An FFT framework for simulating non-local ductile failure in heterogeneous materials"
 * (arXiv 2103.04770).  Citations "P:<n>" are lines of the paper's source; "A-xx"
 * are the readings listed in DESIGN.md.
 *
 * CONVENTIONS
 *  - All reals are IEEE float64.  Moduli/stresses in the caller's unit (the tests use MPa).
 *  - A "field" is contiguous [comp][z][y][x] (x fastest), N = N1*N2*N3 voxels per component.
 *    Tensor fields have 6 Mandel components (11, 22, 33, sqrt2*23, sqrt2*13, sqrt2*12);
 *    scalar fields have 1.  2D plane strain is N3 = 1 (A-19).
 *  - Tangents are 21 packed components (upper triangle of the symmetric 6x6 Mandel matrix,
 *    row-major: (0,0),(0,1)..(0,5),(1,1)..(5,5)), layout [21][z][y][x].
 *  - POINTERS: every field pointer may be a DEVICE pointer (used in place, work enqueued on
 *    the context stream; the call returns after the result is complete) or a HOST pointer
 *    (pageable or pinned; staged through device memory by the library).  The library never
 *    frees or retains caller pointers beyond the call.  Outputs must not alias inputs unless
 *    stated.
 *  - Grids: N1, N2 powers of two in [4, 512]; N3 = 1 or a power of two in [2, 512].
 *  - Thread-compatible, not thread-safe: one host thread per context.
 *  - ERRORS: no exception or abort crosses the ABI; every failure returns a negative
 *    fgd_status and the message is available from fgd_last_error(ctx).
 */
#ifndef FGD_H
#define FGD_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FGD_OK = 0,
  FGD_EINVAL = -1,   /* bad argument: N_i unsupported, L_i <= 0, nu out of range, unknown field */
  FGD_ESHAPE = -2,   /* size/extent mismatch */
  FGD_ECUDA = -3,    /* CUDA runtime error (message has the CUDA error string) */
  FGD_ENCCL = -4,    /* collective error (multi-GPU) */
  FGD_ENOMEM = -5,   /* device allocation failed */
  FGD_ENOCONV = -6,  /* Newton/CG/PCG/staggered did not converge; increment state rolled back */
  FGD_ESTATE = -7    /* call-order violation, e.g. apply before set_phases */
} fgd_status;

typedef struct fgd_ctx fgd_ctx;

/* Grid.  scheme: 0 = continuous frequencies k = i xi (A-06),
 * 1 = Willot rotated finite-difference scheme (A-04; default).
 * The Helmholtz operator is applied as the exact 27-point real-space stencil of the Willot symbol
 * (scheme 1) or in its Fourier form L^ = 1 + sum_j conj(k_j) F(l^2 F^-1(k_j .)) (A-09;
 * scheme 0: two 3-component FFT round trips per apply). */
typedef struct {
  int dims;       /* 2 or 3 */
  int n[3];       /* N1, N2, N3 (N3 = 1 for dims = 2) */
  double L[3];    /* cell edge lengths, > 0 */
  int scheme;
} fgd_grid;

/* Process placement: one process per GPU.  nranks > 1 slab-decomposes the cell along z
 * (N3 and N2 divisible by nranks, powers of two): every field argument is then this rank's
 * z-slab [comp][z0 .. z0+nz)[y][x] (fgd_local_extent), FFT transposes are NCCL block
 * all-to-alls, reductions NCCL allreduces.  nccl_id: 128 bytes from
 * fgd_nccl_id() on rank 0, broadcast to all ranks (ignored for nranks = 1).
 * stream: the cudaStream_t all work is enqueued on; NULL = the legacy default stream (orders
 * against the caller's work on any blocking stream).  With a non-default stream the caller
 * must order its producers of input data against it. */
typedef struct {
  int rank, nranks, device;
  const unsigned char* nccl_id; /* 128 bytes or NULL */
  void* stream;
} fgd_dist;

fgd_status fgd_create(const fgd_grid* grid, const fgd_dist* dist, fgd_ctx** out);
/* 128-byte NCCL unique id for fgd_dist.nccl_id (call on rank 0 only). */
fgd_status fgd_nccl_id(unsigned char* out);
/* 128-byte id of an in-process LOOPBACK group (validation transport): passed as fgd_dist.nccl_id
 * to nranks contexts of ONE process (typically on one GPU, each driven by its own host thread,
 * ranks 0..nranks-1), it makes them a multi-rank group whose collectives are stream-ordered
 * device-to-device copies synchronised by CUDA events and host barriers instead of NCCL.  Every
 * nranks > 1 code path (slab layouts, transposes, z-halos, distributed reductions) runs as with
 * NCCL.  All ranks must issue the same sequence of collective calls (as with NCCL); a rank that
 * stops calling makes the others fail with FGD_ENCCL after 300 s. */
fgd_status fgd_loopback_id(unsigned char* out);
void fgd_destroy(fgd_ctx* ctx);
const char* fgd_last_error(const fgd_ctx* ctx);
fgd_status fgd_local_extent(const fgd_ctx* ctx, int* z0, int* nz);
/* number of CUDA kernels this context has launched so far */
unsigned long long fgd_launch_count(const fgd_ctx* ctx);

/* Phase map (Omega = U Omega_q): one uint8 per voxel, values < nphases <= 16. */
fgd_status fgd_set_phases(fgd_ctx* ctx, const uint8_t* phase, int nphases);

/* Per-phase material (A-17, A-18, A-30..A-33).
 * model 0 elastic (E, nu); 1 J2-Lemaitre with linear hardening sigma_0 = sigma_y + H eps_p and
 * damage D(ebar) = clamp((ebar - eps_c)/(eps_r - eps_c), 0, d_max); 2 elastic-brittle particle
 * with d = clamp((kappa - kappa0)/(kappa_f - kappa0), 0, d_max); 3 non-local GTN (Sec. 2.1.1
 * P:89-166, Sec. 2.2.2, App. A): yield
 * (q/sigma_0)^2 + 2 f* q1 cosh(-3 q2 p/(2 sigma_0)) - (1 + q3 f*^2), Aravas hardening
 * sigma_0/sigma_y = (sigma_0/sigma_y + 3 mu eps0p/sigma_y)^n_hard, f* law with
 * f_c, f_f capped at fstar_max, Chu-Needleman nucleation f_n, eps_n, s_n
 * (P:151-155).  A GTN phase q needs two consecutive non-local fields j, j+1 with
 * source_phase = q: field j regularises eps0p, field j+1 tr eps^p; its porosity is
 * frozen from them during the mechanics (App. A).  E > 0, -1 < nu < 0.5.  The GTN fields
 * are ignored by the other models. */
typedef struct {
  int model;
  double E, nu, sigma_y, H, eps_c, eps_r, d_max, kappa0, kappa_f;
  double q1, q2, q3, f_c, f_f, f_n, eps_n, s_n, n_hard, fstar_max;
} fgd_material;
fgd_status fgd_set_material(fgd_ctx* ctx, int phase, const fgd_material* m);

/* Non-local fields: nfields <= 4; ell [nfields][nphases] in length units
 * (piecewise-constant ell_j(x), Remark P:394-405); source_phase[j] = the phase whose local
 * variable field j regularises (alpha_j = 0 elsewhere). */
fgd_status fgd_set_nonlocal(fgd_ctx* ctx, int nfields, const double* ell, const int* source_phase);

/* Mixed macroscopic control: stress_mask[6], 1 = stress-controlled. */
fgd_status fgd_set_control(fgd_ctx* ctx, const int* stress_mask);

/* Set the per-voxel tangent used by the projected-tangent apply and the mechanical CG
 * (config 1 supplies a random SPD tangent; fgd_constitutive overwrites it). */
fgd_status fgd_set_tangent(fgd_ctx* ctx, const double* C);

/* y = G*(C : x): the FFT-Galerkin projected tangent apply.  G* is the orthogonal
 * projection onto compatible fields with the zero-frequency Mandel mask of fgd_set_control
 * (A-07, A-08).  x, y: 6-component fields. */
fgd_status fgd_apply_projected_tangent(fgd_ctx* ctx, const double* x, double* y);

/* y = G*(tau - Sigma) with Sigma = S (6 doubles, may be NULL = 0) removed from the mean
 * (the Newton residual is -fgd_apply_projection(sigma, Sigma_bar)). */
fgd_status fgd_apply_projection(fgd_ctx* ctx, const double* tau, const double* S, double* y);

/* y = a - div(ell_j^2(x) grad a) for non-local field j (A-09), real space in/out. */
fgd_status fgd_apply_helmholtz(fgd_ctx* ctx, int field, const double* a, double* y);

/* z = F^-1[ F(r) / (1 + <ell_j^2> |k|^2) ] (A-11). */
fgd_status fgd_apply_helmholtz_precond(fgd_ctx* ctx, int field, const double* r, double* z);

/* Algorithm 2: abar = L_j^{-1} src by preconditioned CG from abar = 0, stop when
 * ||L abar - src|| < tol ||src|| or after maxit iterations (tol <= 0: exactly maxit).
 * src == NULL uses the source alpha_j of the last fgd_constitutive call; abar == NULL keeps
 * the result internal (it becomes the frozen non-local field for the next fgd_constitutive).
 * *iters (may be NULL) receives the iteration count, *relres the final relative residual. */
fgd_status fgd_solve_helmholtz(fgd_ctx* ctx, int field, const double* src, double* abar, double tol,
                               int maxit, int* iters, double* relres);

/* Algorithm 2 from an initial guess x0 (NULL = 0; the warm start of S:262): the same stopping rule
 * ||L abar - src|| < tol ||src|| (relative to the source, not to the initial residual); a guess
 * that already meets it is returned after 0 iterations.  src, x0, abar: 1-component fields. */
fgd_status fgd_solve_helmholtz_from(fgd_ctx* ctx, int field, const double* src, const double* x0, double* abar,
                                    double tol, int maxit, int* iters, double* relres);

/* All J non-local fields of fgd_set_nonlocal in one call (NEXT#3).  The J generalized Helmholtz
 * problems of a staggered iteration are independent ("computed independently"), so
 * they are solved SIDE BY SIDE: one stream, one set of Krylov scalars and work vectors per field,
 * each running Algorithm 2 exactly as fgd_solve_helmholtz_from does (bitwise the same iterates,
 * iteration counts and results as J consecutive calls).  On launch-latency-bound grids (<= 2^21
 * voxels, one GPU) the solves overlap on the device; on larger grids and with nranks > 1 they run
 * one after another.  src, x0 (NULL = 0), abar: J one-component fields one after another
 * ([J][N3_local][N2][N1], host or device); iters, relres: arrays of J (may be NULL).
 * Returns FGD_ENOCONV if any field did not reach tol within maxit (the others are still returned;
 * consecutive mode stops at the first failing field). */
fgd_status fgd_solve_helmholtz_all(fgd_ctx* ctx, const double* src, const double* x0, double* abar, double tol,
                                   int maxit, int* iters, double* relres);

/* Mechanical linear solve of one Newton step: unpreconditioned CG for
 * G*(C : de) = b with de_0 = 0; b must lie in range(G*) (e.g. a Newton residual).  Same
 * stopping rule and NULL conventions as fgd_solve_helmholtz (b == NULL: the residual of the
 * last fgd_mech_residual; de == NULL: keep the correction internal). */
fgd_status fgd_solve_tangent_cg(fgd_ctx* ctx, const double* b, double* de, double tol, int maxit,
                                int* iters, double* relres);

/* Per-voxel constitutive update (A-14..A-18; GTN P:89-166,
 * P:1100-1129, A-30..A-33) at strain eps (6 comps; NULL = the internal iterate) with the
 * committed state and damage / porosity frozen from the current non-local fields
 * (FGD_FIELD_NONLOCAL_ITERATE, A-16).  Produces sigma, the consistent tangent (GTN:
 * its symmetric part) and the Helmholtz sources alpha_j internally; sigma_out (may be NULL)
 * receives sigma; macro[6] (may be NULL) receives <sigma>.  Returns FGD_ENOCONV (outputs
 * written, the failing points hold their last return-mapping iterate) if a GTN return mapping
 * did not converge in 50 Newton steps; FGD_ESTATE if a GTN phase lacks its two consecutive
 * non-local fields. */
fgd_status fgd_constitutive(fgd_ctx* ctx, const double* eps, double* sigma_out, double* macro);

/* Newton residual b = -G*(sigma - Sigma_bar) of the last fgd_constitutive,
 * kept internal; b_out (may be NULL) receives it, *rms (may be NULL) its RMS over voxels. */
fgd_status fgd_mech_residual(fgd_ctx* ctx, const double* S_target, double* b_out, double* rms);

/* One increment of Algorithm 1: mixed-control Newton + CG mechanics and J
 * Helmholtz PCG solves iterated until ERR < tol_stag (A-01, A-02).  Commits on FGD_OK
 * (eps^p, eps_p from the last mechanical solve, histories from the accepted non-local fields,
 * A-16, A-30); on FGD_ENOCONV (Newton, staggered or GTN return-mapping failure) the committed
 * state is unchanged (rollback) and the caller cuts back (A-21, A-34). */
typedef struct {
  double E_target[6], S_target[6];
  double tol_stag, tol_newton, tol_cg, tol_helm;
  int max_stag, max_newton, max_cg, max_helm;
  int warm_start;  /* 1: every Helmholtz PCG of the staggered loop starts from the current iterate
                      abar_j^(k) instead of 0 (fgd_solve_helmholtz_from); 0: Algorithm 2 as
                      printed (abar^(0) = 0) */
  int line_search; /* 1: Newton with residual backtracking (reading R-LS of DESIGN.md: a step that
                      does not lower the RMS of -G*(sigma - Sigma) is halved, at most 5 times);
                      0: plain Newton-Raphson */
  int stag_stall;  /* > 0: return FGD_ENOCONV (rollback) as soon as ERR has not improved on its running
                      minimum for this many consecutive staggered iterations (a diverging staggered
                      loop: the caller cuts the step back, A-34, without paying max_stag iterations);
                      0: off -- Algorithm 1 as printed (the parity setting) */
} fgd_increment;
typedef struct {
  double macro_stress[6], macro_strain[6], err;
  int stag_it, newton_it, cg_it, helm_it;
} fgd_report;
fgd_status fgd_solve_increment(fgd_ctx* ctx, const fgd_increment* inc, fgd_report* rep);

/* Field access.  which: */
enum {
  FGD_FIELD_STRESS = 0,     /* 6 comps, last mechanical solve (get only) */
  FGD_FIELD_STRAIN = 1,     /* 6 comps, committed strain eps_n */
  FGD_FIELD_EPS_P = 2,      /* 6 comps, committed plastic strain */
  FGD_FIELD_EQPS = 3,       /* 1 comp, committed equivalent plastic strain (GTN: matrix eps0p) */
  FGD_FIELD_HIST = 4,       /* 1 comp, committed history: D_n (J2), kappa_n (brittle), porosity f_n (GTN) */
  FGD_FIELD_TANGENT = 5,    /* 21 comps, packed tangent in use (get only) */
  FGD_FIELD_NONLOCAL = 16,  /* + j: 1 comp, non-local field abar_j */
  FGD_FIELD_SOURCE = 32,    /* + j: 1 comp, local source alpha_j of the last constitutive call (get only) */
  FGD_FIELD_ITERATE = 48,   /* 6 comps, current strain iterate */
  FGD_FIELD_NONLOCAL_ITERATE = 64  /* + j: 1 comp, the current (staggered-iterate) abar_j the next
                                      fgd_constitutive is frozen at; FGD_FIELD_NONLOCAL sets both it
                                      and the committed abar_j,n (GTN porosity increments, A-30) */
};
fgd_status fgd_get_field(fgd_ctx* ctx, int which, double* out);
fgd_status fgd_set_field(fgd_ctx* ctx, int which, const double* in);
fgd_status fgd_macro_stress(fgd_ctx* ctx, double out[6]);

/* Per-kernel-class device timing with CUDA events on the context stream (for roofline
 * accounting; adds one event pair per launch while enabled).  fgd_set_timing(1) clears the
 * accumulators and starts recording, fgd_set_timing(0) stops.  fgd_kernel_times synchronises
 * the stream and returns, per class, the summed duration in ms and the launch count.
 * Classes: 0 x-fwd (6 comps), 1 y-fwd (6), 2 z (6), 3 y-inv (6), 4 x-inv (6), 5 x-fwd (1),
 * 6 y-fwd (1), 7 z (1), 8 y-inv (1), 9 x-inv (1), 10 Helmholtz stencil, 11 constitutive,
 * 12 other (dots, axpy, commit, error norms), 13 communication (slab all-to-all transposes,
 * stencil z-halos and Krylov allreduces when nranks > 1; the block copies of the single-GPU slab
 * emulation), 14 x-fwd (6) of the mechanical CG iterations after the first (the steady tangent
 * launch; class 0 then holds the residual pass and the first CG iteration). */
#define FGD_NUM_KCLASS 15
fgd_status fgd_set_timing(fgd_ctx* ctx, int enable);
fgd_status fgd_kernel_times(fgd_ctx* ctx, double* ms, unsigned long long* count, int n);

#ifdef __cplusplus
}
#endif
#endif /* FGD_H */
