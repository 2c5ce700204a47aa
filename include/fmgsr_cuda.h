/*
 * fmgsr_cuda.h -- C ABI of libfmgsr_cuda.so, the B200 (sm_100a) hot path of
 * the FMG-FAS solver with segmental refinement (arXiv 1207.6720, 1D model
 * problem).  This is the drop-in boundary for the reference's kernel-lane
 * interface; citations are into the reference package
 * (/root/reference/pkg/src/fmgsr/).
 *
 * Conventions
 *   - Every field pointer is a DEVICE pointer to a row-major [n][ld] array:
 *     cell index major, right-hand side (RHS) fastest, B <= ld active RHS
 *     columns.  B = 1, ld = 1 is the reference's single 1-D float64 field.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     asynchronous and stream-ordered; no call synchronises the device.
 *   - The library never allocates on the per-call path (the plan allocates
 *     its level workspace once, at fmgsr_plan_create).
 *   - Return 0 on success, a negative code on failure (-1 bad argument,
 *     -2 CUDA error, -3 internal); fmgsr_last_error() has the message (per
 *     host thread).  The Python layer re-raises these as ValueError /
 *     RuntimeError, mirroring the reference's argument checks.
 *   - _f64 computes in IEEE binary64 with the reference's exact operation
 *     order and no FMA contraction (bit-identical to the numba lane);
 *     _f32 is the same algorithm in binary32.
 */
#ifndef FMGSR_CUDA_H
#define FMGSR_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMGSR_ABI_VERSION 1

int fmgsr_abi_version(void);
const char* fmgsr_last_error(void);

/* ---- Kernel-lane entry points (reference _kernels_numba.py) ------------- */

/* replaces gs_sweep(u, f, inv_h2, start, stop, forward, omega),
 * _kernels_numba.py:15-36 / _kernels_numpy.py:13-35; in place on u. */
int fmgsr_gs_sweep_f64(double* u, const double* f, int64_t n, int64_t B, int64_t ld,
                       double inv_h2, int64_t start, int64_t stop, int forward, double omega,
                       void* stream);
int fmgsr_gs_sweep_f32(float* u, const float* f, int64_t n, int64_t B, int64_t ld, double inv_h2,
                       int64_t start, int64_t stop, int forward, double omega, void* stream);

/* replaces kaczmarz_sweep(u, u_coarse, start, stop, forward, proj_diag),
 * _kernels_numba.py:39-57; in place on u; uc is [n/2][ld].  Pairs are
 * disjoint, so `forward` does not change the result (kept for the ABI). */
int fmgsr_kaczmarz_sweep_f64(double* u, const double* uc, int64_t n, int64_t B, int64_t ld,
                             int64_t start, int64_t stop, int forward, double proj_diag,
                             void* stream);
int fmgsr_kaczmarz_sweep_f32(float* u, const float* uc, int64_t n, int64_t B, int64_t ld,
                             int64_t start, int64_t stop, int forward, double proj_diag,
                             void* stream);

/* replaces smooth_patches(u_in, f, inv_h2, owned_lo, owned_hi, ext_lo, ext_hi,
 * ns, omega, use_cr, u_coarse, proj_diag) -> u_out, _kernels_numba.py:60-92.
 * Patch arrays are DEVICE int64[P].  u_out must not alias u_in (the
 * reference returns a new array).  inv_h2 must equal 4^log2(n).
 * ns >= 2 needs a scratch of fmgsr_smooth_scratch_rows() rows x
 * round_up(B, 32) elements (row stride sld), and scratch_off (device
 * int64[P]) = exclusive prefix sum of the per-patch rows
 * (min(n, ext_hi + 1) - max(0, ext_lo - 1)); both may be NULL when ns == 1. */
int fmgsr_smooth_patches_f64(const double* u_in, const double* f, double* u_out, int64_t n,
                             int64_t B, int64_t ld, double inv_h2, const int64_t* owned_lo,
                             const int64_t* owned_hi, const int64_t* ext_lo,
                             const int64_t* ext_hi, int64_t P, int64_t ns, double omega,
                             int use_cr, const double* uc, double proj_diag, double* scratch,
                             const int64_t* scratch_off, int64_t sld, void* stream);
int fmgsr_smooth_patches_f32(const float* u_in, const float* f, float* u_out, int64_t n,
                             int64_t B, int64_t ld, double inv_h2, const int64_t* owned_lo,
                             const int64_t* owned_hi, const int64_t* ext_lo,
                             const int64_t* ext_hi, int64_t P, int64_t ns, double omega,
                             int use_cr, const float* uc, double proj_diag, float* scratch,
                             const int64_t* scratch_off, int64_t sld, void* stream);

/* Uniform patch geometry (owned width W | n, b-cell buffer, clamped): the
 * reference partition() (mesh.py:102-136) is W = 2, b = halo; global mode is
 * W = n, b = 0; the generalised P-patch geometry is W = max(2, n/P). */
int64_t fmgsr_smooth_scratch_rows(int64_t n, int64_t W, int64_t b);
int fmgsr_smooth_uniform_f64(const double* u_in, const double* f, double* u_out, int64_t n,
                             int64_t B, int64_t ld, int64_t W, int64_t b, int64_t ns,
                             double omega, const double* uc, double proj_diag, double* scratch,
                             int64_t sld, void* stream);
int fmgsr_smooth_uniform_f32(const float* u_in, const float* f, float* u_out, int64_t n,
                             int64_t B, int64_t ld, int64_t W, int64_t b, int64_t ns,
                             double omega, const float* uc, double proj_diag, float* scratch,
                             int64_t sld, void* stream);

/* ---- Level operators (reference stencils.py, smoothers.py) -------------- */
/* apply_operator, stencils.py:27-36: out[n] = L_k u */
int fmgsr_apply_operator_f64(const double* u, double* out, int64_t n, int64_t B, int64_t ld, void* stream);
int fmgsr_apply_operator_f32(const float* u, float* out, int64_t n, int64_t B, int64_t ld, void* stream);
/* restrict, stencils.py:39-47: out[n_fine/2] */
int fmgsr_restrict_f64(const double* u, double* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
int fmgsr_restrict_f32(const float* u, float* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
/* prolong_correction, stencils.py:50-64: out[2 n_coarse] */
int fmgsr_prolong_correction_f64(const double* c, double* out, int64_t n_coarse, int64_t B, int64_t ld, void* stream);
int fmgsr_prolong_correction_f32(const float* c, float* out, int64_t n_coarse, int64_t B, int64_t ld, void* stream);
/* prolong_fmg, stencils.py:67-105: out[2 n_coarse], n_coarse >= 4 */
int fmgsr_prolong_fmg_f64(const double* c, double* out, int64_t n_coarse, int64_t B, int64_t ld, void* stream);
int fmgsr_prolong_fmg_f32(const float* c, float* out, int64_t n_coarse, int64_t B, int64_t ld, void* stream);
/* tau_correction, stencils.py:108-116: out[n_fine/2] */
int fmgsr_tau_correction_f64(const double* u, double* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
int fmgsr_tau_correction_f32(const float* u, float* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
/* coarse_rhs, stencils.py:119-125: out = restrict(f) + tau(u) */
int fmgsr_coarse_rhs_f64(const double* f, const double* u, double* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
int fmgsr_coarse_rhs_f32(const float* f, const float* u, float* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
/* nonlinear variants (-u'' + u^3 = f; oracle/fmgsr_oracle.c defines them):
 * coarse RHS with tau of N(u) = L u + u^3, Newton coarse solve (n <= 64),
 * Newton-GS additive smoother (any ns; scratch as fmgsr_smooth_uniform) */
int fmgsr_coarse_rhs_nl_f64(const double* f, const double* u, double* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
int fmgsr_coarse_rhs_nl_f32(const float* f, const float* u, float* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
int fmgsr_direct_solve_nl_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, void* stream);
int fmgsr_direct_solve_nl_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, void* stream);
int fmgsr_smooth_uniform_nl_f64(const double* u_in, const double* f, double* u_out, int64_t n,
                                int64_t B, int64_t ld, int64_t W, int64_t b, int64_t ns,
                                double omega, const double* uc, double proj_diag,
                                double* scratch, int64_t sld, void* stream);
int fmgsr_smooth_uniform_nl_f32(const float* u_in, const float* f, float* u_out, int64_t n,
                                int64_t B, int64_t ld, int64_t W, int64_t b, int64_t ns,
                                double omega, const float* uc, double proj_diag, float* scratch,
                                int64_t sld, void* stream);
/* FAS correction update, cycles.py:120-121: out = u + P(uH - R u) */
int fmgsr_fas_correct_f64(const double* u, const double* uH, double* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
int fmgsr_fas_correct_f32(const float* u, const float* uH, float* out, int64_t n_fine, int64_t B, int64_t ld, void* stream);
/* direct_solve, smoothers.py:210-225 (LAPACK ?ptsv order), n <= 2048 */
int fmgsr_direct_solve_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, void* stream);
int fmgsr_direct_solve_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, void* stream);
/* same for any n, with a DEVICE workspace of 2n elements for the factor
 * (also backs problem.direct_fine_solve, problem.py:61-77) */
int fmgsr_direct_solve_ws_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, double* workspace, void* stream);
int fmgsr_direct_solve_ws_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, float* workspace, void* stream);
/* direct_fine_solve, problem.py:61-77: the reference's INDEPENDENT check
 * solve (scipy solve_banded((1, 1)) -> LAPACK dgbsv: banded LU with partial
 * pivoting, then dgbtrs), restated in that operation order.  DEVICE workspace
 * of 2n elements (the factor); *pivots (device int, zeroed by the caller)
 * receives the number of row swaps the pivot search would have made -- none
 * for this operator; a non-zero count means the result is not the
 * reference's and the caller must reject it. */
int fmgsr_banded_lu_solve_f64(const double* f, double* u, int64_t n, int64_t B, int64_t ld, double* workspace, int* pivots, void* stream);
int fmgsr_banded_lu_solve_f32(const float* f, float* u, int64_t n, int64_t B, int64_t ld, float* workspace, int* pivots, void* stream);

/* ---- Fused level visits and the f cascade -------------------
 * The plan's level-visit kernels, one call per visit, for a caller that drives
 * the FMG schedule itself (the reference driver cycles.py:95-222).  A visit of
 * level n = 2^k (uniform patches: owned width W | n, W even; b-cell buffer;
 * one forward Gauss-Seidel sweep, V(1,1)) is one pass over the fields:
 * prologue, additive patch smoother and, for top / down, the restriction +
 * tau epilogue.  Epilogue visits need a DEVICE workspace of
 * fmgsr_visit_workspace_bytes(n, W, B, dtype) bytes (edge records and
 * arrival counters; dtype 0 = f64, 1 = f32), zero-filled once before its
 * first use: it can then serve every later epilogue visit with the same
 * (n, W, B) -- the counters return to their start state after each visit.
 * Outputs must not alias inputs. */
int64_t fmgsr_visit_workspace_bytes(int64_t n, int64_t W, int64_t B, int32_t dtype);
/* top, cycles.py:188-197 + 101-102 (the paper's fused lines 1-5): the smoother
 * input is prolong_fmg(uH) (uH: [n/2][ld], n >= 8), no CR; then
 * uH_out = restrict(u) and fH_out = coarse_rhs(f, u) on level k-1.  u_out may
 * be NULL (an SR level: u is never stored); uH_out may be NULL.  W >= 4. */
int fmgsr_visit_top_f64(const double* uH, const double* f, double* u_out, double* uH_out,
                        double* fH_out, int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b,
                        double omega, void* work, void* stream);
int fmgsr_visit_top_f32(const float* uH, const float* f, float* u_out, float* uH_out,
                        float* fH_out, int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b,
                        double omega, void* work, void* stream);
/* down, cycles.py:99-105: u_out = S(u), uH_out = restrict(u_out) (may be NULL),
 * fH_out = coarse_rhs(f, u_out).  W >= 4. */
int fmgsr_visit_down_f64(const double* u, const double* f, double* u_out, double* uH_out,
                         double* fH_out, int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b,
                         double omega, void* work, void* stream);
int fmgsr_visit_down_f32(const float* u, const float* f, float* u_out, float* uH_out,
                         float* fH_out, int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b,
                         double omega, void* work, void* stream);
/* up, cycles.py:109-134: sr = 0: u_out = S(u + prolong_correction(uH - restrict(u)));
 * sr = 1 (an SR level): u_out = S(prolong_fmg(uH)) with the Kaczmarz CR step
 * onto uH (u is not read and may be NULL). */
int fmgsr_visit_up_f64(const double* u, const double* uH, const double* f, double* u_out,
                       int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b, int32_t sr,
                       double omega, void* stream);
int fmgsr_visit_up_f32(const float* u, const float* uH, const float* f, float* u_out,
                       int64_t n, int64_t B, int64_t ld, int64_t W, int64_t b, int32_t sr,
                       double omega, void* stream);
/* f cascade, cycles.py:178-180: f_out[j] = restrict^(j+1)(f), a DEVICE
 * [n >> (j+1)][ld] array, for j < levels; f_out is a HOST array of `levels`
 * device pointers.  Streams f once and writes every coarser level (six per
 * launch). */
int fmgsr_f_cascade_f64(const double* f, int64_t n, int64_t B, int64_t ld, int32_t levels,
                        double* const* f_out, void* stream);
int fmgsr_f_cascade_f32(const float* f, int64_t n, int64_t B, int64_t ld, int32_t levels,
                        float* const* f_out, void* stream);

/* ---- Synthetic inputs (BASELINE.json configs; not on the solve path) ---- */
/* f = sum_k coef[r][k-1] sin(k pi x), uex = sum_k coef sin(k pi x)/(k pi)^2;
 * coef is a DEVICE double[B][K]; uex may be NULL. */
int fmgsr_fourier_rhs_f64(const double* coef, int K, int64_t n, int64_t B, int64_t ld, double* f, double* uex, void* stream);
int fmgsr_fourier_rhs_f32(const double* coef, int K, int64_t n, int64_t B, int64_t ld, float* f, float* uex, void* stream);
/* nonlinear manufactured problem (config 3): u = s x(1-x)e^x, f = -u'' + u^3;
 * scale is a DEVICE double[B]; uex may be NULL. */
int fmgsr_nonlinear_rhs_f64(const double* scale, int64_t n, int64_t B, int64_t ld, double* f, double* uex, void* stream);
int fmgsr_nonlinear_rhs_f32(const double* scale, int64_t n, int64_t B, int64_t ld, float* f, float* uex, void* stream);

/* the study harness's manufactured problem (reference problem.py:23-46) for
 * one RHS on the device: f[i] = sum over odd j <= nmodes of sin(j pi x_i)/j,
 * uex[i] = sum sin(j pi x_i)/(j (j pi)^2), x_i = (i + 1/2)/n; uex may be NULL */
int fmgsr_manufactured_rhs_f64(int64_t n, int64_t nmodes, double* f, double* uex, void* stream);

/* ---- Self-test (not on the solve path) ----------------------------------
 * The nonlinear smoother divides x / J with a reciprocal of J computed ahead
 * of the Gauss-Seidel dependency chain plus two Markstein corrections.  This
 * runs that division on DEVICE arrays x[n], J[n] (q may be NULL) and ADDS to
 * the DEVICE counter *bad the number of results not bitwise equal to the IEEE
 * division. */
int fmgsr_div_check_f64(const double* x, const double* J, double* q, int64_t n, unsigned long long* bad, void* stream);
int fmgsr_div_check_f32(const float* x, const float* J, float* q, int64_t n, unsigned long long* bad, void* stream);

/* ---- Whole-solve plan: fmg_solve (cycles.py:137-222) -------------------- */
typedef struct fmgsr_plan_desc {
  int32_t m0, m;      /* hierarchy 2^m0 .. 2^m (cycles.py:39-49 limits) */
  int32_t n_sr;       /* segmental-refinement depth, 0 <= n_sr <= m-m0-1 */
  int32_t ns;         /* inner sweeps: V(ns,ns) */
  int32_t geom_mode;  /* 0 = reference halo (W=2,b), 1 = global, 2 = P patches */
  int32_t dtype;      /* 0 = f64, 1 = f32, 2 = f32 fields with f64 arithmetic */
  int64_t P;          /* patches on the finest level (geom_mode 2) */
  int64_t b;          /* buffer / halo cells */
  int64_t B;          /* right-hand sides per solve */
  int64_t ld;         /* row stride of forcing / solution (>= B) */
  double omega;       /* relaxation weight (reference: 1.0) */
  int32_t fused;      /* 1: fused level visits where eligible; 0: operator-by-operator */
  int32_t use_graph;  /* 1: capture the cycle in a CUDA graph per (in, out) pair */
  int32_t coarse;     /* on-chip coarse hierarchy (fused, ns = 1 only): -1 auto cutoff,
                         0 off, k > 0: cutoff level Lc = k - 1 (capped by the smem budget) */
  int32_t nonlinear;  /* 1: -u'' + u^3 = f (nonlinear FAS: Newton-GS, N(u) in tau, Newton
                         coarse solve); the reference is linear only */
} fmgsr_plan_desc;

typedef struct fmgsr_plan_info {
  int64_t workspace_bytes;
  int64_t launches_per_solve;   /* kernels + memsets issued by one solve */
  int64_t visits_per_solve;     /* level visits (smooths + direct solves) */
  double alg_bytes_per_solve;   /* compulsory HBM traffic model */
  double finest_visit_alg_bytes;/* algorithmic bytes of one finest-level visit */
  int32_t coarse_cutoff;        /* Lc of the on-chip coarse hierarchy, -1 if unused */
  int32_t coarse_columns;       /* RHS columns per coarse CTA */
} fmgsr_plan_info;

int fmgsr_plan_create(const fmgsr_plan_desc* desc, void** plan);
/* Debug aids (compute-sanitizer stand-ins).  FMGSR_DEBUG_POISON: every solve
 * first fills the plan's level fields, edge records and scratch with NaN, and
 * after each FMG step fills the SR levels below it with NaN (the reference's
 * debug_sr, cycles.py:161-165); a correct plan's results are unchanged.
 * Setting flags drops the captured graphs.  fmgsr_plan_check_guards: with
 * FMGSR_GUARDS=1 in the environment at plan creation every workspace array is
 * bracketed by 4 KiB guard zones; *bad_bytes = guard bytes changed since
 * (-1: the plan has no guards). */
#define FMGSR_DEBUG_POISON 1
int fmgsr_plan_set_debug(void* plan, int32_t flags);
int fmgsr_plan_check_guards(void* plan, int64_t* bad_bytes);
int fmgsr_plan_destroy(void* plan);
int fmgsr_plan_get_info(void* plan, fmgsr_plan_info* info);
/* One FMG-FAS(-SR) solve of B RHS: forcing, solution are DEVICE [2^m][ld]. */
int fmgsr_plan_solve(void* plan, const void* forcing, void* solution, void* stream);
/* Host-buffer solve (the end-to-end entry point): HOST arrays [2^m][ld_host]
 * holding chunks * B right-hand sides (B = the plan's batch, built with
 * ld == B; page-locked memory for asynchronous copies).  Chunks are pipelined:
 * H2D of chunk i+1, the solve of chunk i and D2H of chunk i-1 overlap on
 * separate streams.  Ordered after prior work on `stream`; the results are in
 * h_solution once `stream` reaches this point.  Two device buffer sets are
 * allocated on the first call. */
int fmgsr_plan_solve_host(void* plan, const void* h_forcing, void* h_solution, int64_t ld_host,
                          int64_t chunks, void* stream);
/* The same with flags.  FMGSR_HOST_INPUTS_READY: h_forcing is ready when the
 * call is made (filled by the CPU, not by pending work on `stream`), so the
 * H2D copies are not ordered after prior work on `stream` -- only after the
 * plan's previous host solve has released its staging buffers.  Consecutive
 * calls then stream: the H2D of batch k+1 overlaps the D2H of batch k.  The
 * results are still in h_solution once `stream` reaches the end of the call. */
#define FMGSR_HOST_INPUTS_READY 1
int fmgsr_plan_solve_host_ex(void* plan, const void* h_forcing, void* h_solution, int64_t ld_host,
                             int64_t chunks, int32_t flags, void* stream);
/* Functional-only output (the paper's "compute a functional of
 * u"): the same FMG cycle, but the final up visit reduces, per right-hand
 * side r, J_r = sum_i w[i][r] u[i][r] (weights: DEVICE [2^m][ld], or NULL for
 * the midpoint-rule integral h * sum_i u[i][r]) instead of writing u_m -- the
 * finest level is never stored.  functional: DEVICE array of B values (the
 * plan's dtype).  Summation order: per patch over its owned cells, then over
 * patches in order, so the result is deterministic. */
int fmgsr_plan_solve_functional(void* plan, const void* forcing, const void* weights,
                                void* functional, void* stream);
/* CUDA-event durations (ms) of the finest-level top and up visits of the most
 * recent COMPLETED solve on this plan (events recorded inside the captured
 * graph around those two kernels); -1 when the finest level ran inside the
 * on-chip coarse kernel.  Call after the solve's stream has synchronised. */
int fmgsr_plan_probe_ms(void* plan, float* ms_top, float* ms_up);
/* Same solve launched op by op (no graph) with per-visit CUDA events for
 * profiling: writes up to `cap` visit durations (ms) and their levels. */
int fmgsr_plan_solve_timed(void* plan, const void* forcing, void* solution, void* stream,
                           float* visit_ms, int32_t* visit_level, int32_t* visit_kind,
                           int64_t cap, int64_t* n_visits);

/* ---- Patch-slab sharding -----------------------------------
 * One problem split into S contiguous slabs of patches on every level above a
 * replication cutoff Lr (chosen by the plan: every level above it splits into
 * whole patches of owned width >= 4 with room for the halo); levels <= Lr are
 * solved redundantly by every shard.  Each sharded visit is followed by one
 * exchange of halo rows and slab-edge tau records with the two neighbours;
 * the visit into Lr is followed by an all-gather of the restricted level.
 * Fused ns = 1 linear path only (desc->fused = 1, ns = 1, nonlinear = 0). */
/* One shard per GPU over NCCL (libnccl.so.2 is loaded on first use).  The
 * 128-byte id comes from fmgsr_nccl_unique_id on one rank, broadcast to all.
 * The returned plan is driven by fmgsr_plan_solve with the rank's SLAB of the
 * forcing and of the solution: DEVICE [2^m / shards][ld]. */
int fmgsr_nccl_unique_id(void* id /* 128 bytes */);
int fmgsr_shard_plan_create(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                            const void* nccl_id, void** plan);
/* One shard per GPU over PEER MEMORY instead of NCCL: every rank maps its
 * peers' plan workspaces (CUDA IPC; NVLink peer access across GPUs) and pulls
 * the neighbours' halo rows and tau edge records, and every rank's chunk of the
 * replication cutoff level, straight into its own arrays; ordering by
 * per-rank device counters (release / acquire at system scope), bounded waits
 * (FMGSR_P2P_TIMEOUT_S, default 30 s; a timeout sets the status word instead
 * of hanging).  Also works with several processes on ONE device.  Create,
 * export this rank's blob (fmgsr_shard_p2p_export: *len = blob bytes; buf may
 * be NULL to query), all-gather the S blobs (rank order, any host transport),
 * import them (fmgsr_shard_p2p_import: per_rank = the blob size), then
 * fmgsr_plan_solve on the slabs as with the NCCL plan.  fmgsr_shard_p2p_status
 * synchronises the device and returns *err != 0 if any wait timed out. */
int fmgsr_shard_plan_create_p2p(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                                void** plan);
int fmgsr_shard_p2p_export(void* plan, void* buf, int64_t cap, int64_t* len);
int fmgsr_shard_p2p_import(void* plan, const void* all, int64_t per_rank);
int fmgsr_shard_p2p_status(void* plan, int32_t* err);
/* A sharded plan's own finest-level forcing buffer: *slab = the DEVICE address
 * of this rank's [rows][ld] slab inside it (the plan keeps halo rows around
 * it), *rows = 2^m / shards.  A caller that writes its forcing there and passes
 * that address as `forcing` to fmgsr_plan_solve saves the slab copy into the
 * plan (2 x the slab bytes of HBM traffic per solve); any other forcing
 * address is copied as before.  Valid until fmgsr_plan_destroy. */
int fmgsr_shard_plan_forcing_slab(void* plan, void** slab, int64_t* rows);
/* Virtual shards: all S shards of one problem on the current device, run in
 * lockstep on one stream (transfers are device copies).  forcing / solution
 * are the full DEVICE [2^m][ld] arrays; the result is bit-identical to the
 * unsharded plan. */
int fmgsr_shard_group_create(const fmgsr_plan_desc* desc, int32_t shards, void** group);
int fmgsr_shard_group_solve(void* group, const void* forcing, void* solution, void* stream);
int fmgsr_shard_group_cutoff(void* group, int32_t* cutoff, int64_t* halo_rows);
int fmgsr_shard_group_destroy(void* group);
/* One shard's plan with NO transport (no NCCL, no peer): the same kernels and
 * fix-ups as fmgsr_shard_plan_create on rank `rank` of `shards`, halos never
 * arrive.  For timing one shard's share of the work on one GPU; the result is
 * not a solve.  Destroy with fmgsr_plan_destroy. */
int fmgsr_shard_plan_create_local(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                                  void** plan);
/* The communication schedule of shard `rank` of `shards`, computed on the
 * host only (no device call; addresses are plan-relative): one record per
 * ncclSend / ncclRecv / in-place ncclAllGather / slab-edge fix-up launch, in
 * the order the plan issues them after each step.  Records beyond `cap` are
 * counted in *n but not written.  *cutoff = the replication cutoff level,
 * *halo_rows = halo rows per slab side. */
typedef struct fmgsr_comm_rec {
  int32_t step;        /* index in the plan's step list */
  int32_t step_kind;   /* FMGSR_STEP_* */
  int32_t level;       /* the step's level */
  int32_t array_level; /* level of the array moved (-1: a tau edge record) */
  int32_t pad;
  int32_t kind;        /* FMGSR_COMM_* */
  int32_t peer;      /* send / recv: the peer rank; otherwise -1 */
  int32_t tag;       /* send / recv: pairing tag (a send meets the peer's recv of equal tag) */
  int64_t bytes;     /* send / recv / fix-up: bytes; all-gather: bytes per rank */
  uint64_t addr;     /* plan-relative address of the buffer (all-gather: the full array) */
} fmgsr_comm_rec;
enum { FMGSR_COMM_SEND = 0, FMGSR_COMM_RECV = 1, FMGSR_COMM_ALLGATHER = 2, FMGSR_COMM_FIXUP = 3 };
enum { FMGSR_STEP_LOADF = 0, FMGSR_STEP_CASCADE_HI = 1, FMGSR_STEP_CASCADE_LO = 2,
       FMGSR_STEP_COARSE_FMG = 3, FMGSR_STEP_TOP = 4, FMGSR_STEP_DOWN = 5,
       FMGSR_STEP_COARSE_V = 6, FMGSR_STEP_UP = 7 };
int fmgsr_shard_schedule(const fmgsr_plan_desc* desc, int32_t shards, int32_t rank,
                         fmgsr_comm_rec* recs, int64_t cap, int64_t* n, int32_t* cutoff,
                         int64_t* halo_rows);

#ifdef __cplusplus
}
#endif

#endif /* FMGSR_CUDA_H */
