/*
 * jhsvd_b200.h -- C ABI of the B200-native blocked one-sided Jacobi (H)SVD.
 *
 * The reference (arxiv 1401.2720, package `jhsvd`) is pure Python whose
 * arithmetic kernels are numba @njit functions; it has no C ABI.  The entry
 * points below replace those kernels one for one (cited per function) plus
 * the fused sweep driver.  A Python host binds them with ctypes
 * (paper_1401_2720_b200/_lib.py); see INTEGRATION.md for the binding a
 * reference maintainer would add.
 *
 * Conventions
 *   - All matrices are FP64, column-major, DEVICE pointers owned by the
 *     caller (PyTorch allocates them); `ld*` is the column stride in
 *     elements.  Nothing here allocates device memory.
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it
 *     and nothing synchronizes, so results/counters are valid after the
 *     stream is synchronized.
 *   - Pivot tables are int32[steps][n/2][2], 0-based, in the reference's
 *     order (strategy.make_strategy), resident on the device.
 *   - Return value: 0 on success, -1000/-1001 for bad arguments/workspace,
 *     otherwise the negated cudaError_t of the failed launch.
 *   - Numeric failures are reported through device-side outputs (error key /
 *     info / out[3]) exactly where the reference raises; the host maps them
 *     to RankDeficiencyError / JDefinitenessError / UnsafeScalingError.
 */
#ifndef JHSVD_B200_H
#define JHSVD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Device workspace of jh_block_sweep at order n, block width w, for a pivot
 * table of `steps` p-steps (<= 0: the full b - 1 of one block sweep);
 * -1 for an invalid width.
 */
int64_t jh_sweep_workspace_bytes(int64_t n, int w, int64_t steps);

/*
 * 4-cycle plan of a host pivot table int32[steps][b/2][2] (0-based): 0 when
 * every pair of consecutive p-steps pairs the block-columns in 4-cycles
 * (rrow, the Mantharam-Eberlein equivalent), so engine 1 can update V once
 * per two p-steps; 1 otherwise.  plan has jh_cycle_plan_ints(b, steps)
 * entries; jh_block_sweep reads the device copy.
 */
int64_t jh_cycle_plan_ints(int b, int steps);
int jh_cycle_plan(const int32_t *outer, int b, int steps, int32_t *plan);

/*
 * p-steps [first_step, first_step + nsteps) of the pivot table `outer`
 * (device int32[outer_steps][b/2][2], 0-based block-columns, b = n/(w/2)):
 * the sweep loop body of run_block_jacobi_inplace (reference
 * driver.py:180-190) -- per task (driver.py:153-174) the Gram
 * (blockkernel.py:76-107) and Cholesky (:110-145) or, with shortening = 1,
 * the QR peel-off (:148-244; w in {16, 32}, m % w == 0), the inner
 * pointwise Jacobi (:278-400) and, when the task rotated, the
 * post-multiplication of [Gp Gq] and [Vp Vq] (:407-428).
 *   G      m x n (ld ldg), updated in place;
 *   V      nv x n (ld ldv) or NULL, updated in place;
 *   w      block width (shortened order), even, 2 <= w <= 8190, n % w == 0
 *          (above 64: one task at a time through general-purpose kernels;
 *          shortening 0 only);
 *   plan   device copy of jh_cycle_plan for `outer` or NULL;
 *   gblock NULL, or device int32[b]: the global block-column index of each
 *          local block-column (sharded solves; the J signature of a column
 *          follows its global index, column j of the factor is + iff
 *          j < n_plus);
 *   engine 0 per-p-step kernels; 1 the same G path with V updated once per
 *          two p-steps inside the G update launches (needs V, w = 32 and
 *          plan; otherwise engine 0).  Both give bitwise the same results.
 *   counters: uint64[4] device: [0] += rotations, [1] += proper rotations,
 *     [2] = min error key (initialise to UINT64_MAX), [3] += tasks that
 *     rotated; key = p-step<<38 | task<<16 | status<<13 | 1-based index,
 *     status 1 = Cholesky pivot, 2 = zero column, 3 = hyperbolic domain.
 */
int jh_block_sweep(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                   int64_t nv, int w, const int32_t *outer, int outer_steps, const int32_t *plan,
                   const int32_t *gblock, int engine, int shortening, int first_step, int nsteps,
                   const int32_t *inner, int64_t n_plus, int inner_limit, double tol_c,
                   void *workspace, int64_t ws_bytes, unsigned long long *counters,
                   void *stream);

/* Engine 1: 1 (default) lets the update launch start while the inner Jacobi
 * kernel still runs (programmatic dependent launch, per-task flags); 0 keeps
 * the kernels apart (per-kernel timing).  Results are identical. */
int jh_set_overlap(int on);

/* 1: sweeps use only the generic SIMT kernels (reference-order fma loops,
 * any even width); 0 (default): DMMA / TMA kernels where they apply.
 * Results are identical (tests compare the two). */
int jh_set_simple_kernels(int on);

/* gram (blockkernel.py:99-107): H = A^T A, A m x c. */
int jh_gram(const double *A, int64_t lda, int64_t m, int c, double *H, void *stream);

/* cholesky_in_place (blockkernel.py:130-145): H (c x c) overwritten with L,
 * R = L^T; *info (device int) = 0 or the 1-based bad pivot. */
int jh_cholesky(double *H, int c, double *R, int *info, void *stream);

/* qr_peeloff (blockkernel.py:223-244): R (c x c, column-major, nonnegative
 * diagonal) of A (m x c), c even <= 256, m a positive multiple of c (widths
 * above 32 in a global-memory kernel). */
int jh_qr_peeloff(const double *A, int64_t lda, int64_t m, int c, double *R, void *stream);

/* inner_jacobi (blockkernel.py:346-400) on one c x c factor, c even.
 * R in place, V = accumulated transformation (any even order c: up to 64
 * in shared memory, larger orders in global memory); out (device int64[5]) =
 * rotations, proper, sweeps, status (0 ok, 2 zero column, 3 hyperbolic
 * domain), 1-based bad column. */
int jh_inner_jacobi(double *R, double *V, int c, const int32_t *steps, const int8_t *signs,
                    double tol_c, int max_sweeps, int64_t *out, void *stream);

/* postmultiply (blockkernel.py:420-428): C = A B, per-entry in-order fma
 * chains over k; A m x k, B k x n2, C m x n2 (C must not alias A or B). */
int jh_gemm(const double *A, int64_t lda, int64_t m, int k, const double *B, int64_t ldb,
            int n2, double *C, int64_t ldc, void *stream);

/* solve_for_v back substitution (driver.py:203-211): R out = W. */
int jh_back_substitute(const double *R, int n, const double *W, int nc, double *out,
                       void *stream);

/* robustnorm.safe_bounds (robustnorm.py:90-113), host function. */
void jh_safe_bounds(int64_t n, double *mu_tilde, double *nu_hat);

/* robustnorm.norm2 per column (robustnorm.py:295-334): ||G[:, i]|| =
 * s[i] / 2**js[i]; js, s device arrays of length n. */
int jh_column_norms(const double *G, int64_t ldg, int64_t m, int64_t n, int64_t *js, double *s,
                    void *stream);

/* robustnorm.sum_squares / norm2 (robustnorm.py:324-334) of the n columns of
 * G (m x n, ld ldg) with the reference's chunk (leaf length) and
 * force_scaled options: sum of squares vsq * 2**jsq in common form and the
 * norm s / 2**js, device arrays of n (each may be NULL). */
int jh_robust_norms(const double *G, int64_t ldg, int64_t m, int64_t n, int chunk,
                    int force_scaled, int64_t *jsq, double *vsq, int64_t *js, double *s,
                    void *stream);

/* Host DRDSSQ helpers (robustnorm.py:116-162): common_form, add_scaled,
 * scale_exponent (up = 1: smallest j with 2**j f >= t; 0: largest with <=). */
void jh_common_form(int64_t j, double v, int64_t *jo, double *vo);
void jh_add_scaled(int64_t ja, double va, int64_t jb, double vb, int64_t *jo, double *vo);
int jh_scale_exponent(double f, double t, int up);

/* _rotation_core (rotation.py:90-102) of n pivot Grams: in (device, n x 3
 * h_pp, h_qq, h_pq), t (device, +1 trig / -1 hyperbolic), out (device,
 * n x 3: cs, tn, 1 ok / 0 hyperbolic domain failure). */
int jh_rotations(const double *in, const double *t, int64_t n, double *out, void *stream);

/* check_column_scaling (driver.py:99-112): *bad (device, init UINT64_MAX)
 * = smallest 1-based column with norm outside [mu_tilde, sqrt(nu_hat)]. */
int jh_check_scaling(const double *G, int64_t ldg, int64_t m, int64_t n,
                     unsigned long long *bad, void *stream);

/* extract_sigma + U = G / sigma (driver.py:230-238, 294-297); *bad (device,
 * init UINT64_MAX) = smallest 1-based zero column. */
int jh_sigma_u(const double *G, int64_t ldg, int64_t m, int64_t n, double *sigma, double *U,
               int64_t ldu, unsigned long long *bad, void *stream);

/*
 * Synthetic input of the BASELINE workloads (not a reference function; the
 * reference builds its inputs with numpy in testgen.py:82-133):
 * G (m x n, ld ldg) = Q [diag(sigma); 0] W^T with Q, W random Givens
 * butterflies (`passes` rounds of log2 layers) and, when n_plus = n/2, one
 * J-orthogonal hyperbolic layer (|tanh| <= tanh_max) per round; bitwise
 * equal to its host twin oracle/gen_butterfly.c.  m, n powers of two,
 * m >= n, n_plus in {n, n/2}; sigma is a device array of n values.
 * Workspace: jh_gen_workspace_bytes (-1 = unsupported shape).
 */
int64_t jh_gen_workspace_bytes(int64_t m, int64_t n, int64_t n_plus, int passes);
int jh_gen_butterfly(double *G, int64_t ldg, int64_t m, int64_t n, const double *sigma,
                     int64_t n_plus, unsigned long long seed, int passes, double tanh_max,
                     void *workspace, int64_t ws_bytes, void *stream);

/* Launch accounting / per-kernel-class timing (bench.py): classes are
 * 0 Gram, 1 factor + inner Jacobi, 2 update, 3 V-only update launches
 * (arrays of 4).  jh_profile_end synchronizes on the recorded events. */
unsigned long long jh_launch_count(void);
int jh_profile_begin(int max_launches);
int jh_profile_end(double *ms, int64_t *count);

#ifdef __cplusplus
}
#endif

#endif /* JHSVD_B200_H */
