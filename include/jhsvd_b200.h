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

/* Device workspace for jh_block_sweep at order n and block width w. */
int64_t jh_sweep_workspace_bytes(int64_t n, int w);

/*
 * p-steps [first_step, first_step + nsteps) of one block sweep of
 * run_block_jacobi_inplace (reference driver.py:125-200, task :153-174):
 * per task Gram (blockkernel.py:76-107), Cholesky (:110-145), inner
 * pointwise Jacobi (:278-400), and -- when the task rotated -- the
 * post-multiplication of [Gp Gq] and [Vp Vq] (:407-428).
 *   G  m x n (ld ldg), V nv x n (ld ldv) or NULL; updated in place.
 *   w  block width (shortened order), even, 2 <= w <= 64, n % w == 0.
 *   counters: uint64[4] device: [0] += rotations, [1] += proper rotations,
 *     [2] = min error key (initialise to UINT64_MAX), [3] += tasks that
 *     rotated (their pair columns were post-multiplied); key layout
 *     p-step<<38 | task<<16 | status<<13 | 1-based index, status 1 =
 *     Cholesky pivot, 2 = zero column, 3 = hyperbolic domain.
 */
int jh_block_sweep(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                   int64_t nv, int w, const int32_t *outer, int first_step, int nsteps,
                   const int32_t *inner, int64_t n_plus, int inner_limit, double tol_c,
                   void *workspace, int64_t ws_bytes, unsigned long long *counters,
                   void *stream);

/*
 * Sweep engines for pivot tables whose consecutive p-steps pair the
 * block-columns in 4-cycles (rrow, the Mantharam-Eberlein equivalent):
 * jh_cycle_plan (host) checks the structure of a host pivot table
 * int32[b-1][b/2][2] and fills plan[jh_cycle_plan_ints(b)] (return 0 =
 * usable, 1 = not usable).  jh_block_sweep2 runs the same p-steps as
 * jh_block_sweep -- bitwise the same G, V and counters -- on
 *   engine 0: the per-p-step kernels (= jh_block_sweep),
 *   engine 1: per-p-step kernels for G; V updated once per pair of p-steps
 *             on a low-priority stream (needs V, w = 32, the device plan),
 *   engine 2: the cycle engine, one persistent kernel (needs w = 32, the
 *             device plan and jh_cycle_workspace_bytes more workspace).
 * Unsupported cases fall back to engine 0.  Same reference functions as
 * jh_block_sweep (driver.py:153-190).  shortening: 0 = Gram + Cholesky
 * (blockkernel.py:76-145), 1 = QR peel-off (blockkernel.py:148-244; per
 * p-step kernels, w in {16, 32}, m % w == 0; -1000 otherwise).
 */
int64_t jh_cycle_plan_ints(int b);
int jh_cycle_plan(const int32_t *outer, int b, int32_t *plan);
int64_t jh_cycle_workspace_bytes(int64_t n, int w);
int jh_block_sweep2(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                    int64_t nv, int w, const int32_t *outer, const int32_t *plan, int engine,
                    int shortening, int first_step, int nsteps, const int32_t *inner,
                    int64_t n_plus, int inner_limit, double tol_c, void *workspace,
                    int64_t ws_bytes, unsigned long long *counters, void *stream);

/* Engine 1: 1 (default) lets the update launch start while the inner Jacobi
 * kernel still runs (programmatic dependent launch, per-task flags); 0 keeps
 * the kernels apart (per-kernel timing).  Results are identical. */
int jh_set_overlap(int on);

/* Diagnostic: per-work-item trace of the cycle engine, records {item,
 * smid, start ns, end ns} (int64) into device buf[4 + 4 cap], buf[0] =
 * count; NULL disables. */
int jh_cycle_trace(void *buf, int64_t cap);

/* gram (blockkernel.py:99-107): H = A^T A, A m x c. */
int jh_gram(const double *A, int64_t lda, int64_t m, int c, double *H, void *stream);

/* cholesky_in_place (blockkernel.py:130-145): H (c x c) overwritten with L,
 * R = L^T; *info (device int) = 0 or the 1-based bad pivot. */
int jh_cholesky(double *H, int c, double *R, int *info, void *stream);

/* qr_peeloff (blockkernel.py:223-244): R (c x c, column-major, nonnegative
 * diagonal) of A (m x c), c even <= 32, m a positive multiple of c. */
int jh_qr_peeloff(const double *A, int64_t lda, int64_t m, int c, double *R, void *stream);

/* inner_jacobi (blockkernel.py:346-400) on one c x c factor, c even <= 64.
 * R in place, V = accumulated transformation; out (device int64[5]) =
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

/* check_column_scaling (driver.py:99-112): *bad (device, init UINT64_MAX)
 * = smallest 1-based column with norm outside [mu_tilde, sqrt(nu_hat)]. */
int jh_check_scaling(const double *G, int64_t ldg, int64_t m, int64_t n,
                     unsigned long long *bad, void *stream);

/* extract_sigma + U = G / sigma (driver.py:230-238, 294-297); *bad (device,
 * init UINT64_MAX) = smallest 1-based zero column. */
int jh_sigma_u(const double *G, int64_t ldg, int64_t m, int64_t n, double *sigma, double *U,
               int64_t ldu, unsigned long long *bad, void *stream);

/* Launch accounting / per-kernel-class timing (bench.py): classes are
 * 0 Gram, 1 factor + inner Jacobi, 2 update, 3 cycle-engine sweep kernel
 * (arrays of 4).  jh_profile_end synchronizes on the recorded events. */
unsigned long long jh_launch_count(void);
int jh_profile_begin(int max_launches);
int jh_profile_end(double *ms, int64_t *count);

/* Diagnostic: DMMA (mma.sync m8n8k4 f64) vs in-order fma chain. */
int jh_probe_dmma(const double *A, const double *B, const double *C, double *Dm, double *Df,
                  int ntests, void *stream);

/* Diagnostic: sustained DMMA (kind 0) / DFMA (kind 1) issue rate; each warp
 * runs 8 independent chains for `iters` iterations. */
int jh_probe_rate(int kind, int ctas, int threads, int iters, double *out, void *stream);

/* Diagnostic: inner-Jacobi phase timing (cycles of warp 0 in dots, rotation,
 * barrier, R apply, barrier; inner p-steps; inner sweeps; tasks).  on = 1
 * enables, 0 disables; out (host uint64[8]) receives and resets them. */
int jh_inner_profile(int on, unsigned long long *out);
// The same for the default inner kernel K2 (12 counters: cycles of thread 0
// in load + Cholesky, dots, rotation + test, barrier 1, R apply + barrier 2;
// inner p-steps, inner sweeps, tasks, task cycles sum, task cycles max, setup
// cycles, Cholesky cycles; variant 6 only).
int jh_inner5_profile(int on, unsigned long long *out);

/* Diagnostic / test: branch-free division and sqrt fast paths vs the IEEE
 * operators on n operand pairs; cnt (device uint64[4]) += division
 * mismatches, division rejections, sqrt mismatches, sqrt rejections. */
int jh_probe_fastmath(const double *a, const double *b, int64_t n, unsigned long long *cnt,
                      void *stream);

/* Diagnostic: launch inner-Jacobi kernel variant 3, 4 or 5 on the Gram
 * matrices in Hbuf (A/B timing, tools/bench_inner.py). */
int jh_bench_inner(int variant, const double *Hbuf, double *Vbuf, int64_t *trot,
                   const int32_t *pairs, int ntask, int w, int64_t n_plus, const int32_t *inner,
                   int inner_limit, double tol_c, unsigned long long *counters, void *stream);

/* Diagnostic: dependent-chain latencies (cycles/op) of DFMA, DMUL, division,
 * sqrt, the rotation formula and a shared-memory load; out[6]. */
int jh_probe_latency(double *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* JHSVD_B200_H */
