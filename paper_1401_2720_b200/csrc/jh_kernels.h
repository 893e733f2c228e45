// Host-side launchers and runtime helpers shared between the translation
// units of the library.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace jh {

// ---- runtime (jh_runtime.cu)
extern unsigned long long g_launches;
bool opt_overlap();   // engine 1 programmatic overlap (jh_set_overlap)
bool opt_simple();    // generic SIMT kernels only (jh_set_simple_kernels)
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
void ensure_smem(const void *fn, int bytes);
int sm_count();       // SMs of the current device
// per-kernel-class CUDA event timing (jh_profile_begin / _end)
void prof_mark(cudaStream_t st, int cls, bool after);
// TMA tensor map of a column-major FP64 matrix (rows x cols, leading
// dimension ld, 16-byte aligned columns) with boxes of box_rows x box_cols;
// rows past the end read as zeros.  false if the driver entry point is
// unavailable or the shape is not encodable.
bool make_col_tmap(CUtensorMap *map, const double *A, int64_t rows, int64_t cols, int64_t ld,
                   int box_rows, int box_cols);

// ---- DMMA/TMA Gram of every task of a p-step (jh_tiles.cu); w in {16, 32}.
bool gram_tma_ok(int w, int64_t m, int64_t ldg);
void launch_gram_tma(const double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                     int w, double *Hbuf, cudaStream_t st);

// ---- DMMA post-multiplication of every rotated task's pair columns (jh_tiles.cu).
bool update_dmma_ok(int w);
void launch_update_dmma(double *G, int64_t ldg, int64_t m, double *V, int64_t ldv, int64_t nv,
                        const int32_t *pairs, int ntask, int w, const double *Vbuf,
                        const int64_t *trot, cudaStream_t st);

// ---- K2: Cholesky + inner Jacobi per task (jh_inner5.cu); w in {16, 32, 64}.
// from_r: Hbuf holds the shortened factors R (QR peel-off) instead of Grams
// done (optional): done[task] = epoch (release) once the task's V' is written
// gblock (optional): global block-column index of each local block-column
// (the signature of a column follows its global index)
bool inner5_ok(int w);
void launch_inner5(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   bool from_r = false, int64_t *done = nullptr, int64_t epoch = 0,
                   const int32_t *gblock = nullptr);

// register-resident variant for w = 32 (jh_inner8.cu), same arguments
bool inner8_ok(int w);
void launch_inner8(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   bool from_r, int64_t *done, int64_t epoch, const int32_t *gblock);

// ---- QR peel-off shortening of every task of a p-step (jh_qr.cu): Rbuf[task] =
// R (w x w, column-major) of the pair [Gp Gq]; w even <= 32, m % w == 0
bool qr_ok(int w, int64_t m);
void launch_qr_peeloff(const double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                       int w, double *Rbuf, cudaStream_t st);

// ---- 4-cycle plan of a pivot table (jh_plan.cu): for every boundary
// (s-1, s), s = 1..steps-1, the pairs of the two p-steps form 4-cycles over
// four block-columns; plan[(s * ncyc + c) * 8 ..] = t1, t2 (tasks of p-step
// s-1), u1, u2 (tasks of p-step s), slots of u1's and u2's block-columns
int64_t cycle_plan_ints(int b, int steps);
int cycle_plan(const int32_t *outer, int b, int steps, int32_t *plan);

// ---- engine 1 update launches (jh_vpair.cu)
// one launch: the G update of one p-step (pairs / Vbuf / trot as for
// launch_update_dmma) and V-pair row slabs of up to two sources; with
// pairs_next the Grams of p-step cur_step + 1 run as trailing CTAs that wait
// for the G slabs of their block-columns (colpos: [b] task of p-step
// cur_step per block-column; gcnt: ntask epoch-tagged counters)
void launch_update_mix(double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                       const double *Vbuf, const int64_t *trot, double *V, int64_t ldv,
                       int64_t nv, const int32_t *outer, const int32_t *plan, int b, int steps,
                       int nsrc, const int *sa, const bool *second, const double *const *VpA,
                       const int64_t *const *rotA, const double *const *VpB,
                       const int64_t *const *rotB, const int *k0, const int *kstep,
                       cudaStream_t st, const int64_t *done = nullptr, int64_t epoch = 0,
                       int cur_step = -1, const int32_t *pairs_next = nullptr,
                       const int32_t *colpos = nullptr, int64_t *gcnt = nullptr,
                       double *Hgram = nullptr);
void launch_colpos(const int32_t *outer, int nsteps, int T, int b, int32_t *colpos,
                   cudaStream_t st);

}  // namespace jh
