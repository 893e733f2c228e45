// Host-side launchers shared between the translation units of the library.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace jh {

// DMMA/TMA Gram of every task of a p-step (jh_tiles.cu); w in {16, 32}.
bool gram_tma_ok(int w, int64_t m, int64_t ldg);
void launch_gram_tma(const double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                     int w, double *Hbuf, cudaStream_t st);

// DMMA post-multiplication of every rotated task's pair columns (jh_tiles.cu).
bool update_dmma_ok(int w);
void launch_update_dmma(double *G, int64_t ldg, int64_t m, double *V, int64_t ldv, int64_t nv,
                        const int32_t *pairs, int ntask, int w, const double *Vbuf,
                        const int64_t *trot, cudaStream_t st);

// Cholesky + inner Jacobi per task, specialised widths (jh_inner.cu); w in {16, 32, 64}.
bool inner3_ok(int w);
void launch_inner3(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   int task_base = 0);

// register-resident inner Jacobi, w in {16, 32} (jh_inner.cu)
bool inner4_ok(int w);
void launch_inner4(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   int task_base = 0);

// the first v3 inner Jacobi, kept for A/B timing (jh_inner5.cu)
bool inner5_ok(int w);
// from_r: Hbuf holds the shortened factors R (QR peel-off) instead of Grams
// done (optional): done[task] = epoch (release) once the task's V' is written
void launch_inner5(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   bool from_r = false, int64_t *done = nullptr, int64_t epoch = 0);

// QR peel-off shortening of every task of a p-step (jh_qr.cu): Rbuf[task] =
// R (w x w, column-major) of the pair [Gp Gq]; w even <= 32, m % w == 0
bool qr_ok(int w, int64_t m);
void launch_qr_peeloff(const double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                       int w, double *Rbuf, cudaStream_t st);

// cycle engine (jh_cycle.cu): p-steps [s_begin, s_begin + nsteps) of one
// sweep in one persistent kernel, w = 32, pivot tables with the 4-cycle
// structure of consecutive p-steps (plan from cycle_plan)
int64_t cycle_plan_ints(int b);
int cycle_plan(const int32_t *outer, int b, int32_t *plan);
bool cycle_ok(int w, int64_t m, int64_t ldg, int64_t nv, int64_t ldv);
int64_t cycle_workspace_bytes(int64_t n, int w);
void cycle_trace(void *buf, int64_t cap);
// V update of the p-step pair (sa, sa+1) (or sa alone), per cycle and row
// slab, from the tasks' V' and rotation counts (jh_vpair.cu)
void launch_vpair(double *V, int64_t ldv, int64_t nv, const int32_t *outer, const int32_t *plan,
                  int b, int sa, bool second, const double *VpA, const int64_t *rotA,
                  const double *VpB, const int64_t *rotB, cudaStream_t st);
// one launch: the G update of one p-step (pairs / Vbuf / trot as for
// launch_update_dmma) and V-pair row slabs of up to two sources (jh_vpair.cu)
void launch_update_mix(double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                       const double *Vbuf, const int64_t *trot, double *V, int64_t ldv,
                       int64_t nv, const int32_t *outer, const int32_t *plan, int b, int nsrc,
                       const int *sa, const bool *second, const double *const *VpA,
                       const int64_t *const *rotA, const double *const *VpB,
                       const int64_t *const *rotB, const int *k0, const int *kstep,
                       cudaStream_t st, const int64_t *done = nullptr, int64_t epoch = 0,
                       int cur_step = -1, double *Hnext = nullptr, double *gstate = nullptr,
                       int64_t *sflag = nullptr, const int32_t *pairs_next = nullptr,
                       const int32_t *colpos = nullptr, int64_t *gcnt = nullptr,
                       double *Hgram = nullptr);
// pairs_next != null: Gram CTAs of p-step cur_step + 1 (pairs_next) at the end
// of the grid write Hgram once the G slabs of their block-columns' tasks
// (colpos: [b] task of p-step cur_step per block-column) are done (gcnt:
// ntask epoch-tagged counters)
void launch_colpos(const int32_t *outer, int nsteps, int T, int b, int32_t *colpos,
                   cudaStream_t st);
// Hnext != null: the G items also form the Gram matrices of p-step
// cur_step + 1 into Hnext (gstate: cycles x 2 x 640 doubles of chain state,
// sflag: cycles int64, both scratch)
int launch_cycle(double *G, int64_t ldg, int64_t m, double *V, int64_t ldv, int64_t nv,
                 const int32_t *outer, const int32_t *plan, int b, int s_begin, int nsteps,
                 const int32_t *inner, int64_t n_plus, int inner_limit, double tol_c,
                 unsigned long long *counters, void *ws, cudaStream_t st);

}  // namespace jh
