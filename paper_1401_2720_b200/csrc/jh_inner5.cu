// K2, the factor + inner Jacobi kernel: one CTA of 4 warps per task
// (jh_inner5.cuh): warp-0 Cholesky in the reference element order
// (blockkernel.py:110-127), then the inner sweeps -- the pairs' dot products
// and rotation parameters by w/2 lanes of warp 0, R applied by all threads
// one pair at a time, V' applied by warps 1-3 one inner p-step behind
// (blockkernel.py:278-334).  For w = 32 and many tasks per SM the
// register-resident variant (jh_inner8.cu) runs instead.
#include "jh_inner5.cuh"
#include "jh_kernels.h"

namespace jh {

template <int W>
__global__ void __launch_bounds__(InnerCfg5<W>::NTH, 4)
k_factor_inner5(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                int64_t n_plus, const int32_t *__restrict__ inner, int inner_limit,
                double tol_c, unsigned long long *counters, int pstep, bool from_r,
                int64_t *done, int64_t epoch, const int32_t *__restrict__ gblock) {
  extern __shared__ __align__(16) unsigned char smraw[];
  // a programmatically dependent launch (the engine-1 update) may start now:
  // it waits for each task's `done` flag instead of for this whole grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int task = blockIdx.x;
  inner5_task<W, InnerCfg5<W>::NTH>(smraw, Hbuf + (size_t)task * W * W, Vbuf + (size_t)task * W * W,
                                    pairs[2 * task], pairs[2 * task + 1], n_plus, inner,
                                    inner_limit, tol_c, counters, pstep, task, &task_rot[task],
                                    from_r, gblock);
  if (done) {
    // done[task] = epoch; then, in completion order, ready list slot k =
    // this task (done + ntask: int64 count, then ntask slots of (epoch << 24
    // | task)) so that the update starts with the tasks that finish first
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(done + task), "l"(epoch) : "memory");
      int64_t *rl = done + gridDim.x;
      const unsigned long long k = atomicAdd((unsigned long long *)rl, 1ull);
      asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(rl + 1 + k),
                   "l"((epoch << 24) | task) : "memory");
    }
  }
}

bool inner5_ok(int w) { return w == 16 || w == 32 || w == 64; }

template <int W>
static void launch_inner5_t(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                            int ntask, int64_t n_plus, const int32_t *inner, int inner_limit,
                            double tol_c, unsigned long long *counters, int pstep,
                            cudaStream_t st, bool from_r, int64_t *done, int64_t epoch,
                            const int32_t *gblock) {
  const size_t smem = sizeof(InnerSmem5<W>);
  ensure_smem((const void *)k_factor_inner5<W>, (int)smem);
  k_factor_inner5<W><<<ntask, InnerCfg5<W>::NTH, smem, st>>>(Hbuf, Vbuf, trot, pairs, n_plus,
                                                             inner, inner_limit, tol_c, counters,
                                                             pstep, from_r, done, epoch, gblock);
}

void launch_inner5(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   bool from_r, int64_t *done, int64_t epoch, const int32_t *gblock) {
#ifndef JH_INNER8
#define JH_INNER8 1
#endif
  // the register-resident kernel, with its V' rotations one inner p-step
  // late (issued under the next rotation's division / square-root chain),
  // wins at every task count: 512 tasks 1.763 vs 1.783 ms per p-step, worker
  // of the sharded solve at 256 / 128 / 64 tasks 0.994 / 0.644 / 0.458 vs
  // 1.006 / 0.648 / 0.465 ms against the shared-memory kernel
  // (tools/ab_pstep.py, tools/worker_profile.py; profiles/r02/README.md)
#ifndef JH_INNER8_PER_SM
#define JH_INNER8_PER_SM 0
#endif
  if (JH_INNER8 && inner8_ok(w) && ntask > JH_INNER8_PER_SM * sm_count()) {
    launch_inner8(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c, counters,
                  pstep, st, from_r, done, epoch, gblock);
    return;
  }
  if (w == 16)
    launch_inner5_t<16>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                        counters, pstep, st, from_r, done, epoch, gblock);
  else if (w == 32)
    launch_inner5_t<32>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                        counters, pstep, st, from_r, done, epoch, gblock);
  else
    launch_inner5_t<64>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                        counters, pstep, st, from_r, done, epoch, gblock);
}

}  // namespace jh
