// K2, the default inner Jacobi kernel (variant 5; fastest at n = 16384 in
// tools/bench_inner.py): one CTA of 4 warps per task, pairs' dot products
// by w/2 lanes of warp 0, R applied by all threads one pair at a time, V
// applied by warps 1-3 one inner p-step behind (jh_inner5.cuh).  Variants 3
// and 4 (jh_inner.cu) give bitwise the same results and stay for A/B runs
// (JHSVD_INNER=3/4).
#include "jh_inner5.cuh"
#include "jh_inner6.cuh"
#include "jh_inner7.cuh"
#include "jh_kernels.h"

namespace jh {

#ifndef JH_I5_MINB
#define JH_I5_MINB 4
#endif
template <int W>
__global__ void __launch_bounds__(InnerCfg5<W>::NTH, JH_I5_MINB)
k_factor_inner5(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                int64_t n_plus, const int32_t *__restrict__ inner, int inner_limit,
                double tol_c, unsigned long long *counters, int pstep, bool from_r,
                int64_t *done, int64_t epoch) {
  extern __shared__ __align__(16) unsigned char smraw[];
  // a programmatically dependent launch (the engine-1 update) may start now:
  // it waits for each task's `done` flag instead of for this whole grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int task = blockIdx.x;
  inner5_task<W, InnerCfg5<W>::NTH>(smraw, Hbuf + (size_t)task * W * W, Vbuf + (size_t)task * W * W,
                                    pairs[2 * task], pairs[2 * task + 1], n_plus, inner,
                                    inner_limit, tol_c, counters, pstep, task, &task_rot[task],
                                    from_r);
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

// Variant 6 (jh_inner6.cuh): the same task with warp 0 alone on the serial
// chain (w <= 32, opt-in: JHSVD_I6=1; slower than variant 5 on B200, the
// R columns then cost one warp's FP64 issue instead of four warps').
template <int W>
__global__ void __launch_bounds__(InnerCfg5<W>::NTH, 4)
k_factor_inner6(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                int64_t n_plus, const int32_t *__restrict__ inner, int inner_limit,
                double tol_c, unsigned long long *counters, int pstep, bool from_r,
                int64_t *done, int64_t epoch) {
  extern __shared__ __align__(16) unsigned char smraw[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int task = blockIdx.x;
  inner6_task<W, InnerCfg5<W>::NTH>(smraw, Hbuf + (size_t)task * W * W, Vbuf + (size_t)task * W * W,
                                    pairs[2 * task], pairs[2 * task + 1], n_plus, inner,
                                    inner_limit, tol_c, counters, pstep, task, &task_rot[task],
                                    from_r);
  if (done) {
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

// Variant 7 (jh_inner7.cuh): one barrier per inner p-step, stored-R and V
// updates off warp 0's chain (w <= 32; opt-in JHSVD_I7=1: bitwise equal but
// slower, 368 vs 254 us per launch at n = 16384 -- the on-the-fly columns and
// the per-row shuffles lengthen warp 0's chain more than the barrier saves).
template <int W>
__global__ void __launch_bounds__(InnerCfg5<W>::NTH, 4)
k_factor_inner7(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                int64_t n_plus, const int32_t *__restrict__ inner, int inner_limit,
                double tol_c, unsigned long long *counters, int pstep, bool from_r,
                int64_t *done, int64_t epoch) {
  extern __shared__ __align__(16) unsigned char smraw[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int task = blockIdx.x;
  inner7_task<W, InnerCfg5<W>::NTH>(smraw, Hbuf + (size_t)task * W * W, Vbuf + (size_t)task * W * W,
                                    pairs[2 * task], pairs[2 * task + 1], n_plus, inner,
                                    inner_limit, tol_c, counters, pstep, task, &task_rot[task],
                                    from_r);
  if (done) {
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

static bool use_inner7(int w) {
  static const bool on = [] {
    const char *e = getenv("JHSVD_I7");
    return e && e[0] == '1';
  }();
  return on && w <= 32;
}

static bool use_inner6(int w) {
  static const bool on = [] {
    const char *e = getenv("JHSVD_I6");
    return e && e[0] == '1';
  }();
  return on && w <= 32;
}

template <int W>
static void launch_inner5_t(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                           int ntask, int64_t n_plus, const int32_t *inner, int inner_limit,
                           double tol_c, unsigned long long *counters, int pstep,
                           cudaStream_t st, bool from_r, int64_t *done, int64_t epoch) {
  if constexpr (W <= 32) {
    if (use_inner7(W) && !use_inner6(W)) {
      const size_t smem7 = sizeof(InnerSmem7<W>);
      static bool attr7 = false;
      if (!attr7) {
        cudaFuncSetAttribute(k_factor_inner7<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem7);
        attr7 = true;
      }
      k_factor_inner7<W><<<ntask, InnerCfg5<W>::NTH, smem7, st>>>(
          Hbuf, Vbuf, trot, pairs, n_plus, inner, inner_limit, tol_c, counters, pstep, from_r,
          done, epoch);
      return;
    }
    if (use_inner6(W)) {
      const size_t smem6 = sizeof(InnerSmem6<W>);
      static bool attr6 = false;
      if (!attr6) {
        cudaFuncSetAttribute(k_factor_inner6<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem6);
        attr6 = true;
      }
      k_factor_inner6<W><<<ntask, InnerCfg5<W>::NTH, smem6, st>>>(
          Hbuf, Vbuf, trot, pairs, n_plus, inner, inner_limit, tol_c, counters, pstep, from_r,
          done, epoch);
      return;
    }
  }
  const size_t smem = sizeof(InnerSmem5<W>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_factor_inner5<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  k_factor_inner5<W><<<ntask, InnerCfg5<W>::NTH, smem, st>>>(Hbuf, Vbuf, trot, pairs, n_plus, inner,
                                                           inner_limit, tol_c, counters, pstep,
                                                           from_r, done, epoch);
}

void launch_inner5(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   bool from_r, int64_t *done, int64_t epoch) {
  if (w == 16)
    launch_inner5_t<16>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                       counters, pstep, st, from_r, done, epoch);
  else if (w == 32)
    launch_inner5_t<32>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                       counters, pstep, st, from_r, done, epoch);
  else
    launch_inner5_t<64>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                       counters, pstep, st, from_r, done, epoch);
}

}  // namespace jh

// A/B harness (tools/bench_inner.py): run one inner-Jacobi kernel variant on
// the Gram matrices already in Hbuf.  variant 3 / 4 / 5.
extern "C" int jh_bench_inner(int variant, const double *Hbuf, double *Vbuf, int64_t *trot,
                              const int32_t *pairs, int ntask, int w, int64_t n_plus,
                              const int32_t *inner, int inner_limit, double tol_c,
                              unsigned long long *counters, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (variant == 3 && jh::inner3_ok(w))
    jh::launch_inner3(Hbuf, Vbuf, trot, pairs, ntask, w, n_plus, inner, inner_limit, tol_c,
                      counters, 0, st);
  else if (variant == 4 && jh::inner4_ok(w))
    jh::launch_inner4(Hbuf, Vbuf, trot, pairs, ntask, w, n_plus, inner, inner_limit, tol_c,
                      counters, 0, st);
  else if ((variant == 5 || variant == 6) && jh::inner5_ok(w))
    jh::launch_inner5(Hbuf, Vbuf, trot, pairs, ntask, w, n_plus, inner, inner_limit, tol_c,
                      counters, 0, st);
  else
    return -1000;
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// Enable (1) / disable (0) the phase timing of K2 (g_i5 in jh_inner5.cuh);
// when out != NULL, copies the 12 counters to host memory and resets them.
extern "C" int jh_inner5_profile(int on, unsigned long long *out) {
  cudaDeviceSynchronize();
  if (out) {
    cudaMemcpyFromSymbol(out, jh::g_i5, sizeof(unsigned long long) * 12);
    unsigned long long z[12] = {};
    cudaMemcpyToSymbol(jh::g_i5, z, sizeof(z));
  }
  cudaMemcpyToSymbol(jh::g_i5_on, &on, sizeof(int));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}
