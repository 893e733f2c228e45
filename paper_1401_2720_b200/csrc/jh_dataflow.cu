// Dataflow execution of a block sweep: one persistent kernel runs every task
// of every p-step as soon as its inputs are ready, instead of one launch per
// kernel per p-step with a device-wide barrier between them.
//
// Work items, executed by CTAs of 4 warps pulling from a device work queue:
//   G(s, t)     Gram of task t of p-step s          (K1, TMA ring + DMMA)
//   I(s, t)     Cholesky + inner Jacobi of the task (K2, the v5 design)
//   U(s, t, k)  post-multiplication of row slab k of the task's G / V pair
//               columns by V' (K3, TMA ring + DMMA)
// Dependencies (reference order of the sweep, driver.py:180-190):
//   I(s, t) after G(s, t); U(s, t, *) after I(s, t) (none when the task did
//   not rotate, driver.py:165); G(s+1, t') after the two tasks of p-step s
//   that own t''s block-columns are complete.
// A task's arithmetic is exactly the three-kernel path's (same device code),
// so results are bitwise identical; only the schedule changes: latency-bound
// inner phases and per-task Gram chains overlap the streaming updates of
// other tasks and the next p-step's Grams.
//
// Queue: a ring of (item, sequence) slots; producers reserve an index with
// atomicAdd(tail) and publish the item with a release store of the index;
// consumers reserve with atomicAdd(head) and spin until the slot carries
// their index.  An item is pushed only after everything it reads is written
// and fenced (gpu scope); consumers fence.proxy.async before their TMA reads
// of columns written by other CTAs.  Deadlock-free: a CTA only waits for an
// item to be published, and every published item's dependencies are done.
#include "jh_gram.cuh"
#include "jh_inner5.cuh"
#include "jh_kernels.h"

#include <cstdlib>

namespace jh {

constexpr int kDfThreads = 128;
constexpr int kQCap = 1 << 17;        // queue slots
constexpr int kDfSlab = 2048;         // rows per update item
constexpr int kUpRows = 48;           // rows per update chunk (3 consumer warps x 16)
constexpr int kUpLd = kUpRows + 4;    // == 4 (mod 16): conflict-free fragment loads
constexpr int kUpStages = 4;

enum ItemType : int { kItemG = 0, kItemI = 1, kItemU = 2 };

__host__ __device__ inline long long item_pack(int type, int s, int t, int k) {
  return ((long long)type << 60) | ((long long)s << 40) | ((long long)t << 16) | (long long)k;
}

struct DfSched {
  unsigned long long head, tail;
  int done_tasks, abort;
};

struct DfArgs {
  double *G;
  int64_t ldg, m;
  double *V;
  int64_t ldv, nv;
  const int32_t *outer;   // [steps][T][2]
  const int32_t *colpos;  // [steps][b]: task holding block-column c
  const int32_t *inner;
  int64_t n_plus;
  int inner_limit;
  double tol_c;
  unsigned long long *counters;
  int T, b, s_begin, s_end, nslab_g, nslab_v;
  double *Hs;       // [steps][T][w][w]
  double *Vs;       // [steps][T][w][w]
  int64_t *rot;     // [steps][T]
  int *ready;       // [steps][T]
  int *slabs;       // [steps][T]
  DfSched *sched;
  long long *qitem;
  long long *qseq;
};

template <int W>
struct DfSmem {
  union {
    double gram_ring[kStages][W][kLd];
    InnerSmem5<W> inner;
    double up_ring[kUpStages][W][kUpLd];
  } u;
  uint64_t full[kUpStages > kStages ? kUpStages : kStages];
  uint64_t empty[kUpStages > kStages ? kUpStages : kStages];
  long long item;
  long long irot;
};

__device__ __forceinline__ long long ld_acquire_s64(const long long *p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_s64(long long *p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_s32(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void mbar_inval(uint64_t *bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// thread 0: publish items (reserve `cnt` consecutive queue indices)
__device__ void df_push(const DfArgs &a, const long long *items, int cnt) {
  const unsigned long long j0 = atomicAdd(&a.sched->tail, (unsigned long long)cnt);
  for (int i = 0; i < cnt; i++) {
    const unsigned long long j = j0 + i;
    const size_t slot = j & (kQCap - 1);
    a.qitem[slot] = items[i];
    __threadfence();
    st_release_s64(&a.qseq[slot], (long long)j);
  }
}

// thread 0: a task is complete -- count it and release the next p-step's
// Grams that were waiting for its block-columns
__device__ void df_task_done(const DfArgs &a, int s, int t) {
  __threadfence();
  atomicAdd(&a.sched->done_tasks, 1);
  if (s + 1 >= a.s_end) return;
  const int32_t *pr = a.outer + ((int64_t)s * a.T + t) * 2;
  for (int j = 0; j < 2; j++) {
    const int c = pr[j];
    const int tn = a.colpos[(int64_t)(s + 1) * a.b + c];
    int *rd = &a.ready[(int64_t)(s + 1) * a.T + tn];
    if (atomicAdd(rd, 1) == 1) {
      __threadfence();
      const long long it = item_pack(kItemG, s + 1, tn, 0);
      df_push(a, &it, 1);
    }
  }
}

template <int W>
__device__ void df_gram(DfSmem<W> &S, const DfArgs &a, int s, int t) {
  constexpr int NW = 2, BW = W / 2, MY = GramTiles<W, NW>::MY;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int32_t *pr = a.outer + ((int64_t)s * a.T + t) * 2;
  const int p = pr[0], q = pr[1];
  const int64_t m = a.m, ldg = a.ldg;
  const int64_t nchunk = cdiv(m, kRch);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; i++) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    fence_proxy_async_global();
    for (int64_t c = 0; c < nchunk; c++) {
      const int st = (int)(c % kStages);
      if (c >= kStages) mbar_wait(&S.empty[st], (uint32_t)(((c / kStages) - 1) & 1));
      const int64_t r0 = c * kRch;
      const uint32_t bytes = (uint32_t)min64(kRch, m - r0) * 8u;
      if (lane == 0) mbar_expect_tx(&S.full[st], bytes * W);
      __syncwarp();
      for (int j = lane; j < W; j += 32) {
        const int64_t col = j < BW ? (int64_t)p * BW + j : (int64_t)q * BW + (j - BW);
        bulk_g2s(&S.u.gram_ring[st][j][0], a.G + col * ldg + r0, bytes, &S.full[st]);
      }
    }
  } else if (warp <= NW) {
    const int cw = warp - 1;
    double acc[MY][2];
#pragma unroll
    for (int i = 0; i < MY; i++) acc[i][0] = acc[i][1] = 0.0;
    for (int64_t c = 0; c < nchunk; c++) {
      const int st = (int)(c % kStages);
      mbar_wait(&S.full[st], (uint32_t)((c / kStages) & 1));
      const double *buf = &S.u.gram_ring[st][0][0] + (size_t)g * kLd + tq;
      const int nr = (int)min64(kRch, m - c * kRch);
      if (cw == 0)
        gram_chunk<W, NW, 0>(buf, nr, acc, tq);
      else
        gram_chunk<W, NW, 1>(buf, nr, acc, tq);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[st]);
    }
    double *H = a.Hs + ((int64_t)s * a.T + t) * W * W;
    if (cw == 0)
      gram_store<W, NW, 0>(H, acc, g, tq);
    else
      gram_store<W, NW, 1>(H, acc, g, tq);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; i++) {
      mbar_inval(&S.full[i]);
      mbar_inval(&S.empty[i]);
    }
    __threadfence();
    const long long it = item_pack(kItemI, s, t, 0);
    df_push(a, &it, 1);
  }
}

template <int W>
__device__ void df_inner(DfSmem<W> &S, const DfArgs &a, int s, int t) {
  const int32_t *pr = a.outer + ((int64_t)s * a.T + t) * 2;
  const int64_t idx = (int64_t)s * a.T + t;
  const long long rot = inner5_task<W, kDfThreads>(
      reinterpret_cast<unsigned char *>(&S.u.inner), a.Hs + idx * W * W, a.Vs + idx * W * W,
      pr[0], pr[1], a.n_plus, a.inner, a.inner_limit, a.tol_c, a.counters, s, t, &a.rot[idx]);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (rot < 0) {
      atomicExch(&a.sched->abort, 1);
    } else if (rot == 0) {
      df_task_done(a, s, t);
    } else {
      __threadfence();
      const int K = a.nslab_g + a.nslab_v;
      long long items[64];
      for (int k0 = 0; k0 < K; k0 += 64) {
        const int cnt = K - k0 < 64 ? K - k0 : 64;
        for (int i = 0; i < cnt; i++) items[i] = item_pack(kItemU, s, t, k0 + i);
        df_push(a, items, cnt);
      }
    }
  }
}

template <int W>
__device__ void df_update(DfSmem<W> &S, const DfArgs &a, int s, int t, int k) {
  constexpr int NT = W / 8, NK = W / 4, BW = W / 2, NCONS = 3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int32_t *pr = a.outer + ((int64_t)s * a.T + t) * 2;
  const int p = pr[0], q = pr[1];
  double *A;
  int64_t ld, rows, s0;
  if (k < a.nslab_g) {
    A = a.G; ld = a.ldg; rows = a.m; s0 = (int64_t)k * kDfSlab;
  } else {
    A = a.V; ld = a.ldv; rows = a.nv; s0 = (int64_t)(k - a.nslab_g) * kDfSlab;
  }
  const int64_t s1 = min64(s0 + kDfSlab, rows);
  const int nchunk = (int)cdiv(s1 - s0, kUpRows);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kUpStages; i++) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], NCONS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    fence_proxy_async_global();
    for (int c = 0; c < nchunk; c++) {
      const int st = c % kUpStages;
      if (c >= kUpStages) mbar_wait(&S.empty[st], (uint32_t)(((c / kUpStages) - 1) & 1));
      const int64_t r0 = s0 + (int64_t)c * kUpRows;
      const uint32_t bytes = (uint32_t)min64(kUpRows, s1 - r0) * 8u;
      if (lane == 0) mbar_expect_tx(&S.full[st], bytes * W);
      __syncwarp();
      for (int j = lane; j < W; j += 32) {
        const int64_t col = j < BW ? (int64_t)p * BW + j : (int64_t)q * BW + (j - BW);
        bulk_g2s(&S.u.up_ring[st][j][0], A + col * ld + r0, bytes, &S.full[st]);
      }
    }
  } else {
    const int cw = warp - 1;
    const double *Vt = a.Vs + ((int64_t)s * a.T + t) * W * W;
    double bf[NK][NT];
#pragma unroll
    for (int kk = 0; kk < NK; kk++)
#pragma unroll
      for (int Y = 0; Y < NT; Y++) bf[kk][Y] = Vt[(8 * Y + g) * W + 4 * kk + tq];
    double *pout = A + ((int64_t)p * BW + 2 * tq) * ld;
    double *qout = A + ((int64_t)q * BW + 2 * tq) * ld;
    for (int c = 0; c < nchunk; c++) {
      const int st = c % kUpStages;
      mbar_wait(&S.full[st], (uint32_t)((c / kUpStages) & 1));
      const int64_t r0 = s0 + (int64_t)c * kUpRows;
#pragma unroll
      for (int rb = 0; rb < 2; rb++) {
        const int rl = cw * 16 + rb * 8;
        double av[NK];
#pragma unroll
        for (int kk = 0; kk < NK; kk++) av[kk] = S.u.up_ring[st][4 * kk + tq][rl + g];
        double acc[NT][2];
#pragma unroll
        for (int Y = 0; Y < NT; Y++) acc[Y][0] = acc[Y][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < NK; kk++)
#pragma unroll
          for (int Y = 0; Y < NT; Y++) dmma(acc[Y][0], acc[Y][1], av[kk], bf[kk][Y]);
        const int64_t row = r0 + rl + g;
        if (row < s1) {
#pragma unroll
          for (int Y = 0; Y < NT; Y++)
#pragma unroll
            for (int j = 0; j < 2; j++) {
              double *dst = Y < NT / 2 ? pout + (int64_t)(8 * Y + j) * ld
                                       : qout + (int64_t)(8 * Y + j - BW) * ld;
              st_f64(dst + row, acc[Y][j]);
            }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[st]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kUpStages; i++) {
      mbar_inval(&S.full[i]);
      mbar_inval(&S.empty[i]);
    }
    __threadfence();
    const int K = a.nslab_g + a.nslab_v;
    if (atomicAdd(&a.slabs[(int64_t)s * a.T + t], 1) == K - 1) df_task_done(a, s, t);
  }
}

template <int W>
__global__ void __launch_bounds__(kDfThreads)
k_dataflow(DfArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  DfSmem<W> &S = *reinterpret_cast<DfSmem<W> *>(smraw);
  const int total = a.T * (a.s_end - a.s_begin);
  for (;;) {
    if (threadIdx.x == 0) {
      long long item = -1;
      const unsigned long long j = atomicAdd(&a.sched->head, 1ull);
      const size_t slot = j & (kQCap - 1);
      for (;;) {
        if (ld_acquire_s64(&a.qseq[slot]) == (long long)j) {
          item = a.qitem[slot];
          break;
        }
        if (ld_acquire_s32(&a.sched->done_tasks) >= total ||
            ld_acquire_s32(&a.sched->abort) != 0)
          break;
        __nanosleep(64);
      }
      S.item = item;
    }
    __syncthreads();
    const long long item = S.item;
    __syncthreads();
    if (item < 0) return;
    const int type = (int)(item >> 60), s = (int)((item >> 40) & 0xfffff),
              t = (int)((item >> 16) & 0xffffff), k = (int)(item & 0xffff);
    if (type == kItemG)
      df_gram<W>(S, a, s, t);
    else if (type == kItemI)
      df_inner<W>(S, a, s, t);
    else
      df_update<W>(S, a, s, t, k);
    __syncthreads();
  }
}

__global__ void k_dataflow_init(DfArgs a) {
  // queue slots unpublished, first p-step's Grams published
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = tid; i < kQCap; i += gridDim.x * blockDim.x)
    if (i >= a.T) a.qseq[i] = -1;
  if (tid == 0) {
    a.sched->head = 0;
    a.sched->tail = (unsigned long long)a.T;
    a.sched->done_tasks = 0;
    a.sched->abort = 0;
  }
  for (int t = tid; t < a.T; t += gridDim.x * blockDim.x) {
    a.qitem[t] = item_pack(kItemG, a.s_begin, t, 0);
    a.qseq[t] = t;
  }
}

// colpos[s][c] = task of p-step s that holds block-column c
__global__ void k_colpos(const int32_t *__restrict__ outer, int nsteps, int T, int b,
                         int32_t *__restrict__ colpos) {
  const int64_t n = (int64_t)nsteps * T;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / T;
    const int t = (int)(i - s * T);
    colpos[s * b + outer[2 * i]] = t;
    colpos[s * b + outer[2 * i + 1]] = t;
  }
}

bool dataflow_ok(int w, int64_t m, int64_t ldg, int64_t nv, int64_t ldv) {
  static const char *e = getenv("JHSVD_DATAFLOW");
  if (e && e[0] == '0') return false;
  return (w == 16 || w == 32) && m % 2 == 0 && ldg % 2 == 0 && nv % 2 == 0 && ldv % 2 == 0;
}

int64_t dataflow_workspace_bytes(int64_t n, int w, int nsteps_total) {
  const int64_t T = n / w, b = n / (w / 2);
  int64_t bytes = 0;
  bytes += (int64_t)nsteps_total * T * w * w * 8 * 2;    // Hs, Vs
  bytes += (int64_t)nsteps_total * T * 8;                // rot
  bytes += (int64_t)nsteps_total * T * 4 * 2;            // ready, slabs
  bytes += (int64_t)nsteps_total * b * 4;                // colpos
  bytes += 256 + (int64_t)kQCap * 16;                    // sched, queue
  return bytes + 4096;
}

template <int W>
static int launch_dataflow_t(DfArgs a, cudaStream_t st) {
  const size_t smem = sizeof(DfSmem<W>);
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_dataflow<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dataflow<W>, kDfThreads, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = (per_sm > 0 ? per_sm : 1) * sms;
  }
  k_dataflow_init<<<64, 256, 0, st>>>(a);
  k_dataflow<W><<<grid, kDfThreads, smem, st>>>(a);
  return 0;
}

// Carves the dataflow workspace (after the per-step scratch of the regular
// path) and launches one persistent kernel for p-steps [s_begin, s_end).
int launch_dataflow(double *G, int64_t ldg, int64_t m, double *V, int64_t ldv, int64_t nv, int w,
                    const int32_t *outer, int s_begin, int s_end,
                    int nsteps_total, const int32_t *inner, int64_t n_plus, int inner_limit,
                    double tol_c, unsigned long long *counters, void *ws, int64_t n,
                    cudaStream_t st) {
  DfArgs a{};
  a.G = G; a.ldg = ldg; a.m = m;
  a.V = V; a.ldv = ldv; a.nv = V ? nv : 0;
  a.outer = outer; a.inner = inner;
  a.n_plus = n_plus; a.inner_limit = inner_limit; a.tol_c = tol_c; a.counters = counters;
  a.T = (int)(n / w); a.b = (int)(n / (w / 2));
  a.s_begin = s_begin; a.s_end = s_end;
  a.nslab_g = (int)cdiv(m, kDfSlab);
  a.nslab_v = V ? (int)cdiv(nv, kDfSlab) : 0;
  char *p = (char *)ws;
  auto take = [&](int64_t bytes) {
    char *r = p;
    p += (bytes + 255) / 256 * 256;
    return (void *)r;
  };
  const int64_t T = a.T;
  a.Hs = (double *)take((int64_t)nsteps_total * T * w * w * 8);
  a.Vs = (double *)take((int64_t)nsteps_total * T * w * w * 8);
  a.rot = (int64_t *)take((int64_t)nsteps_total * T * 8);
  a.ready = (int *)take((int64_t)nsteps_total * T * 4);
  a.slabs = (int *)take((int64_t)nsteps_total * T * 4);
  int32_t *cp = (int32_t *)take((int64_t)nsteps_total * a.b * 4);
  a.sched = (DfSched *)take(256);
  a.qitem = (long long *)take((int64_t)kQCap * 8);
  a.qseq = (long long *)take((int64_t)kQCap * 8);
  k_colpos<<<256, 256, 0, st>>>(outer, nsteps_total, a.T, a.b, cp);
  a.colpos = cp;
  cudaMemsetAsync(a.ready, 0, (size_t)nsteps_total * T * 4, st);
  cudaMemsetAsync(a.slabs, 0, (size_t)nsteps_total * T * 4, st);
  if (w == 16) return launch_dataflow_t<16>(a, st);
  return launch_dataflow_t<32>(a, st);
}

}  // namespace jh
