// The p-step of the blocked one-sided Jacobi (H)SVD on one B200.
//
// Reference: run_block_jacobi_inplace / task (pkg/src/jhsvd/driver.py:125-200)
// with the block-pair kernels of pkg/src/jhsvd/blockkernel.py.  One p-step is
// b/2 independent tasks, task t pairing block-columns (p, q) of width bw = w/2:
//
//   K1 gram      H = [Gp Gq]^T [Gp Gq]           (blockkernel.py:76-107)
//   K2 factor    H = L L^T, R = L^T              (blockkernel.py:110-145)
//   K2 inner     pointwise Jacobi on R -> V'     (blockkernel.py:278-400)
//   K3 update    [Gp Gq] <- [Gp Gq] V', [Vp Vq] <- [Vp Vq] V'  if rotations
//                                                (blockkernel.py:407-428,
//                                                 driver.py:165-173)
//
// Layout in HBM: G is m x n column-major (column c at G + c*ldg), V is nv x n
// column-major; block-column p is the contiguous range of bw columns
// starting at p*bw.  Per-task scratch (H, V', rotation counts) is a small
// workspace that stays L2-resident.
#include "jh_common.cuh"
#include "jh_kernels.h"
#include "jhsvd_b200.h"

#include <atomic>

namespace jh {

constexpr int kMaxW = 64;          // largest block width the fused kernels take
constexpr int kGramThreads = 256;
constexpr int kGramChunk = 64;     // rows staged per smem chunk
constexpr int kGramMaxEnt = (kMaxW * (kMaxW + 1) / 2 + kGramThreads - 1) / kGramThreads;
constexpr int kUpdRows = 128;      // rows per update CTA
constexpr int kUpdThreads = 256;

__device__ __forceinline__ const double *pair_col(const double *base, int64_t ld, int p, int q,
                                                  int bw, int j) {
  const int64_t col = j < bw ? (int64_t)p * bw + j : (int64_t)q * bw + (j - bw);
  return base + col * ld;
}

// ---------------------------------------------------------------------------
// K1: Gram matrix of the block-column pair.  Every entry h[x][y] (x >= y) is
// one fma chain over the m rows in ascending order starting from +0.0,
// exactly _gram_kernel's; rows are staged through shared memory in chunks
// (chunking does not reorder a chain).  Lower triangle mirrored.
__global__ void __launch_bounds__(kGramThreads)
k_gram(const double *__restrict__ G, int64_t ldg, int64_t m, const int32_t *__restrict__ pairs,
       int bw, double *__restrict__ Hbuf) {
  const int w = 2 * bw;
  const int task = blockIdx.x;
  const int p = pairs[2 * task], q = pairs[2 * task + 1];
  extern __shared__ double sm[];
  double *T = sm;  // [kGramChunk][w] row-major chunk
  const int ne = w * (w + 1) / 2;
  int ex[kGramMaxEnt], ey[kGramMaxEnt];
  double acc[kGramMaxEnt];
  int nmine = 0;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    // triangular index -> (x, y) with x >= y, column by column
    int y = 0, rem = e;
    while (rem >= w - y) {
      rem -= w - y;
      y++;
    }
    ex[nmine] = y + rem;
    ey[nmine] = y;
    acc[nmine] = 0.0;
    nmine++;
  }
  for (int64_t c0 = 0; c0 < m; c0 += kGramChunk) {
    const int nr = (int)min64(kGramChunk, m - c0);
    for (int idx = threadIdx.x; idx < nr * w; idx += blockDim.x) {
      const int i = idx % nr, x = idx / nr;
      T[i * w + x] = pair_col(G, ldg, p, q, bw, x)[c0 + i];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kGramMaxEnt; k++) {
      if (k < nmine) {
        const int x = ex[k], y = ey[k];
        double a = acc[k];
        for (int i = 0; i < nr; i++) a = fma(T[i * w + x], T[i * w + y], a);
        acc[k] = a;
      }
    }
    __syncthreads();
  }
  double *H = Hbuf + (int64_t)task * w * w;
#pragma unroll
  for (int k = 0; k < kGramMaxEnt; k++) {
    if (k < nmine) {
      H[ey[k] * w + ex[k]] = acc[k];  // h[x, y]
      H[ex[k] * w + ey[k]] = acc[k];  // h[y, x]
    }
  }
}

// ---------------------------------------------------------------------------
// K2 building blocks, executed by one CTA of 32*max(1, w/2) threads.

// Forward-looking Cholesky of the w x w matrix in smem (column-major, ld w),
// lower triangle, _cholesky_kernel order.  Returns 0 or the 1-based pivot.
__device__ int cta_cholesky(double *H, int w, int *s_status) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = 0; k < w; k++) {
    if (tid == 0) {
      const double d = H[k * w + k];
      if (!(d > 0.0) || !isfinite(d))
        *s_status = k + 1;
      else
        H[k * w + k] = sqrt(d);
    }
    __syncthreads();
    if (*s_status) return *s_status;
    const double l = H[k * w + k];
    for (int x = k + 1 + tid; x < w; x += nt) H[k * w + x] = H[k * w + x] / l;
    __syncthreads();
    // trailing update: h[x][j] = fma(-h[x][k], h[j][k], h[x][j]) for k < j <= x
    const int r = w - k - 1;
    const int nupd = r * (r + 1) / 2;
    for (int e = tid; e < nupd; e += nt) {
      int jj = 0, rem = e;
      while (rem >= r - jj) {
        rem -= r - jj;
        jj++;
      }
      const int j = k + 1 + jj, x = j + rem;
      H[j * w + x] = fma(-H[k * w + x], H[k * w + j], H[j * w + x]);
    }
    __syncthreads();
  }
  return 0;
}

// Sweep loop of the pointwise one-sided Jacobi on R (w x w, smem col-major)
// accumulating V (smem, starts at I); _inner_jacobi_kernel order
// (blockkernel.py:278-334).  Warp pi owns pair pi of each inner p-step: its
// lane 0 forms the three dot products as in-order fma chains and the
// rotation parameters; all lanes apply the rotation (and the sorting swap)
// to their rows.  Pairs of one p-step touch disjoint columns, so a single
// CTA barrier per p-step orders everything.  On failure returns the status
// of the first failing pair in reference order (smallest pair index in the
// first failing p-step) with its 1-based local column.
struct InnerOut {
  int64_t rot, proper;
  int sweeps, status, bad;
};

struct InnerShared {
  int cnt[kMaxW];        // per warp: applied, proper (this sweep)
  int fail[kMaxW / 2];   // per warp: (status << 16) | bad
  int fail_min;          // smallest failing pair index in the current step
};

__device__ InnerOut cta_inner_jacobi(double *R, double *V, int w, const int32_t *__restrict__ steps,
                                     const int8_t *sg, double tol_c, int max_sweeps,
                                     InnerShared *sh) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = w / 2;
  InnerOut out{0, 0, 0, 0, -1};
  if (threadIdx.x == 0) sh->fail_min = 0x7fffffff;
  __syncthreads();
  for (int sw = 0; sw < max_sweeps; sw++) {
    int a_r = 0, b_r = 0;
    for (int si = 0; si < w - 1; si++) {
      const int p = steps[(si * half + warp) * 2];
      const int q = steps[(si * half + warp) * 2 + 1];
      double cs = 1.0, tn = 0.0;
      int act = 0;  // 0 skip, 1 rotate, 2 rotate + swap, -1 failure
      int hyp = 0;
      if (lane == 0) {
        const double *cp = R + p * w, *cq = R + q * w;
        double hpp = 0.0, hqq = 0.0, hpq = 0.0;
        for (int i = 0; i < w; i++) {
          const double gp = cp[i], gq = cq[i];
          hpp = fma(gp, gp, hpp);
          hqq = fma(gq, gq, hqq);
          hpq = fma(gp, gq, hpq);
        }
        int st = 0, bad = 0;
        if (hpp == 0.0) {
          st = kZeroColumn;
          bad = p + 1;
        } else if (hqq == 0.0) {
          st = kZeroColumn;
          bad = q + 1;
        } else if (!(fabs(hpq) < tol_c * sqrt(hpp) * sqrt(hqq))) {
          hyp = (sg[p] > 0 && sg[q] < 0) ? 1 : 0;
          const double t = hyp ? -1.0 : 1.0;
          if (!rotation_core(hpp, hqq, hpq, t, cs, tn)) {
            st = kHypDomain;
            bad = p + 1;
          } else {
            a_r++;
            if (cs != 1.0) b_r++;
            act = 1;
            if (!hyp) {
              const double h1 = fma(-tn, hpq, hpp);
              const double h2 = fma(tn, hpq, hqq);
              if ((sg[p] > 0 && h1 < h2) || (sg[p] < 0 && h1 > h2)) act = 2;
            }
          }
        }
        if (st) {
          act = -1;
          sh->fail[warp] = (st << 16) | bad;
          atomicMin(&sh->fail_min, warp);
        }
      }
      act = __shfl_sync(0xffffffffu, act, 0);
      if (act > 0) {
        cs = __shfl_sync(0xffffffffu, cs, 0);
        tn = __shfl_sync(0xffffffffu, tn, 0);
        hyp = __shfl_sync(0xffffffffu, hyp, 0);
        const double s = hyp ? tn : -tn;
        const bool scale = cs != 1.0;
        for (int i = lane; i < w; i += 32) {
          double *rp = R + p * w + i, *rq = R + q * w + i;
          double *vp = V + p * w + i, *vq = V + q * w + i;
          const double gp = *rp, gq = *rq, xp = *vp, xq = *vq;
          double np = fma(s, gq, gp), nq = fma(tn, gp, gq);
          double mp = fma(s, xq, xp), mq = fma(tn, xp, xq);
          if (scale) {
            np = np * cs;
            nq = nq * cs;
            mp = mp * cs;
            mq = mq * cs;
          }
          if (act == 2) {  // _swap_columns after the rotation
            *rp = nq;
            *rq = np;
            *vp = mq;
            *vq = mp;
          } else {
            *rp = np;
            *rq = nq;
            *vp = mp;
            *vq = mq;
          }
        }
      }
      __syncthreads();
      if (sh->fail_min != 0x7fffffff) {
        const int f = sh->fail[sh->fail_min];
        out.status = f >> 16;
        out.bad = f & 0xffff;
        out.sweeps = sw;
        return out;
      }
    }
    // sweep end: totals of applied / proper rotations over all warps
    if (lane == 0) {
      sh->cnt[2 * warp] = a_r;
      sh->cnt[2 * warp + 1] = b_r;
    }
    __syncthreads();
    int64_t ta = 0, tb = 0;
    for (int k = 0; k < half; k++) {
      ta += sh->cnt[2 * k];
      tb += sh->cnt[2 * k + 1];
    }
    __syncthreads();
    out.sweeps++;
    out.rot += ta;
    out.proper += tb;
    if (ta == 0) break;
  }
  return out;
}

// K2: Cholesky + inner Jacobi for every task of the p-step; one CTA of
// 32 * max(1, w/2) threads per task.  Dynamic smem: H/R and V (2 w^2 doubles).
//   counters[0] += rotations, counters[1] += proper rotations,
//   counters[2] = min error key (ULLONG_MAX when clean), counters[3] += tasks rotated
__global__ void k_factor_inner(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                               int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                               int bw, int64_t n_plus, const int32_t *__restrict__ inner,
                               int inner_limit, double tol_c, unsigned long long *counters,
                               int pstep, const int32_t *__restrict__ gblock) {
  const int w = 2 * bw;
  const int task = blockIdx.x;
  const int p = pairs[2 * task], q = pairs[2 * task + 1];
  extern __shared__ double sm[];
  double *H = sm;           // H, then R in place
  double *V = sm + w * w;
  __shared__ int8_t sg[kMaxW];
  __shared__ InnerShared sh;
  __shared__ int s_status;
  const double *Hg = Hbuf + (int64_t)task * w * w;
  for (int i = threadIdx.x; i < w * w; i += blockDim.x) {
    H[i] = Hg[i];
    V[i] = (i % w == i / w) ? 1.0 : 0.0;
  }
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    const int64_t gp = gblock ? gblock[p] : p, gq = gblock ? gblock[q] : q;
    const int64_t gcol = (j < bw ? gp * bw + j : gq * bw + (j - bw)) + 1;
    sg[j] = gcol <= n_plus ? 1 : -1;
  }
  if (threadIdx.x == 0) s_status = 0;
  __syncthreads();
  const int info = cta_cholesky(H, w, &s_status);
  if (info) {
    if (threadIdx.x == 0) {
      task_rot[task] = 0;
      atomicMin(&counters[2], err_key(pstep, task, kCholesky, info));
    }
    return;
  }
  // R = L^T in place: upper <- lower transposed, strict lower <- 0
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int i = e % w, j = e / w;
    if (i < j) {
      H[j * w + i] = H[i * w + j];
      H[i * w + j] = 0.0;
    }
  }
  __syncthreads();
  const InnerOut o = cta_inner_jacobi(H, V, w, inner, sg, tol_c, inner_limit, &sh);
  if (o.status) {
    if (threadIdx.x == 0) {
      task_rot[task] = 0;
      atomicMin(&counters[2], err_key(pstep, task, o.status, o.bad));
    }
    return;
  }
  double *Vg = Vbuf + (int64_t)task * w * w;
  for (int i = threadIdx.x; i < w * w; i += blockDim.x) Vg[i] = V[i];
  if (threadIdx.x == 0) {
    task_rot[task] = o.rot;
    atomicAdd(&counters[0], (unsigned long long)o.rot);
    atomicAdd(&counters[1], (unsigned long long)o.proper);
    if (o.rot) atomicAdd(&counters[3], 1ull);
  }
}

// ---------------------------------------------------------------------------
// K3: post-multiplication of the tall pair columns by V' (in place), for G
// rows (blockIdx.y < nbg) and V rows.  out[i][j] is one fma chain over k in
// ascending order starting from +0.0 (_postmultiply_kernel).  Skipped for a
// task without rotations (driver.py:165).
__global__ void __launch_bounds__(kUpdThreads)
k_update(double *__restrict__ G, int64_t ldg, int64_t m, double *__restrict__ Vm, int64_t ldv,
         int64_t nv, const int32_t *__restrict__ pairs, int bw, const double *__restrict__ Vbuf,
         const int64_t *__restrict__ task_rot, int nbg) {
  const int w = 2 * bw;
  const int task = blockIdx.x;
  if (task_rot[task] == 0) return;
  const int p = pairs[2 * task], q = pairs[2 * task + 1];
  double *A;
  int64_t ld, rows, r0;
  if ((int)blockIdx.y < nbg) {
    A = G;
    ld = ldg;
    rows = m;
    r0 = (int64_t)blockIdx.y * kUpdRows;
  } else {
    A = Vm;
    ld = ldv;
    rows = nv;
    r0 = (int64_t)(blockIdx.y - nbg) * kUpdRows;
  }
  if (r0 >= rows) return;
  const int nr = (int)min64(kUpdRows, rows - r0);
  extern __shared__ double sm[];
  double *Vs = sm;                // [w][w] col-major: Vs[j*w + k] = v'[k][j]
  double *As = sm + w * w;        // [w][kUpdRows]: As[k*kUpdRows + i]
  const double *Vg = Vbuf + (int64_t)task * w * w;
  for (int i = threadIdx.x; i < w * w; i += blockDim.x) Vs[i] = Vg[i];
  for (int idx = threadIdx.x; idx < nr * w; idx += blockDim.x) {
    const int i = idx % nr, k = idx / nr;
    As[k * kUpdRows + i] = pair_col(A, ld, p, q, bw, k)[r0 + i];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nr * w; idx += blockDim.x) {
    const int i = idx % nr, j = idx / nr;
    double acc = 0.0;
    for (int k = 0; k < w; k++) acc = fma(As[k * kUpdRows + i], Vs[j * w + k], acc);
    const_cast<double *>(pair_col(A, ld, p, q, bw, j))[r0 + i] = acc;
  }
}

// ---------------------------------------------------------------------------
// Kernel-level entry points (blockkernel.cholesky_in_place / inner_jacobi).

// Inner Jacobi of one c x c factor (c even, <= kMaxW).  R updated in place,
// V receives the accumulated transformation.  out: rotations, proper,
// sweeps, status, bad (1-based).
__global__ void k_inner_single(double *__restrict__ R, double *__restrict__ V, int c,
                               const int32_t *__restrict__ steps, const int8_t *__restrict__ signs,
                               double tol_c, int max_sweeps, int64_t *out) {
  extern __shared__ double sm[];
  double *Rs = sm, *Vs = sm + c * c;
  __shared__ int8_t sg[kMaxW];
  __shared__ InnerShared sh;
  for (int i = threadIdx.x; i < c * c; i += blockDim.x) {
    Rs[i] = R[i];
    Vs[i] = (i % c == i / c) ? 1.0 : 0.0;
  }
  for (int j = threadIdx.x; j < c; j += blockDim.x) sg[j] = signs[j];
  __syncthreads();
  const InnerOut o = cta_inner_jacobi(Rs, Vs, c, steps, sg, tol_c, max_sweeps, &sh);
  for (int i = threadIdx.x; i < c * c; i += blockDim.x) {
    R[i] = Rs[i];
    V[i] = Vs[i];
  }
  if (threadIdx.x == 0) {
    out[0] = o.rot;
    out[1] = o.proper;
    out[2] = o.sweeps;
    out[3] = o.status;
    out[4] = o.bad;
  }
}

// Inner Jacobi of one c x c factor of any even order above kMaxW
// (blockkernel.py:346-400: the reference takes any even order).  R and V
// live in global memory (L2-resident) and one CTA of kWideThreads runs the
// sweeps: warp k handles pairs k, k + 32, ... of every inner p-step with
// exactly the per-pair arithmetic of cta_inner_jacobi (lane 0 forms the
// three in-order chains and the rotation, all lanes apply it), one CTA
// barrier per p-step.  On failure the smallest failing pair of the first
// failing p-step is reported, as in the reference.
constexpr int kWideThreads = 1024;

__global__ void __launch_bounds__(kWideThreads)
k_inner_wide(double *__restrict__ R, double *__restrict__ V, int c,
             const int32_t *__restrict__ steps, const int8_t *__restrict__ sg, double tol_c,
             int max_sweeps, int64_t *out, const int *skip = nullptr) {
  extern __shared__ int fail[];  // per pair of the current p-step: (status << 16) | column
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (skip && *skip) {  // the factorisation failed (sweep_wide): nothing to do
    if (threadIdx.x < 5) out[threadIdx.x] = 0;
    return;
  }
  const int half = c / 2;
  __shared__ unsigned long long s_rot, s_proper;
  __shared__ int s_fail_min;
  for (int64_t i = threadIdx.x; i < (int64_t)c * c; i += blockDim.x)
    V[i] = (i % c == i / c) ? 1.0 : 0.0;
  if (threadIdx.x == 0) s_fail_min = 0x7fffffff;
  __syncthreads();
  int64_t rot = 0, proper = 0;
  int sweeps = 0, status = 0, bad = 0;
  for (int sw = 0; sw < max_sweeps; sw++) {
    if (threadIdx.x == 0) s_rot = s_proper = 0;
    __syncthreads();
    unsigned long long a_r = 0, b_r = 0;
    for (int si = 0; si < c - 1 && !status; si++) {
      for (int pi = warp; pi < half; pi += nw) {
        const int p = steps[((int64_t)si * half + pi) * 2];
        const int q = steps[((int64_t)si * half + pi) * 2 + 1];
        double cs = 1.0, tn = 0.0;
        int act = 0, hyp = 0;
        if (lane == 0) {
          const double *cp = R + (int64_t)p * c, *cq = R + (int64_t)q * c;
          double hpp = 0.0, hqq = 0.0, hpq = 0.0;
          for (int i = 0; i < c; i++) {
            const double gp = cp[i], gq = cq[i];
            hpp = fma(gp, gp, hpp);
            hqq = fma(gq, gq, hqq);
            hpq = fma(gp, gq, hpq);
          }
          int st = 0, bd = 0;
          if (hpp == 0.0) {
            st = kZeroColumn;
            bd = p + 1;
          } else if (hqq == 0.0) {
            st = kZeroColumn;
            bd = q + 1;
          } else if (!(fabs(hpq) < tol_c * sqrt(hpp) * sqrt(hqq))) {
            hyp = (sg[p] > 0 && sg[q] < 0) ? 1 : 0;
            const double t = hyp ? -1.0 : 1.0;
            if (!rotation_core(hpp, hqq, hpq, t, cs, tn)) {
              st = kHypDomain;
              bd = p + 1;
            } else {
              a_r++;
              if (cs != 1.0) b_r++;
              act = 1;
              if (!hyp) {
                const double h1 = fma(-tn, hpq, hpp);
                const double h2 = fma(tn, hpq, hqq);
                if ((sg[p] > 0 && h1 < h2) || (sg[p] < 0 && h1 > h2)) act = 2;
              }
            }
          }
          if (st) {
            act = -1;
            fail[pi] = (st << 16) | bd;
            atomicMin(&s_fail_min, pi);
          }
        }
        act = __shfl_sync(0xffffffffu, act, 0);
        if (act > 0) {
          cs = __shfl_sync(0xffffffffu, cs, 0);
          tn = __shfl_sync(0xffffffffu, tn, 0);
          hyp = __shfl_sync(0xffffffffu, hyp, 0);
          const double s = hyp ? tn : -tn;
          const bool scale = cs != 1.0;
          for (int i = lane; i < c; i += 32) {
            double *rp = R + (int64_t)p * c + i, *rq = R + (int64_t)q * c + i;
            double *vp = V + (int64_t)p * c + i, *vq = V + (int64_t)q * c + i;
            const double gp = *rp, gq = *rq, xp = *vp, xq = *vq;
            double np = fma(s, gq, gp), nq = fma(tn, gp, gq);
            double mp = fma(s, xq, xp), mq = fma(tn, xp, xq);
            if (scale) {
              np = np * cs;
              nq = nq * cs;
              mp = mp * cs;
              mq = mq * cs;
            }
            if (act == 2) {
              *rp = nq;
              *rq = np;
              *vp = mq;
              *vq = mp;
            } else {
              *rp = np;
              *rq = nq;
              *vp = mp;
              *vq = mq;
            }
          }
        }
      }
      __syncthreads();
      if (s_fail_min != 0x7fffffff) {
        const int f = fail[s_fail_min];
        status = f >> 16;
        bad = f & 0xffff;
      }
    }
    if (status) {
      sweeps = sw;
      break;
    }
    if (lane == 0) {
      atomicAdd(&s_rot, a_r);
      atomicAdd(&s_proper, b_r);
    }
    __syncthreads();
    const unsigned long long ta = s_rot, tb = s_proper;
    __syncthreads();
    sweeps++;
    rot += (int64_t)ta;
    proper += (int64_t)tb;
    if (ta == 0) break;
  }
  if (threadIdx.x == 0) {
    out[0] = rot;
    out[1] = proper;
    out[2] = sweeps;
    out[3] = status;
    out[4] = bad;
  }
}

// ---------------------------------------------------------------------------
// Block widths above kMaxW (the reference takes any even width,
// driver.py:73-74): each task of a p-step in turn through the
// general-purpose kernels -- the pair gathered into a contiguous m x w
// scratch, DMMA SYRK (jh_gram), blocked Cholesky (jh_cholesky), the
// global-memory inner Jacobi (k_inner_wide), DMMA GEMM (jh_gemm) and the
// scatter back when the task rotated (driver.py:165) -- every entry in the
// reference's order, as in the fused kernels.  A correctness path: one task
// at a time, ~15 launches per task.

__global__ void k_pair_gather(const double *__restrict__ src, int64_t lds, int64_t rows,
                              const int32_t *__restrict__ pairs, int task, int bw,
                              double *__restrict__ A) {
  const int64_t p = pairs[2 * task], q = pairs[2 * task + 1];
  const int64_t total = rows * 2 * bw;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    const int64_t col = j < bw ? p * bw + j : q * bw + (j - bw);
    A[e] = src[col * lds + i];
  }
}

__global__ void k_pair_scatter(const double *__restrict__ B, int64_t rows, double *__restrict__ dst,
                               int64_t ldd, const int32_t *__restrict__ pairs, int task, int bw,
                               const int64_t *__restrict__ trot) {
  if (trot[task] == 0) return;  // no rotations: the pair stays as it is
  const int64_t p = pairs[2 * task], q = pairs[2 * task + 1];
  const int64_t total = rows * 2 * bw;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    const int64_t col = j < bw ? p * bw + j : q * bw + (j - bw);
    dst[col * ldd + i] = B[e];
  }
}

// J signature of the task's local columns (global index + 1 <= n_plus: +1)
__global__ void k_task_signs(const int32_t *__restrict__ pairs, int task, int bw,
                             const int32_t *__restrict__ gblock, int64_t n_plus, int8_t *sg) {
  const int64_t p = pairs[2 * task], q = pairs[2 * task + 1];
  const int64_t gp = gblock ? gblock[p] : p, gq = gblock ? gblock[q] : q;
  for (int j = threadIdx.x; j < 2 * bw; j += blockDim.x) {
    const int64_t gcol = (j < bw ? gp * bw + j : gq * bw + (j - bw)) + 1;
    sg[j] = gcol <= n_plus ? 1 : -1;
  }
}

// the task's outcome: counters, rotation flag, first-error key; the
// Cholesky status is cleared for the next task
__global__ void k_task_finish(const int64_t *out, int *info, int pstep, int task, int64_t *trot,
                              unsigned long long *counters) {
  if (threadIdx.x != 0) return;
  if (*info) {
    trot[task] = 0;
    atomicMin(&counters[2], err_key(pstep, task, kCholesky, *info));
    *info = 0;
    return;
  }
  if (out[3]) {
    trot[task] = 0;
    atomicMin(&counters[2], err_key(pstep, task, (int)out[3], (int)out[4]));
    return;
  }
  trot[task] = out[0];
  atomicAdd(&counters[0], (unsigned long long)out[0]);
  atomicAdd(&counters[1], (unsigned long long)out[1]);
  if (out[0]) atomicAdd(&counters[3], 1ull);
}

static int sweep_wide(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                      int64_t nv, int w, const int32_t *outer, const int32_t *gblock,
                      int first_step, int nsteps, const int32_t *inner, int64_t n_plus,
                      int inner_limit, double tol_c, void *workspace,
                      unsigned long long *counters, cudaStream_t st) {
  const int bw = w / 2, ntask = (int)(n / w);
  const int64_t ww = (int64_t)w * w, rows = V && nv > m ? nv : m;
  int64_t *trot = (int64_t *)workspace;  // per task of the current p-step
  // scratch: A, B (rows x w), H, R, V' (w x w), out[5], info, signs
  const size_t bytes = sizeof(double) * (2 * rows * w + 3 * ww) + 8 * 8 + 8 + (size_t)w + 64;
  char *scr = nullptr;
  if (cudaMallocAsync((void **)&scr, bytes, st) != cudaSuccess)
    return -(int)cudaErrorMemoryAllocation;
  double *A = (double *)scr, *B = A + rows * w, *H = B + rows * w, *R = H + ww, *Vp = R + ww;
  int64_t *out = (int64_t *)(Vp + ww);
  int *info = (int *)(out + 8);
  int8_t *sg = (int8_t *)(info + 2);
  cudaMemsetAsync(info, 0, sizeof(int), st);
  const int smem_inner = (int)sizeof(int) * (w / 2);
  ensure_smem((const void *)k_inner_wide, smem_inner);
  auto grid_for = [](int64_t total) { return (unsigned)min64(cdiv(total, 256), 148 * 8); };
  int rc = 0;
  for (int s = first_step; s < first_step + nsteps && !rc; s++) {
    const int32_t *pairs = outer + (int64_t)s * ntask * 2;
    for (int t = 0; t < ntask && !rc; t++) {
      k_pair_gather<<<grid_for(m * w), 256, 0, st>>>(G, ldg, m, pairs, t, bw, A);
      rc = jh_gram(A, m, m, w, H, st);
      if (!rc) rc = jh_cholesky(H, w, R, info, st);
      if (rc) break;
      k_task_signs<<<1, 256, 0, st>>>(pairs, t, bw, gblock, n_plus, sg);
      k_inner_wide<<<1, kWideThreads, smem_inner, st>>>(R, Vp, w, inner, sg, tol_c, inner_limit,
                                                        out, info);
      k_task_finish<<<1, 32, 0, st>>>(out, info, s, t, trot, counters);
      rc = jh_gemm(A, m, m, w, Vp, w, w, B, m, st);
      if (rc) break;
      k_pair_scatter<<<grid_for(m * w), 256, 0, st>>>(B, m, G, ldg, pairs, t, bw, trot);
      if (V) {
        k_pair_gather<<<grid_for(nv * w), 256, 0, st>>>(V, ldv, nv, pairs, t, bw, A);
        rc = jh_gemm(A, nv, nv, w, Vp, w, w, B, nv, st);
        if (rc) break;
        k_pair_scatter<<<grid_for(nv * w), 256, 0, st>>>(B, nv, V, ldv, pairs, t, bw, trot);
      }
      g_launches += V ? 8 : 5;
    }
  }
  cudaFreeAsync(scr, st);
  if (rc) return rc;
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// ---------------------------------------------------------------------------
// host side

// Workspace of a sweep over a pivot table of `steps` p-steps at order n:
//   H | V' ring (4 p-steps) | rotation-count ring (4) | per-task done flags
//   + ready list (engine 1) | second H | per-task G slab counters |
//   block-column -> task tables (engine 1, Grams in the update launch)
// The per-task V' and counts of the last four p-steps stay until the paired
// V pass of engine 1 has read them.
static int64_t ws_bytes_for(int64_t n, int w, int64_t steps) {
  const int64_t ntask = n / w, b = 2 * ntask, ww = (int64_t)w * w;
  if (steps <= 0) steps = b > 1 ? b - 1 : 1;
  return ntask * ww * 8 * 5 + ntask * 8 * 4 + (2 * ntask + 1) * 8 + ntask * ww * 8 + ntask * 8 +
         steps * b * 4 + 1024;
}

static int finish(cudaStream_t) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// Engine 0: per p-step K1 Gram, K2 factor + inner Jacobi, K3 update of the
// rotated tasks' G and V columns.  The DMMA / TMA kernels where the width
// allows, the generic SIMT kernels otherwise (or when opt_simple()).
static int sweep_basic(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                       int64_t nv, int w, const int32_t *outer, const int32_t *gblock,
                       int first_step, int nsteps, const int32_t *inner, int64_t n_plus,
                       int inner_limit, double tol_c, void *workspace,
                       unsigned long long *counters, cudaStream_t st) {
  const int bw = w / 2;
  const int ntask = (int)(n / w);
  double *Hbuf = (double *)workspace;
  double *Vbuf = Hbuf + (int64_t)ntask * w * w;                    // ring slot 0
  int64_t *trot = (int64_t *)(Hbuf + (int64_t)ntask * w * w * 5);  // ring slot 0
  const int thr_inner = 32 * (bw > 1 ? bw : 1);
  const int nbg = (int)cdiv(m, kUpdRows);
  const int nbv = V ? (int)cdiv(nv, kUpdRows) : 0;
  const size_t smem_gram = sizeof(double) * kGramChunk * w;
  const size_t smem_inner = sizeof(double) * 2 * (size_t)w * w;
  const size_t smem_upd = sizeof(double) * ((size_t)w * w + (size_t)w * kUpdRows);
  ensure_smem((const void *)k_factor_inner, (int)smem_inner);
  ensure_smem((const void *)k_update, (int)smem_upd);
  const bool simple = opt_simple();
  const bool tma_gram = !simple && gram_tma_ok(w, m, ldg);
  const bool fast_inner = !simple && inner5_ok(w);
  const bool dmma_update = !simple && update_dmma_ok(w);
  for (int s = first_step; s < first_step + nsteps; s++) {
    const int32_t *pairs = outer + (int64_t)s * ntask * 2;
    prof_mark(st, 0, false);
    if (tma_gram)
      launch_gram_tma(G, ldg, m, pairs, ntask, w, Hbuf, st);
    else
      k_gram<<<ntask, kGramThreads, smem_gram, st>>>(G, ldg, m, pairs, bw, Hbuf);
    prof_mark(st, 0, true);
    prof_mark(st, 1, false);
    if (fast_inner)
      launch_inner5(Hbuf, Vbuf, trot, pairs, ntask, w, n_plus, inner, inner_limit, tol_c,
                    counters, s, st, false, nullptr, 0, gblock);
    else
      k_factor_inner<<<ntask, thr_inner, smem_inner, st>>>(Hbuf, Vbuf, trot, pairs, bw, n_plus,
                                                           inner, inner_limit, tol_c, counters, s,
                                                           gblock);
    prof_mark(st, 1, true);
    prof_mark(st, 2, false);
    if (dmma_update)
      launch_update_dmma(G, ldg, m, V, ldv, nv, pairs, ntask, w, Vbuf, trot, st);
    else
      k_update<<<dim3(ntask, nbg + nbv), kUpdThreads, smem_upd, st>>>(G, ldg, m, V, ldv, nv,
                                                                     pairs, bw, Vbuf, trot, nbg);
    prof_mark(st, 2, true);
    g_launches += 3;
  }
  return finish(st);
}

// Engine 1 (default for rrow-like tables with V accumulated): the
// per-p-step Gram and inner Jacobi kernels, then one mixed update launch per
// p-step: the G update CTAs of p-step s and -- the V update deferred to one
// pass per pair of p-steps (a, a+1) over the 4-cycles of the pair
// (jh_vpair.cu) -- half of a pair's V row slabs (the other half in the next
// launch).  V is read by nothing else during the sweep and every V row still
// receives the same transformations in the same order, so the results are
// bitwise those of engine 0; V moves through HBM once per two p-steps, and
// its DMMA-bound slabs share the SMs with the HBM-bound G slabs.  The update
// launch is a programmatic dependent launch: its CTAs start while the inner
// kernel's slow tasks finish, each waiting for its own tasks' release flags.
// For G of at most 2^26 entries the Grams of p-step s+1 run as trailing CTAs
// of the update launch of p-step s (profiles/r01/cycle_engine.md).
static int sweep_vpaired(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                         int64_t nv, int w, const int32_t *outer, int steps, const int32_t *plan,
                         const int32_t *gblock, int first_step, int nsteps, const int32_t *inner,
                         int64_t n_plus, int inner_limit, double tol_c, void *workspace,
                         unsigned long long *counters, cudaStream_t st) {
  const int b = (int)(n / (w / 2));
  const int ntask = (int)(n / w);
  const int64_t ww = (int64_t)w * w;
  double *Hbuf = (double *)workspace;
  double *Vring = Hbuf + (int64_t)ntask * ww;
  int64_t *rring = (int64_t *)(Vring + 4 * (int64_t)ntask * ww);
  int64_t *done = rring + 4 * (int64_t)ntask;
  double *Hbuf2 = (double *)(done + 2 * ntask + 1);
  int64_t *gcnt = (int64_t *)(Hbuf2 + (int64_t)ntask * ww);
  int32_t *colpos = (int32_t *)(gcnt + ntask);
  auto hb = [&](int i) { return (i % 2) ? Hbuf2 : Hbuf; };
  auto vp = [&](int i) { return Vring + (int64_t)(i % 4) * ntask * ww; };
  auto rt = [&](int i) { return rring + (int64_t)(i % 4) * ntask; };
  const bool pdl = opt_overlap();
  // release-flag epochs: process-wide and atomic, so that solves issued from
  // several host threads never share one
  static std::atomic<int64_t> epoch_ctr{0};
  int64_t epoch = 0;
  if (pdl) cudaMemsetAsync(done, 0xff, sizeof(int64_t) * (2 * ntask + 1), st);
  // Grams of p-step s+1 in the update launch of p-step s (trailing CTAs
  // that start when their block-columns are final): a gain where the Gram
  // chains are short (m <= 8192 and G of at most 2^26 entries: n = 8192,
  // 0.626 vs 0.649 ms per p-step) or where 1-2 tasks per SM leave room for
  // them (256 tasks at m = 16384: 1.00 vs 1.04 ms); a loss at 512 tasks
  // (16384^2: 1.83 vs 1.80) and with fewer tasks than SMs, where the split
  // Gram kernel is faster (profiles/r02/README.md)
  const int sms = sm_count();
  const bool gmix = w == 32 && nsteps > 1 &&
                    ((m <= 8192 && m * n <= (int64_t(1) << 26)) ||
                     (ntask > sms && ntask <= 2 * sms && m <= 16384));
  if (gmix) {
    cudaMemsetAsync(gcnt, 0, sizeof(int64_t) * ntask, st);
    launch_colpos(outer + (int64_t)first_step * ntask * 2, nsteps, ntask, b, colpos, st);
    g_launches += 1;
  }
  for (int i = 0; i < nsteps; i++) {
    const int s = first_step + i;
    const int32_t *pairs = outer + (int64_t)s * ntask * 2;
    if (!gmix || i == 0) {
      prof_mark(st, 0, false);
      launch_gram_tma(G, ldg, m, pairs, ntask, w, hb(i), st);
      prof_mark(st, 0, true);
    }
    if (pdl) {
      epoch = ++epoch_ctr;
      cudaMemsetAsync(done + ntask, 0, sizeof(int64_t), st);  // ready-list count
    }
    // (with the programmatic launch, class 1 times the inner Jacobi and the
    // overlapped update together)
    prof_mark(st, 1, false);
    launch_inner5(hb(i), vp(i), rt(i), pairs, ntask, w, n_plus, inner, inner_limit, tol_c,
                  counters, s, st, false, pdl ? done : nullptr, epoch, gblock);
    if (!pdl) prof_mark(st, 1, true);
    const bool last = (i == nsteps - 1);
    // V work: pair j = (2j, 2j+1) is applied to its even row slabs in the
    // launch of p-step 2j+2 and to its odd ones in that of 2j+3, so the V
    // items of a launch never wait for the inner kernel still running;
    // whatever is due later than the last p-step is flushed after it, in
    // p-step order (launches of one stream run in order)
    int nsrc = 0, sa[2], k0[2], kstep[2];
    bool second[2];
    const double *VpA[2], *VpB[2];
    const int64_t *rotA[2], *rotB[2];
    auto add = [&](int i0, bool sec, int kk0, int kst) {
      sa[nsrc] = first_step + i0;
      second[nsrc] = sec;
      VpA[nsrc] = vp(i0);
      rotA[nsrc] = rt(i0);
      VpB[nsrc] = sec ? vp(i0 + 1) : nullptr;
      rotB[nsrc] = sec ? rt(i0 + 1) : nullptr;
      k0[nsrc] = kk0;
      kstep[nsrc] = kst;
      nsrc++;
    };
    auto flush = [&](int i0, bool sec, int kk0, int kst) {  // a V-only launch
      nsrc = 0;
      add(i0, sec, kk0, kst);
      prof_mark(st, 3, false);
      launch_update_mix(G, ldg, 0, pairs, ntask, vp(i), rt(i), V, ldv, nv, outer, plan, b, steps,
                        nsrc, sa, second, VpA, rotA, VpB, rotB, k0, kstep, st);
      prof_mark(st, 3, true);
      g_launches += 1;
    };
    if (i % 2 == 0 && i >= 2) add(i - 2, true, 0, 2);
    if (i % 2 == 1 && i >= 3) add(i - 3, true, 1, 2);
    if (!pdl) prof_mark(st, 2, false);
    launch_update_mix(G, ldg, m, pairs, ntask, vp(i), rt(i), V, ldv, nv, outer, plan, b, steps,
                      nsrc, sa, second, VpA, rotA, VpB, rotB, k0, kstep, st,
                      pdl ? done : nullptr, epoch, s,
                      gmix && !last ? pairs + ntask * 2 : nullptr, colpos + (int64_t)i * b, gcnt,
                      hb(i + 1));
    prof_mark(st, pdl ? 1 : 2, true);
    g_launches += 3;
    if (last) {
      if (i % 2 == 1) {
        flush(i - 1, true, 0, 1);              // the last pair, all slabs
      } else {
        if (i >= 2) flush(i - 2, true, 1, 2);  // odd slabs of the previous pair
        flush(i, false, 0, 1);                 // the last p-step alone
      }
    }
  }
  return finish(st);
}

// QR peel-off shortening (shortening = 1, reference blockkernel.py:223-244):
// per p-step the R factors of every task (jh_qr.cu), the inner Jacobi on R
// (no Gram, no Cholesky), and the same post-multiplication.
static int sweep_qr(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                    int64_t nv, int w, const int32_t *outer, const int32_t *gblock,
                    int first_step, int nsteps, const int32_t *inner, int64_t n_plus,
                    int inner_limit, double tol_c, void *workspace,
                    unsigned long long *counters, cudaStream_t st) {
  if (!qr_ok(w, m)) return -1000;
  const int ntask = (int)(n / w);
  const int64_t ww = (int64_t)w * w;
  double *Rbuf = (double *)workspace;
  double *Vbuf = Rbuf + (int64_t)ntask * ww;
  int64_t *trot = (int64_t *)(Rbuf + (int64_t)ntask * ww * 5);
  for (int s = first_step; s < first_step + nsteps; s++) {
    const int32_t *pairs = outer + (int64_t)s * ntask * 2;
    prof_mark(st, 0, false);
    launch_qr_peeloff(G, ldg, m, pairs, ntask, w, Rbuf, st);
    prof_mark(st, 0, true);
    prof_mark(st, 1, false);
    launch_inner5(Rbuf, Vbuf, trot, pairs, ntask, w, n_plus, inner, inner_limit, tol_c, counters,
                  s, st, true, nullptr, 0, gblock);
    prof_mark(st, 1, true);
    prof_mark(st, 2, false);
    launch_update_dmma(G, ldg, m, V, ldv, nv, pairs, ntask, w, Vbuf, trot, st);
    prof_mark(st, 2, true);
    g_launches += 3;
  }
  return finish(st);
}

}  // namespace jh

using namespace jh;

extern "C" {

int64_t jh_sweep_workspace_bytes(int64_t n, int w, int64_t steps) {
  if (w < 2 || w % 2 || n % w) return -1;
  return ws_bytes_for(n, w, steps);
}

int64_t jh_cycle_plan_ints(int b, int steps) { return cycle_plan_ints(b, steps); }

int jh_cycle_plan(const int32_t *outer, int b, int steps, int32_t *plan) {
  return cycle_plan(outer, b, steps, plan);
}

int jh_block_sweep(double *G, int64_t ldg, int64_t m, int64_t n, double *V, int64_t ldv,
                   int64_t nv, int w, const int32_t *outer, int outer_steps, const int32_t *plan,
                   const int32_t *gblock, int engine, int shortening, int first_step, int nsteps,
                   const int32_t *inner, int64_t n_plus, int inner_limit, double tol_c,
                   void *workspace, int64_t ws_bytes, unsigned long long *counters,
                   void *stream) {
  if (w < 2 || w % 2 || w > 8190 || n % w || m < 1 || ldg < m) return -1000;
  if (V && (nv < 1 || ldv < nv)) return -1000;
  if (first_step < 0 || nsteps < 0 || first_step + nsteps > outer_steps) return -1000;
  if (ws_bytes < ws_bytes_for(n, w, outer_steps)) return -1001;
  if (nsteps == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (w > kMaxW) {
    if (shortening != 0) return -1000;
    return sweep_wide(G, ldg, m, n, V, ldv, nv, w, outer, gblock, first_step, nsteps, inner,
                      n_plus, inner_limit, tol_c, workspace, counters, st);
  }
  if (shortening == 1)
    return sweep_qr(G, ldg, m, n, V, ldv, nv, w, outer, gblock, first_step, nsteps, inner, n_plus,
                    inner_limit, tol_c, workspace, counters, st);
  if (shortening != 0) return -1000;
  const bool vpaired_ok = engine == 1 && plan && V && !opt_simple() && w == 32 && m % 2 == 0 &&
                          ldg % 2 == 0 && nv % 2 == 0 && ldv % 2 == 0;
  if (vpaired_ok)
    return sweep_vpaired(G, ldg, m, n, V, ldv, nv, w, outer, outer_steps, plan, gblock,
                         first_step, nsteps, inner, n_plus, inner_limit, tol_c, workspace,
                         counters, st);
  return sweep_basic(G, ldg, m, n, V, ldv, nv, w, outer, gblock, first_step, nsteps, inner,
                     n_plus, inner_limit, tol_c, workspace, counters, st);
}

// inner_jacobi (blockkernel.py:346-400) on one c x c factor, c even <= 64.
int jh_inner_jacobi(double *R, double *V, int c, const int32_t *steps, const int8_t *signs,
                    double tol_c, int max_sweeps, int64_t *out, void *stream) {
  if (c < 2 || c % 2 || c > 0x7fff) return -1000;
  if (c > kMaxW) {
    // any larger even order: R, V in global memory, one CTA (k_inner_wide);
    // one shared int per pair for the failure report
    const int smem = (int)sizeof(int) * (c / 2);
    ensure_smem((const void *)k_inner_wide, smem);
    g_launches++;
    k_inner_wide<<<1, kWideThreads, smem, (cudaStream_t)stream>>>(R, V, c, steps, signs, tol_c,
                                                                  max_sweeps, out);
    return finish((cudaStream_t)stream);
  }
  const size_t smem = sizeof(double) * 2 * (size_t)c * c;
  ensure_smem((const void *)k_inner_single, (int)(sizeof(double) * 2 * kMaxW * kMaxW));
  g_launches++;
  k_inner_single<<<1, 32 * (c / 2), smem, (cudaStream_t)stream>>>(R, V, c, steps, signs, tol_c,
                                                                  max_sweeps, out);
  return finish((cudaStream_t)stream);
}

}  // extern "C"
