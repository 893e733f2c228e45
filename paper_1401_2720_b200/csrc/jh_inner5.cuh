// Inner Jacobi of one task by a CTA of NTH threads (device function shared
// by the per-p-step kernel k_factor_inner5 and the dataflow kernel):
// Cholesky of the task's Gram matrix, then the pointwise sweeps; warp 0
// forms the w/2 pairs' dot products and rotations (lane = pair), all threads
// rotate R one pair at a time, warps 1.. apply the previous inner step's
// rotations to V.  Reference: blockkernel.py:110-145 and 278-334.
#pragma once

#include "jh_common.cuh"
#include "jh_fastmath.cuh"

#ifndef JH_I5_ROLLED
#define JH_I5_ROLLED 1
#endif
// JH_I5_PROF=1 builds K2 variant 5 with clock64 phase stamps of thread 0
// (jh_inner5_profile; dev builds only, tools/build_variant.sh)
#ifndef JH_I5_DOTU
#define JH_I5_DOTU 32  // unroll of the dot-product loop
#endif
#ifndef JH_I5_PREF
#define JH_I5_PREF 1
#endif
#ifndef JH_I5_SPLIT
#define JH_I5_SPLIT 0
#endif
#ifndef JH_I5_PROF
#define JH_I5_PROF 0
#endif
#if JH_I5_PROF
#define I5_LAP(acc)                            \
  do {                                         \
    if (tid == 0) {                            \
      const long long now_ = clock64();        \
      acc += (unsigned long long)(now_ - t5_); \
      t5_ = now_;                              \
    }                                          \
  } while (0)
#else
#define I5_LAP(acc) \
  do {              \
  } while (0)
#endif

namespace jh {

constexpr int kI5DotUnroll = JH_I5_DOTU;

// IEEE a / b and sqrt(x) through the branch-free fast paths when they are in
// range (bitwise the same values), the operators otherwise
__device__ __forceinline__ double div_ieee(double a, double b) {
  bool ok = true;
  double q = div_fp(a, b, ok);
  if (!ok) q = a / b;
  return q;
}
__device__ __forceinline__ double sqrt_ieee(double x) {
  bool ok = true;
  double r = sqrt_fp(x, ok);
  if (!ok) r = sqrt(x);
  return r;
}

// optional phase timing (jh_inner5_profile; one copy per translation unit):
// cycles seen by thread 0 in [load + Cholesky, dots, rotation + test,
// barrier 1, R apply + barrier 2], inner p-steps, inner sweeps, tasks, task
// cycles (sum), task cycles (max)
static __device__ int g_i5_on = 0;
static __device__ unsigned long long g_i5[12];

template <int W>
struct InnerCfg5 {
  static constexpr int HALF = W / 2;
  static constexpr int LD = W + 1;
  static constexpr int NTH = W <= 32 ? 128 : 256;
};

struct StepParams5 {
  double cs, tn;
  int act;  // 0 skip, 1 rotate, 2 rotate + swap, 4 | 1 hyperbolic rotate
};

template <int W>
struct InnerSmem5 {
  double H[W * W];
  double R[W * (W + 1)];
  double V[W * (W + 1)];
  StepParams5 prm[2][W / 2];
  int8_t steps[(W - 1) * W];  // (p, q) per pair per inner p-step
  int8_t sg[W];
  int fail_status, fail_bad, stop, sweep_rot, sweep_proper, chol;
};

// rotate (+ swap) columns p, q of M (ld LD) at row i
__device__ __forceinline__ void rot_apply5(double *M, int ld, int p, int q, int i,
                                          const StepParams5 &pr) {
  const double cs = pr.cs, tn = pr.tn;
  const double s = (pr.act & 4) ? tn : -tn;
  double *mp = M + p * ld + i, *mq = M + q * ld + i;
  const double gp = *mp, gq = *mq;
  double np = fma(s, gq, gp), nq = fma(tn, gp, gq);
  if (cs != 1.0) {
    np = np * cs;
    nq = nq * cs;
  }
  if ((pr.act & 3) == 2) {
    *mp = nq;
    *mq = np;
  } else {
    *mp = np;
    *mq = nq;
  }
}

// Cholesky of the task's Gram matrix by one warp (reference element order:
// element (j, x) receives its updates for pivots 0..j-1 in order, then the
// square root or the division by l_j, as in the reference's forward-looking
// loop; shuffles and warp syncs instead of CTA barriers);
// writes R = L^T (zero strict lower triangle, ld W + 1) and returns 0, or
// the 1-based index of the first bad pivot.  Lane x keeps column x of the
// trailing triangle in registers, shifted by one row per pivot so that the
// pivot row is always e[0]: the pivot loop stays rolled (the fully unrolled
// form is ~10k instructions executed once per task, i.e. i-cache misses).
// colk: W doubles of scratch shared memory.
template <int W>
__device__ __noinline__ int chol6_warp(const double *__restrict__ Hg, double *R, double *colk,
                                      int lane) {
  constexpr int LD = W + 1;
  constexpr unsigned FULL = 0xffffffffu;
  const int x = lane;
  double e[W];  // e[j] = element (k + j, x) at pivot k
#pragma unroll
  for (int j = 0; j < W; j++) e[j] = (x < W && j <= x) ? __ldcg(Hg + j * W + x) : 0.0;
  if (x < W)
#pragma unroll
    for (int i = 0; i < W; i++)
      if (i > x) R[x * LD + i] = 0.0;
  int chol = 0;
#pragma unroll 1
  for (int k = 0; k < W; k++) {
    int bad = 0;
    if (x == k) {
      const double d = e[0];
      if (!(d > 0.0) || !isfinite(d))
        bad = 1;
      else
        e[0] = sqrt_ieee(d);
    }
    if (__shfl_sync(FULL, bad, k)) {
      chol = k + 1;
      break;
    }
    const double l = __shfl_sync(FULL, e[0], k);
    if (x > k && x < W) e[0] = div_ieee(e[0], l);
    if (x >= k && x < W) R[x * LD + k] = e[0];  // element (k, x) is final
    colk[x] = e[0];                             // row k, element (k, x) per lane
    __syncwarp();
#pragma unroll
    for (int j = 1; j < W; j++) {
      const int jj = k + j;
      if (jj < W && x >= jj) e[j] = fma(-e[0], colk[jj], e[j]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < W - 1; j++) e[j] = e[j + 1];
    e[W - 1] = 0.0;
  }
  return chol;
}

// Rotations of one inner p-step applied to row i of M for the pairs g,
// g + G, g + 2G, ... (< HALF): all loads first, then the arithmetic and the
// stores (a loop of rot_apply5 calls serialises on the possible aliasing of
// each store with the next pair's loads).  Same arithmetic as rot_apply5.
template <int HALF, int G>
__device__ __forceinline__ void rot_apply_rows(double *M, int ld, const int8_t *pst,
                                               const StepParams5 *prm, int g, int i) {
  constexpr int MP = (HALF + G - 1) / G;
  double vp[MP], vq[MP];
  StepParams5 P[MP];
  int cp[MP], cq[MP];
#pragma unroll
  for (int u = 0; u < MP; u++) {
    const int pi = g + u * G;
    if (pi < HALF) {
      P[u] = prm[pi];
      cp[u] = pst[2 * pi];
      cq[u] = pst[2 * pi + 1];
      vp[u] = M[cp[u] * ld + i];
      vq[u] = M[cq[u] * ld + i];
    }
  }
#pragma unroll
  for (int u = 0; u < MP; u++) {
    const int pi = g + u * G;
    if (pi < HALF && P[u].act) {
      const double cs = P[u].cs, tn = P[u].tn;
      const double sn = (P[u].act & 4) ? tn : -tn;
      double np = fma(sn, vq[u], vp[u]), nq = fma(tn, vp[u], vq[u]);
      if (cs != 1.0) {
        np = np * cs;
        nq = nq * cs;
      }
      const bool sw = (P[u].act & 3) == 2;
      M[cp[u] * ld + i] = sw ? nq : np;
      M[cq[u] * ld + i] = sw ? np : nq;
    }
  }
}

// Rotations of one inner p-step applied to M by all NTH threads, one pair
// per NTH / HALF threads: thread (pair, sub) rotates rows sub, sub + NTH /
// HALF, ... of its pair's two columns, all loads before the stores (same
// arithmetic as rot_apply5; one parameter fetch per thread).
template <int W, int HALF, int NTH>
__device__ __forceinline__ void rot_apply_pair(double *M, int ld, const int8_t *pst,
                                               const StepParams5 *prm, int tid) {
  constexpr int TPP = NTH / HALF;  // threads per pair
  constexpr int RPT = W / TPP;     // rows per thread
  static_assert(NTH % HALF == 0 && W % TPP == 0, "apply layout");
  const int pi = tid / TPP, sub = tid - pi * TPP;
  const StepParams5 P = prm[pi];
  if (!P.act) return;
  const int cp = pst[2 * pi], cq = pst[2 * pi + 1];
  double *mp = M + cp * ld + sub, *mq = M + cq * ld + sub;
  double vp[RPT], vq[RPT];
#pragma unroll
  for (int u = 0; u < RPT; u++) {
    vp[u] = mp[u * TPP];
    vq[u] = mq[u * TPP];
  }
  const double cs = P.cs, tn = P.tn;
  const double sn = (P.act & 4) ? tn : -tn;
  const bool sw = (P.act & 3) == 2;
#pragma unroll
  for (int u = 0; u < RPT; u++) {
    double np = fma(sn, vq[u], vp[u]), nq = fma(tn, vp[u], vq[u]);
    if (cs != 1.0) {
      np = np * cs;
      nq = nq * cs;
    }
    mp[u * TPP] = sw ? nq : np;
    mq[u * TPP] = sw ? np : nq;
  }
}

// Returns the task's rotation count (>= 0, V' written to Vg column-major,
// counters updated) or -1 after recording a numerical failure under key
// (pstep, task_key).  smem must hold an InnerSmem5<W>.  All NTH threads call.
template <int W, int NTH>
__device__ __noinline__ long long inner5_task(unsigned char *smem, const double *__restrict__ Hg,
                                              double *__restrict__ Vg, int p0, int q0,
                                              int64_t n_plus, const int32_t *__restrict__ inner,
                                              int inner_limit, double tol_c,
                                              unsigned long long *counters, int pstep,
                                              int task_key, int64_t *rot_out,
                                              bool from_r = false,
                                              const int32_t *__restrict__ gblock = nullptr) {
  constexpr int HALF = InnerCfg5<W>::HALF, LD = InnerCfg5<W>::LD;
  constexpr int BW = W / 2, NSTEP = W - 1;
  InnerSmem5<W> &S = *reinterpret_cast<InnerSmem5<W> *>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- load H, inner table, signs; V = I
  for (int i = tid; i < W * W; i += NTH) S.H[i] = __ldcg(Hg + i);  // L2: produced this launch
  for (int i = tid; i < W * LD; i += NTH) {
    const int col = i / LD, row = i - col * LD;
    S.V[i] = (row == col) ? 1.0 : 0.0;
  }
  for (int i = tid; i < NSTEP * W; i += NTH) S.steps[i] = (int8_t)inner[i];
  // signature of the pair's columns from their global (1-based) indices;
  // gblock maps a local block-column to its global index (sharded solves)
  for (int j = tid; j < W; j += NTH) {
    const int64_t gp = gblock ? gblock[p0] : p0, gq = gblock ? gblock[q0] : q0;
    const int64_t gcol = (j < BW ? gp * BW + j : gq * BW + (j - BW)) + 1;
    S.sg[j] = gcol <= n_plus ? 1 : -1;
  }
  if (tid == 0) {
    S.chol = 0;
    S.stop = 0;
  }
  __syncthreads();
  if (from_r) {
    // Hg already holds the shortened factor R (QR peel-off, column-major,
    // zero strict lower triangle): no Cholesky
    for (int e = tid; e < W * W; e += NTH) {
      const int j = e / W, i = e - j * W;
      S.R[j * LD + i] = S.H[e];
    }
    __syncthreads();
  } else {

  if constexpr (W <= 32) {
    // one warp, no CTA barriers (chol6_warp; H is read from global again,
    // S.H serves as its scratch row)
    if (warp == 0) {
      const int c = chol6_warp<W>(Hg, S.R, S.H, lane);
      if (lane == 0) S.chol = c;
    }
    __syncthreads();
  } else {
    // ---- forward-looking Cholesky (reference element order), lower triangle
    {
      const int x = tid % W, jg = tid / W;
      constexpr int JS = NTH / W;
      for (int k = 0; k < W; k++) {
        if (tid == 0) {
          const double d = S.H[k * W + k];
          if (!(d > 0.0) || !isfinite(d))
            S.chol = k + 1;
          else
            S.H[k * W + k] = sqrt_ieee(d);
        }
        __syncthreads();
        if (S.chol) break;
        const double l = S.H[k * W + k];
        if (jg == 0 && x > k) S.H[k * W + x] = div_ieee(S.H[k * W + x], l);
        __syncthreads();
        for (int j = k + 1 + jg; j < W; j += JS)
          if (x >= j) S.H[j * W + x] = fma(-S.H[k * W + x], S.H[k * W + j], S.H[j * W + x]);
        __syncthreads();
      }
    }
  }
  if (S.chol) {
    if (tid == 0) {
      *rot_out = 0;
      atomicMin(&counters[2], err_key(pstep, task_key, kCholesky, S.chol));
    }
    return -1;
  }
  if constexpr (W > 32) {
    // R = L^T (R[i][j] = H[i * W + j] for i <= j)
    for (int e = tid; e < W * W; e += NTH) {
      const int j = e / W, i = e - j * W;
      S.R[j * LD + i] = (i <= j) ? S.H[i * W + j] : 0.0;
    }
    __syncthreads();
  }
  }  // !from_r

  // ---- inner sweeps
  int a_r = 0, b_r = 0;  // lane-private counters of warp 0
  int64_t tot_rot = 0, tot_proper = 0;
  int sweeps = 0, status = 0, bad = -1;
  int gstep = 0;  // global inner p-step counter (for the lagged V update)
#if JH_I5_PROF
  long long t5_ = clock64();
  unsigned long long p5_dots = 0, p5_rot = 0, p5_bar1 = 0, p5_app = 0;
  const long long t5_task = t5_;
#endif
  const int ri = tid % W;         // row handled in the R / V applies
  const int rg = tid / W;         // pair group
  constexpr int RGS = NTH / W;    // pair groups in the R apply
  // pair of warp-0 lane i in the next inner p-step, loaded one step ahead
  // (the table is read-only; JH_I5_PREF=0 loads it in the step)
  int p_next = 0, q_next = 0;
  if (JH_I5_PREF && warp == 0 && lane < HALF) {
    p_next = S.steps[2 * lane];
    q_next = S.steps[2 * lane + 1];
  }
  for (int sw = 0; sw < inner_limit && !status; sw++) {
    for (int si = 0; si < NSTEP; si++, gstep++) {
      const int8_t *st = S.steps + si * W;
      StepParams5 *cur = S.prm[gstep & 1];
      if (warp == 0) {
        int fail = 0, fb = 0;
#if JH_I5_SPLIT
        // (build option, measured slower: 289 vs 259 us per launch) the three
        // chains of pair i on two lanes: lane i runs hpp and hpq,
        // lane i + w/2 runs hqq (same fma order; its second chain is unused)
        double hpp, hqq, hpq;
        {
          const bool upper = lane >= HALF;
          const int pl = lane < 2 * HALF ? (upper ? lane - HALF : lane) : 0;
          const int pa = st[2 * pl + (upper ? 1 : 0)], pb = st[2 * pl + (upper ? 0 : 1)];
          const double *ca = S.R + pa * LD, *cb = S.R + pb * LD;
          double a1 = 0.0, a2 = 0.0;
#pragma unroll
          for (int i = 0; i < W; i++) {
            const double x = ca[i], y = cb[i];
            a1 = fma(x, x, a1);
            a2 = fma(x, y, a2);
          }
          hpp = a1;
          hpq = a2;
          hqq = __shfl_down_sync(0xffffffffu, a1, HALF);
        }
#endif
        if (lane < HALF) {
#if JH_I5_PREF
          const int p = p_next, q = q_next;
          {
            const int8_t *stn = S.steps + (si + 1 < NSTEP ? si + 1 : 0) * W;
            p_next = stn[2 * lane];
            q_next = stn[2 * lane + 1];
          }
#else
          const int p = st[2 * lane], q = st[2 * lane + 1];
#endif
#if !JH_I5_SPLIT
          const double *cp = S.R + p * LD, *cq = S.R + q * LD;
          double hpp = 0.0, hqq = 0.0, hpq = 0.0;
#pragma unroll kI5DotUnroll
          for (int i = 0; i < W; i++) {
            const double gp = cp[i], gq = cq[i];
            hpp = fma(gp, gp, hpp);
            hqq = fma(gq, gq, hqq);
            hpq = fma(gp, gq, hpq);
          }
#endif
          StepParams5 pr{1.0, 0.0, 0};
          // the rotation is formed speculatively, in parallel with the
          // orthogonality test (it has no side effects; a pair that passes
          // the test discards it, exactly like the reference never forms it)
#if JH_I5_PROF
          asm volatile("" ::"d"(hpp), "d"(hqq), "d"(hpq));
#endif
          I5_LAP(p5_dots);
          const bool hyp = S.sg[p] > 0 && S.sg[q] < 0;
          // branch-free fast paths of the IEEE division / square root
          // (jh_fastmath.cuh; the IEEE operators when an operand leaves
          // their range): bitwise the same values, without the seven
          // serialised slow-path regions
          double cs, tn, sp, sq;
          bool fast_ok;
          bool rot_ok = rotation_core_fast(hpp, hqq, hpq, hyp ? -1.0 : 1.0, cs, tn, sp, sq,
                                           fast_ok);
          if (!fast_ok) {
            // out of the fast paths' range (e.g. hpq == 0): IEEE operators,
            // the rotation only when the pair is rotated
            sp = sqrt(hpp);
            sq = sqrt(hqq);
          }
          if (hpp == 0.0) {
            fail = kZeroColumn;
            fb = p + 1;
          } else if (hqq == 0.0) {
            fail = kZeroColumn;
            fb = q + 1;
          } else if (!(fabs(hpq) < tol_c * sp * sq)) {
            if (!fast_ok) rot_ok = rotation_core(hpp, hqq, hpq, hyp ? -1.0 : 1.0, cs, tn);
            if (!rot_ok) {
              fail = kHypDomain;
              fb = p + 1;
            } else {
              a_r++;
              if (cs != 1.0) b_r++;
              pr.cs = cs;
              pr.tn = tn;
              pr.act = hyp ? 5 : 1;
              if (!hyp) {
                const double h1 = fma(-tn, hpq, hpp);
                const double h2 = fma(tn, hpq, hqq);
                if ((S.sg[p] > 0 && h1 < h2) || (S.sg[p] < 0 && h1 > h2)) pr.act = 2;
              }
            }
          }
          cur[lane] = pr;
          I5_LAP(p5_rot);
        }
        const unsigned fm = __ballot_sync(0xffffffffu, fail != 0);
        if (fm) {
          const int first = __ffs(fm) - 1;  // first failing pair in reference order
          const int fs = __shfl_sync(0xffffffffu, fail, first);
          const int fbb = __shfl_sync(0xffffffffu, fb, first);
          if (lane == 0) {
            S.fail_status = fs;
            S.fail_bad = fbb;
            S.stop = 1;
          }
        }
      } else if (gstep > 0) {
        // lagged V update of the previous inner p-step (warps 1..)
        const int8_t *pst = S.steps + ((si + NSTEP - 1) % NSTEP) * W;
        const StepParams5 *prev = S.prm[(gstep - 1) & 1];
        const int vt = tid - 32, vrow = vt % W, vg = vt / W;
        constexpr int VGS = (NTH - 32) / W;
        if (vt < VGS * W)
          for (int pi = vg; pi < HALF; pi += VGS)
            if (prev[pi].act) rot_apply5(S.V, LD, pst[2 * pi], pst[2 * pi + 1], vrow, prev[pi]);
      }
      __syncthreads();
      I5_LAP(p5_bar1);
      if (S.stop) {
        status = S.fail_status;
        bad = S.fail_bad;
        break;
      }
      // R update of this inner p-step (all threads); the per-pair loop
      // (JH_I5_ROLLED, default) keeps K2 at 104 registers and measured as
      // fast as the batched form at n = 16384 (275 vs 285 us per launch)
#if JH_I5_ROLLED == 2
      for (int pi = rg; pi < HALF; pi += RGS)
        if (cur[pi].act) rot_apply5(S.R, LD, st[2 * pi], st[2 * pi + 1], ri, cur[pi]);
#elif JH_I5_ROLLED == 1
      rot_apply_pair<W, HALF, NTH>(S.R, LD, st, cur, tid);
#else
      rot_apply_rows<HALF, RGS>(S.R, LD, st, cur, rg, ri);
#endif
      __syncthreads();
      I5_LAP(p5_app);
    }
    if (status) break;
    // sweep end: totals of applied / proper rotations
    if (warp == 0) {
      const int ta = __reduce_add_sync(0xffffffffu, a_r);
      const int tb = __reduce_add_sync(0xffffffffu, b_r);
      a_r = b_r = 0;
      if (lane == 0) {
        S.sweep_rot = ta;
        S.sweep_proper = tb;
      }
    }
    __syncthreads();
    const int ta = S.sweep_rot, tb = S.sweep_proper;
    __syncthreads();
    sweeps++;
    tot_rot += ta;
    tot_proper += tb;
    if (ta == 0) break;
  }
  if (status) {
    if (tid == 0) {
      *rot_out = 0;
      atomicMin(&counters[2], err_key(pstep, task_key, status, bad));
    }
    return -1;
  }
  // flush the lagged V update of the last inner p-step
  if (gstep > 0) {
    const int last = (gstep - 1) % NSTEP;
    const int8_t *pst = S.steps + last * W;
    const StepParams5 *prev = S.prm[(gstep - 1) & 1];
    rot_apply_rows<HALF, RGS>(S.V, LD, pst, prev, rg, ri);
  }
  __syncthreads();
  for (int e = tid; e < W * W; e += NTH) {
    const int j = e / W, i = e - j * W;
    Vg[e] = S.V[j * LD + i];
  }
#if JH_I5_PROF
  if (tid == 0 && g_i5_on) {
    atomicAdd(&g_i5[1], p5_dots);
    atomicAdd(&g_i5[2], p5_rot);
    atomicAdd(&g_i5[3], p5_bar1);
    atomicAdd(&g_i5[4], p5_app);
    atomicAdd(&g_i5[5], (unsigned long long)gstep);
    atomicAdd(&g_i5[6], (unsigned long long)sweeps);
    atomicAdd(&g_i5[7], 1ull);
    atomicAdd(&g_i5[8], (unsigned long long)(clock64() - t5_task));
  }
#endif
  if (tid == 0) {
    *rot_out = tot_rot;
    atomicAdd(&counters[0], (unsigned long long)tot_rot);
    atomicAdd(&counters[1], (unsigned long long)tot_proper);
    if (tot_rot) atomicAdd(&counters[3], 1ull);
  }
  return tot_rot;
}

}  // namespace jh
