// K2: shortening + pointwise Jacobi of one block pair per CTA (latency-bound
// part of the p-step), specialised on the block width W.
//
//   Cholesky     H = L L^T, R = L^T                 (blockkernel.py:110-145)
//   inner sweep  dots -> test -> rotation -> apply  (blockkernel.py:278-334)
//
// Per inner p-step the w/2 pairs' dot products and rotation parameters are
// formed by w/2 lanes of warp 0 (lane = pair, the reference's three in-order
// fma chains over the w rows) while warps 1.. apply the PREVIOUS p-step's
// rotations to V (V is never read by the dot products, so its updates may lag
// one p-step; per column they still happen in reference order).  After a
// barrier all threads rotate (and swap) the pairs' columns of R; a second
// barrier ends the p-step.  Everything lives in shared memory with column
// stride W + 1.
#include "jh_common.cuh"
#include "jh_dmma.cuh"
#include "jh_fastmath.cuh"
#include "jh_kernels.h"

namespace jh {

// optional phase timing of the inner Jacobi (jh_inner_profile): cycles spent
// by warp 0 in [dots, rotation, barrier 1, R apply, barrier 2], the number of
// inner p-steps, inner sweeps and tasks
__device__ int g_inner_prof_on = 0;
__device__ unsigned long long g_inner_prof[8];

template <int W>
struct InnerCfg {
  static constexpr int HALF = W / 2;
  static constexpr int LD = W + 1;
  static constexpr int NTH = W <= 32 ? 128 : 256;
};

struct StepParams {
  double cs, tn;
  int act;  // 0 skip, 1 rotate, 2 rotate + swap, 4 | 1 hyperbolic rotate
};

template <int W>
struct InnerSmem {
  double H[W * W];
  double R[W * (W + 1)];
  double V[W * (W + 1)];
  StepParams prm[2][W / 2];
  int8_t steps[(W - 1) * W];  // (p, q) per pair per inner p-step
  int8_t sg[W];
  int fail_status, fail_bad, stop, sweep_rot, sweep_proper, chol;
};

// rotate (+ swap) columns p, q of M (ld LD) at row i
__device__ __forceinline__ void rot_apply(double *M, int ld, int p, int q, int i,
                                          const StepParams &pr) {
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

// Rotate rows i of the pairs g0, g0 + STRIDE, ... (< HALF) of one inner
// p-step.  All parameters and operands are loaded first (independent
// shared-memory loads in flight together), then the rotated pairs are
// written; a pair that was not rotated is left untouched bit for bit.
template <int HALF, int STRIDE>
__device__ __forceinline__ void apply_rows(double *M, int ld, const int8_t *st,
                                           const StepParams *prm, int g0, int i) {
  constexpr int NP = (HALF + STRIDE - 1) / STRIDE;
  int act[NP], p[NP], q[NP];
  double cs[NP], tn[NP], gp[NP], gq[NP];
#pragma unroll
  for (int k = 0; k < NP; k++) {
    const int pi = g0 + k * STRIDE;
    act[k] = 0;
    if (pi < HALF) {
      act[k] = prm[pi].act;
      cs[k] = prm[pi].cs;
      tn[k] = prm[pi].tn;
      p[k] = st[2 * pi];
      q[k] = st[2 * pi + 1];
    }
  }
#pragma unroll
  for (int k = 0; k < NP; k++)
    if (act[k]) {
      gp[k] = M[p[k] * ld + i];
      gq[k] = M[q[k] * ld + i];
    }
#pragma unroll
  for (int k = 0; k < NP; k++)
    if (act[k]) {
      const double s = (act[k] & 4) ? tn[k] : -tn[k];
      double np = fma(s, gq[k], gp[k]), nq = fma(tn[k], gp[k], gq[k]);
      if (cs[k] != 1.0) {
        np = np * cs[k];
        nq = nq * cs[k];
      }
      const bool sw = (act[k] & 3) == 2;
      M[p[k] * ld + i] = sw ? nq : np;
      M[q[k] * ld + i] = sw ? np : nq;
    }
}

template <int W>
__global__ void __launch_bounds__(InnerCfg<W>::NTH)
k_factor_inner3(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                int64_t n_plus, const int32_t *__restrict__ inner, int inner_limit,
                double tol_c, unsigned long long *counters, int pstep, int task_base) {
  constexpr int HALF = InnerCfg<W>::HALF, LD = InnerCfg<W>::LD, NTH = InnerCfg<W>::NTH;
  constexpr int BW = W / 2, NSTEP = W - 1;
  extern __shared__ __align__(16) unsigned char smraw[];
  InnerSmem<W> &S = *reinterpret_cast<InnerSmem<W> *>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int task = blockIdx.x;
  const int p0 = pairs[2 * task], q0 = pairs[2 * task + 1];

  // ---- load H, inner table, signs; V = I
  const double *Hg = Hbuf + (size_t)task * W * W;
  for (int i = tid; i < W * W; i += NTH) S.H[i] = Hg[i];
  for (int i = tid; i < W * LD; i += NTH) {
    const int col = i / LD, row = i - col * LD;
    S.V[i] = (row == col) ? 1.0 : 0.0;
  }
  for (int i = tid; i < NSTEP * W; i += NTH) S.steps[i] = (int8_t)inner[i];
  for (int j = tid; j < W; j += NTH) {
    const int64_t gcol = (j < BW ? (int64_t)p0 * BW + j : (int64_t)q0 * BW + (j - BW)) + 1;
    S.sg[j] = gcol <= n_plus ? 1 : -1;
  }
  if (tid == 0) {
    S.chol = 0;
    S.stop = 0;
  }
  __syncthreads();

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
          S.H[k * W + k] = sqrt(d);
      }
      __syncthreads();
      if (S.chol) break;
      const double l = S.H[k * W + k];
      if (jg == 0 && x > k) S.H[k * W + x] = S.H[k * W + x] / l;
      __syncthreads();
      for (int j = k + 1 + jg; j < W; j += JS)
        if (x >= j) S.H[j * W + x] = fma(-S.H[k * W + x], S.H[k * W + j], S.H[j * W + x]);
      __syncthreads();
    }
  }
  if (S.chol) {
    if (tid == 0) {
      task_rot[task] = 0;
      atomicMin(&counters[2], err_key(pstep, task_base + task, kCholesky, S.chol));
    }
    return;
  }
  // R = L^T (R[i][j] = H[i * W + j] for i <= j)
  for (int e = tid; e < W * W; e += NTH) {
    const int j = e / W, i = e - j * W;
    S.R[j * LD + i] = (i <= j) ? S.H[i * W + j] : 0.0;
  }
  __syncthreads();

  // ---- inner sweeps
  int a_r = 0, b_r = 0;  // lane-private counters of warp 0
  int64_t tot_rot = 0, tot_proper = 0;
  int sweeps = 0, status = 0, bad = -1;
  int gstep = 0;  // global inner p-step counter (for the lagged V update)
  const int ri = tid % W;         // row handled in the R / V applies
  const int rg = tid / W;         // pair group
  constexpr int RGS = NTH / W;    // pair groups in the R apply
  const bool prof = g_inner_prof_on != 0;
  unsigned long long pt[5] = {0, 0, 0, 0, 0};
  long long c0 = 0, c1 = 0;
  for (int sw = 0; sw < inner_limit && !status; sw++) {
    for (int si = 0; si < NSTEP; si++, gstep++) {
      const int8_t *st = S.steps + si * W;
      StepParams *cur = S.prm[gstep & 1];
      if (prof && tid == 0) c0 = clock64();
      if (warp == 0) {
        int fail = 0, fb = 0;
        if (lane < HALF) {
          const int p = st[2 * lane], q = st[2 * lane + 1];
          const double *cp = S.R + p * LD, *cq = S.R + q * LD;
          double hpp = 0.0, hqq = 0.0, hpq = 0.0;
#pragma unroll
          for (int i = 0; i < W; i++) {
            const double gp = cp[i], gq = cq[i];
            hpp = fma(gp, gp, hpp);
            hqq = fma(gq, gq, hqq);
            hpq = fma(gp, gq, hpq);
          }
          StepParams pr{1.0, 0.0, 0};
          // the rotation is formed speculatively, in parallel with the
          // orthogonality test (it has no side effects; a pair that passes
          // the test discards it, exactly like the reference never forms it)
          if (prof && lane == 0) {
            c1 = clock64() + (long long)(hpp * 0.0);
            pt[0] += c1 - c0;
            c0 = c1;
          }
          const bool hyp = S.sg[p] > 0 && S.sg[q] < 0;
          double cs, tn;
          const bool rot_ok = rotation_core_sel(hpp, hqq, hpq, hyp ? -1.0 : 1.0, cs, tn);
          if (hpp == 0.0) {
            fail = kZeroColumn;
            fb = p + 1;
          } else if (hqq == 0.0) {
            fail = kZeroColumn;
            fb = q + 1;
          } else if (!(fabs(hpq) < tol_c * sqrt(hpp) * sqrt(hqq))) {
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
          if (prof && lane == 0) {
            c1 = clock64();
            pt[1] += c1 - c0;
            c0 = c1;
          }
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
        const StepParams *prev = S.prm[(gstep - 1) & 1];
        const int vt = tid - 32, vrow = vt % W, vg = vt / W;
        constexpr int VGS = (NTH - 32) / W;
        if (vt < VGS * W) apply_rows<HALF, VGS>(S.V, LD, pst, prev, vg, vrow);
      }
      __syncthreads();
      if (prof && tid == 0) {
        c1 = clock64();
        pt[2] += c1 - c0;
        c0 = c1;
      }
      if (S.stop) {
        status = S.fail_status;
        bad = S.fail_bad;
        break;
      }
      // R update of this inner p-step (all threads)
      apply_rows<HALF, RGS>(S.R, LD, st, cur, rg, ri);
      if (prof && tid == 0) {
        c1 = clock64();
        pt[3] += c1 - c0;
        c0 = c1;
      }
      __syncthreads();
      if (prof && tid == 0) pt[4] += clock64() - c0;
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
      task_rot[task] = 0;
      atomicMin(&counters[2], err_key(pstep, task_base + task, status, bad));
    }
    return;
  }
  // flush the lagged V update of the last inner p-step
  if (gstep > 0) {
    const int last = (gstep - 1) % NSTEP;
    const int8_t *pst = S.steps + last * W;
    const StepParams *prev = S.prm[(gstep - 1) & 1];
    apply_rows<HALF, RGS>(S.V, LD, pst, prev, rg, ri);
  }
  __syncthreads();
  double *Vg = Vbuf + (size_t)task * W * W;
  for (int e = tid; e < W * W; e += NTH) {
    const int j = e / W, i = e - j * W;
    Vg[e] = S.V[j * LD + i];
  }
  if (prof && tid == 0) {
    for (int k = 0; k < 5; k++) atomicAdd(&g_inner_prof[k], pt[k]);
    atomicAdd(&g_inner_prof[5], (unsigned long long)gstep);
    atomicAdd(&g_inner_prof[6], (unsigned long long)sweeps);
    atomicAdd(&g_inner_prof[7], 1ull);
  }
  if (tid == 0) {
    task_rot[task] = tot_rot;
    atomicAdd(&counters[0], (unsigned long long)tot_rot);
    atomicAdd(&counters[1], (unsigned long long)tot_proper);
    if (tot_rot) atomicAdd(&counters[3], 1ull);
  }
}

bool inner3_ok(int w) { return w == 16 || w == 32 || w == 64; }

template <int W>
static void launch_inner_t(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                           int ntask, int64_t n_plus, const int32_t *inner, int inner_limit,
                           double tol_c, unsigned long long *counters, int pstep,
                           cudaStream_t st, int task_base) {
  const size_t smem = sizeof(InnerSmem<W>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_factor_inner3<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  k_factor_inner3<W><<<ntask, InnerCfg<W>::NTH, smem, st>>>(Hbuf, Vbuf, trot, pairs, n_plus, inner,
                                                           inner_limit, tol_c, counters, pstep,
                                                           task_base);
}

void launch_inner3(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   int task_base) {
  if (w == 16)
    launch_inner_t<16>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                       counters, pstep, st, task_base);
  else if (w == 32)
    launch_inner_t<32>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                       counters, pstep, st, task_base);
  else
    launch_inner_t<64>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                       counters, pstep, st, task_base);
}

}  // namespace jh

// Enable (1) / disable (0) inner-Jacobi phase timing; when out != NULL,
// copies the 8 accumulated counters (see g_inner_prof) to host memory and
// resets them.
extern "C" int jh_inner_profile(int on, unsigned long long *out) {
  cudaDeviceSynchronize();
  if (out) {
    cudaMemcpyFromSymbol(out, jh::g_inner_prof, sizeof(unsigned long long) * 8);
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(jh::g_inner_prof, z, sizeof(z));
  }
  cudaMemcpyToSymbol(jh::g_inner_prof_on, &on, sizeof(int));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

namespace jh {

// ===========================================================================
// K2 v4 (W = 16, 32): one warp owns R in registers.
//
// Lane group g (LPP = 32 / (W/2) lanes) holds the two columns of pair g of
// the current inner p-step, RPL = W / LPP rows per lane.  Dots: the three
// in-order fma chains run through the group's lanes in row order (partial
// chain in lane k, handed to lane k+1 by a shuffle), so each value is the
// reference's chain; the last lane broadcasts the sums and every lane of the
// group forms the same rotation parameters.  Each lane rotates its rows in
// registers, then the columns are redistributed for the next p-step through
// shared memory with __syncwarp only.  Warp 1 applies the rotations to V
// from a ring of per-step parameters, lagging behind; warps 0 and 1 only
// synchronise through shared counters.  No CTA barrier on the critical path.

constexpr int kRing = 8;

template <int W>
struct Inner4Smem {
  double H[W * W];
  double R[W * (W + 2)];     // column exchange buffer, stride W + 2
  double V[W * (W + 1)];
  StepParams prm[kRing][W / 2];
  int8_t steps[(W - 1) * W];
  int8_t sg[W];
  int chol, status, bad;
  volatile int produced;      // inner p-steps published by warp 0
  volatile int consumed;      // inner p-steps applied to V by warp 1
  volatile int finished;      // warp 0 done: total steps in `produced`
  long long tot_rot;          // rotations of the task (all inner sweeps)
};

// Cholesky + inner sweeps of task `task` by a CTA of NTH >= 64 threads
// (warps 0 and 1 work, others only join the barriers).  On success returns
// true with V' in S.V (stride W + 1) and the task's rotation count in
// S.tot_rot (counters and task_rot updated); on a numerical failure records
// the error key and returns false.
template <int W, int NTH>
__device__ __forceinline__ bool inner4_body(Inner4Smem<W> &S, const double *__restrict__ Hbuf,
                                            int64_t *__restrict__ task_rot,
                                            const int32_t *__restrict__ pairs, int64_t n_plus,
                                            const int32_t *__restrict__ inner, int inner_limit,
                                            double tol_c, unsigned long long *counters,
                                            int pstep, int task_base, int task) {
  constexpr int HALF = W / 2, NSTEP = W - 1, BW = W / 2;
  constexpr int LPP = 32 / HALF;     // lanes per pair
  constexpr int RPL = W / LPP;       // rows per lane
  constexpr int LDR = W + 2, LDV = W + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p0 = pairs[2 * task], q0 = pairs[2 * task + 1];

  const double *Hg = Hbuf + (size_t)task * W * W;
  for (int i = tid; i < W * W; i += NTH) S.H[i] = Hg[i];
  for (int i = tid; i < W * LDV; i += NTH) {
    const int col = i / LDV, row = i - col * LDV;
    S.V[i] = (row == col) ? 1.0 : 0.0;
  }
  for (int i = tid; i < NSTEP * W; i += NTH) S.steps[i] = (int8_t)inner[i];
  for (int j = tid; j < W; j += NTH) {
    const int64_t gcol = (j < BW ? (int64_t)p0 * BW + j : (int64_t)q0 * BW + (j - BW)) + 1;
    S.sg[j] = gcol <= n_plus ? 1 : -1;
  }
  if (tid == 0) {
    S.chol = 0;
    S.status = 0;
    S.produced = 0;
    S.consumed = 0;
    S.finished = 0;
    S.tot_rot = 0;
  }
  __syncthreads();
  // forward-looking Cholesky (reference element order)
  {
    const int x = tid % W, jg = tid / W;
    constexpr int JS = NTH / W;
    for (int k = 0; k < W; k++) {
      if (tid == 0) {
        const double d = S.H[k * W + k];
        if (!(d > 0.0) || !isfinite(d))
          S.chol = k + 1;
        else
          S.H[k * W + k] = sqrt(d);
      }
      __syncthreads();
      if (S.chol) break;
      const double l = S.H[k * W + k];
      if (jg == 0 && x > k) S.H[k * W + x] = S.H[k * W + x] / l;
      __syncthreads();
      for (int j = k + 1 + jg; j < W; j += JS)
        if (x >= j) S.H[j * W + x] = fma(-S.H[k * W + x], S.H[k * W + j], S.H[j * W + x]);
      __syncthreads();
    }
  }
  if (S.chol) {
    if (tid == 0) {
      task_rot[task] = 0;
      atomicMin(&counters[2], err_key(pstep, task_base + task, kCholesky, S.chol));
    }
    return false;
  }
  for (int e = tid; e < W * W; e += NTH) {
    const int j = e / W, i = e - j * W;
    S.R[j * LDR + i] = (i <= j) ? S.H[i * W + j] : 0.0;
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- R owner ----------------
    const int gi = lane / LPP, k = lane % LPP;  // pair, position in the group
    const int r0 = k * RPL;
    int p = S.steps[2 * gi], q = S.steps[2 * gi + 1];
    double cp[RPL], cq[RPL];
#pragma unroll
    for (int r = 0; r < RPL; r++) {
      cp[r] = S.R[p * LDR + r0 + r];
      cq[r] = S.R[q * LDR + r0 + r];
    }
    int64_t tot_rot = 0, tot_proper = 0;
    int gstep = 0, status = 0, bad = -1;
    const bool prof = g_inner_prof_on != 0;
    unsigned long long pt[4] = {0, 0, 0, 0};
    long long c0 = 0, c1 = 0;
    int nsw = 0;
    for (int sw = 0; sw < inner_limit && !status; sw++) {
      int a_r = 0, b_r = 0;
      nsw++;
      for (int si = 0; si < NSTEP; si++, gstep++) {
        if (prof) c0 = clock64();
        // dots: chains through the group's lanes in row order
        double hpp = 0.0, hqq = 0.0, hpq = 0.0;
#pragma unroll
        for (int j = 0; j < LPP; j++) {
          if (k == j) {
#pragma unroll
            for (int r = 0; r < RPL; r++) {
              hpp = fma(cp[r], cp[r], hpp);
              hqq = fma(cq[r], cq[r], hqq);
              hpq = fma(cp[r], cq[r], hpq);
            }
          }
          if (j + 1 < LPP) {
            // hand the partial chains to the next lane of the group
            const int src = gi * LPP + j;
            const double a = __shfl_sync(0xffffffffu, hpp, src);
            const double b = __shfl_sync(0xffffffffu, hqq, src);
            const double c = __shfl_sync(0xffffffffu, hpq, src);
            if (k == j + 1) {
              hpp = a;
              hqq = b;
              hpq = c;
            }
          }
        }
        {
          const int src = gi * LPP + LPP - 1;
          hpp = __shfl_sync(0xffffffffu, hpp, src);
          hqq = __shfl_sync(0xffffffffu, hqq, src);
          hpq = __shfl_sync(0xffffffffu, hpq, src);
        }
        if (prof) {
          c1 = clock64() + (long long)(hpp * 0.0 + hqq * 0.0 + hpq * 0.0);
          pt[0] += c1 - c0;
          c0 = c1;
        }
        const bool hyp = S.sg[p] > 0 && S.sg[q] < 0;
        double cs, tn, sp, sq;
        bool fast_ok;
        bool rot_ok = rotation_core_fast(hpp, hqq, hpq, hyp ? -1.0 : 1.0, cs, tn, sp, sq, fast_ok);
        if (__any_sync(0xffffffffu, !fast_ok)) {
          // some operand left the fast paths' range: IEEE operators throughout
          rot_ok = rotation_core_sel(hpp, hqq, hpq, hyp ? -1.0 : 1.0, cs, tn);
          sp = sqrt(hpp);
          sq = sqrt(hqq);
        }
        int act = 0, fail = 0, fb = 0;
        if (hpp == 0.0) {
          fail = kZeroColumn;
          fb = p + 1;
        } else if (hqq == 0.0) {
          fail = kZeroColumn;
          fb = q + 1;
        } else if (!(fabs(hpq) < tol_c * sp * sq)) {
          if (!rot_ok) {
            fail = kHypDomain;
            fb = p + 1;
          } else {
            act = hyp ? 5 : 1;
            if (!hyp) {
              const double h1 = fma(-tn, hpq, hpp);
              const double h2 = fma(tn, hpq, hqq);
              if ((S.sg[p] > 0 && h1 < h2) || (S.sg[p] < 0 && h1 > h2)) act = 2;
            }
          }
        }
        const unsigned fm = __ballot_sync(0xffffffffu, fail != 0);
        if (fm) {
          const int first = __ffs(fm) - 1;  // lowest pair fails first in reference order
          status = __shfl_sync(0xffffffffu, fail, first);
          bad = __shfl_sync(0xffffffffu, fb, first);
          break;
        }
        if (act && k == 0) {
          a_r++;
          if (cs != 1.0) b_r++;
        }
        if (prof) {
          c1 = clock64() + (long long)(cs * 0.0 + tn * 0.0);
          pt[1] += c1 - c0;
          c0 = c1;
        }
        // publish for the V warp (ring slot free once V consumed step gstep - kRing)
        if (k == 0) {
          while (gstep - S.consumed >= kRing) {
          }
          StepParams pr;
          pr.cs = cs;
          pr.tn = tn;
          pr.act = act;
          S.prm[gstep % kRing][gi] = pr;
        }
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          S.produced = gstep + 1;
        }
        if (prof) {
          c1 = clock64();
          pt[2] += c1 - c0;
          c0 = c1;
        }
        // rotate my rows in registers
        if (act) {
          const double s = (act & 4) ? tn : -tn;
          const bool scale = cs != 1.0, swp = (act & 3) == 2;
#pragma unroll
          for (int r = 0; r < RPL; r++) {
            double np = fma(s, cq[r], cp[r]), nq = fma(tn, cp[r], cq[r]);
            if (scale) {
              np = np * cs;
              nq = nq * cs;
            }
            cp[r] = swp ? nq : np;
            cq[r] = swp ? np : nq;
          }
        }
        // redistribute columns for the next inner p-step
        const int nsi = (si + 1 == NSTEP) ? 0 : si + 1;
#pragma unroll
        for (int r = 0; r < RPL; r++) {
          S.R[p * LDR + r0 + r] = cp[r];
          S.R[q * LDR + r0 + r] = cq[r];
        }
        __syncwarp();  // all columns of this step written
        p = S.steps[nsi * W + 2 * gi];
        q = S.steps[nsi * W + 2 * gi + 1];
#pragma unroll
        for (int r = 0; r < RPL; r++) {
          cp[r] = S.R[p * LDR + r0 + r];
          cq[r] = S.R[q * LDR + r0 + r];
        }
        __syncwarp();
        if (prof) {
          c1 = clock64() + (long long)(cp[RPL - 1] * 0.0);
          pt[3] += c1 - c0;
        }
      }
      if (status) break;
      const int ta = __reduce_add_sync(0xffffffffu, a_r);
      const int tb = __reduce_add_sync(0xffffffffu, b_r);
      tot_rot += ta;
      tot_proper += tb;
      if (ta == 0) break;
    }
    if (lane == 0) {
      S.status = status;
      S.bad = bad;
      __threadfence_block();
      S.finished = 1;
    }
    if (prof && lane == 0) {
      for (int j = 0; j < 4; j++) atomicAdd(&g_inner_prof[j], pt[j]);
      atomicAdd(&g_inner_prof[5], (unsigned long long)gstep);
      atomicAdd(&g_inner_prof[6], (unsigned long long)nsw);
      atomicAdd(&g_inner_prof[7], 1ull);
    }
    if (lane == 0 && !status) {
      S.tot_rot = tot_rot;
      task_rot[task] = tot_rot;
      atomicAdd(&counters[0], (unsigned long long)tot_rot);
      atomicAdd(&counters[1], (unsigned long long)tot_proper);
      if (tot_rot) atomicAdd(&counters[3], 1ull);
    }
  } else if (warp == 1) {
    // ---------------- V applier (warp 1): lane = row ----------------
    int done = 0;
    for (;;) {
      int avail = S.produced;
      if (avail == done) {
        if (S.finished) {
          avail = S.produced;
          if (avail == done) break;
        } else {
          continue;
        }
      }
      __threadfence_block();
      for (; done < avail; done++) {
        const int si = done % NSTEP;
        const int8_t *st = S.steps + si * W;
        const StepParams *pr = S.prm[done % kRing];
        if (lane < W) {
#pragma unroll
          for (int g0 = 0; g0 < 4; g0++) apply_rows<HALF, 4>(S.V, LDV, st, pr, g0, lane);
        }
        __syncwarp();
        if (lane == 0) S.consumed = done + 1;
      }
    }
  }
  __syncthreads();
  if (S.status) {
    if (tid == 0) {
      task_rot[task] = 0;
      atomicMin(&counters[2], err_key(pstep, task_base + task, S.status, S.bad));
    }
    return false;
  }
  return true;
}

template <int W>
__global__ void __launch_bounds__(64)
k_factor_inner4(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                int64_t n_plus, const int32_t *__restrict__ inner, int inner_limit,
                double tol_c, unsigned long long *counters, int pstep, int task_base) {
  constexpr int NTH = 64, LDV = W + 1;
  extern __shared__ __align__(16) unsigned char smraw[];
  Inner4Smem<W> &S = *reinterpret_cast<Inner4Smem<W> *>(smraw);
  const int task = blockIdx.x;
  if (!inner4_body<W, NTH>(S, Hbuf, task_rot, pairs, n_plus, inner, inner_limit, tol_c, counters,
                           pstep, task_base, task))
    return;
  double *Vg = Vbuf + (size_t)task * W * W;
  for (int e = threadIdx.x; e < W * W; e += NTH) {
    const int j = e / W, i = e - j * W;
    Vg[e] = S.V[j * LDV + i];
  }
}

bool inner4_ok(int w) { return w == 16 || w == 32; }

template <int W>
static void launch_inner4_t(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                            int ntask, int64_t n_plus, const int32_t *inner, int inner_limit,
                            double tol_c, unsigned long long *counters, int pstep,
                            cudaStream_t st, int task_base) {
  const size_t smem = sizeof(Inner4Smem<W>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_factor_inner4<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  k_factor_inner4<W><<<ntask, 64, smem, st>>>(Hbuf, Vbuf, trot, pairs, n_plus, inner, inner_limit,
                                              tol_c, counters, pstep, task_base);
}

void launch_inner4(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int w, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   int task_base) {
  if (w == 16)
    launch_inner4_t<16>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                        counters, pstep, st, task_base);
  else
    launch_inner4_t<32>(Hbuf, Vbuf, trot, pairs, ntask, n_plus, inner, inner_limit, tol_c,
                        counters, pstep, st, task_base);
}

}  // namespace jh
