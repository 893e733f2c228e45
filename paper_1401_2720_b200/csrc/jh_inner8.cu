// K2 for w = 32 with the factor in registers: one warp per task, lane j owns
// column j of R and of V' for the whole inner solve.
//
// The pairs of an inner p-step are disjoint, so each lane has exactly one
// partner per step.  Both lanes of a pair fetch the partner's column with
// 32 shuffles, run the reference's three in-order fma chains over the 32
// rows (hpp, hqq, hpq: blockkernel.py:299-304; the lane that owns q forms
// the same chains with the roles of its own and its partner's values
// swapped), evaluate the same guarded rotation (rotation.py:90-102, through
// the branch-free IEEE fast paths of jh_fastmath.cuh) and the same sorting
// test, and then each lane writes the new value of its own column:
// gp' = fma(s, gq, gp) * cs, gq' = fma(tn, gp, gq) * cs, swapped when the
// sort requires it (blockkernel.py:251-275, 309-328).  Column ownership
// never moves, so an inner p-step needs no shared memory and no barrier:
// the critical path is the chain (32 dependent fmas), the rotation (two
// divisions and two square roots) and one fma + mul per row.  The same
// rotations are applied to the lane's V' column.  Results are bitwise those
// of the shared-memory kernel (jh_inner5.cuh) and of the reference.
#include "jh_inner5.cuh"
#include "jh_kernels.h"

namespace jh {

namespace {

constexpr int kW8 = 32;
constexpr unsigned kFull = 0xffffffffu;

struct Inner8Smem {
  double R[kW8 * (kW8 + 1)];  // Cholesky output, ld W + 1
  double colk[kW8];           // Cholesky scratch
  uint8_t lt[kW8 - 1][kW8];   // per step and column: partner column | (column is q) << 5
  uint8_t pi[kW8 - 1][kW8];   // per step and column: index of its pair in the step
  uint8_t lane_of[kW8];       // lane that holds a (logical) column
  int8_t sg[kW8];
};

// The sorting swap of a pair (blockkernel.py:321-328) exchanges two columns;
// here it exchanges which lane holds which column instead (lane_of), so no
// value moves: each lane computes the new value of its own storage with
// the p or q formula of its current column and, on a swap, takes over the
// partner's column index.
__global__ void __launch_bounds__(32)
k_factor_inner8(const double *__restrict__ Hbuf, double *__restrict__ Vbuf,
                int64_t *__restrict__ task_rot, const int32_t *__restrict__ pairs,
                int64_t n_plus, const int32_t *__restrict__ inner, int inner_limit,
                double tol_c, unsigned long long *counters, int pstep, bool from_r,
                int64_t *done, int64_t epoch, const int32_t *__restrict__ gblock) {
  constexpr int W = kW8, HALF = W / 2, NSTEP = W - 1, BW = W / 2, LD = W + 1;
  __shared__ Inner8Smem S;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int task = blockIdx.x, lane = threadIdx.x;
  const double *Hg = Hbuf + (size_t)task * W * W;
  double *Vg = Vbuf + (size_t)task * W * W;
  const int p0 = pairs[2 * task], q0 = pairs[2 * task + 1];
  {
    const int64_t gp = gblock ? gblock[p0] : p0, gq = gblock ? gblock[q0] : q0;
    const int64_t gcol = (lane < BW ? gp * BW + lane : gq * BW + (lane - BW)) + 1;
    S.sg[lane] = gcol <= n_plus ? 1 : -1;
    S.lane_of[lane] = (uint8_t)lane;
  }
  for (int si = 0; si < NSTEP; si++) {
    if (lane < HALF) {
      const int p = inner[(si * HALF + lane) * 2], q = inner[(si * HALF + lane) * 2 + 1];
      S.lt[si][p] = (uint8_t)q;
      S.lt[si][q] = (uint8_t)(p | 32);
      S.pi[si][p] = (uint8_t)lane;
      S.pi[si][q] = (uint8_t)lane;
    }
  }
  double col[W], vc[W];
  int status = 0, bad = 0;
  if (!from_r) {
    const int c = chol6_warp<W>(Hg, S.R, S.colk, lane);
    if (c) {
      status = kCholesky;
      bad = c;
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < W; i++) {
    col[i] = from_r ? __ldcg(Hg + lane * W + i) : S.R[lane * LD + i];
    vc[i] = (i == lane) ? 1.0 : 0.0;
  }
  int me = lane;  // the column this lane holds
  int64_t tot_rot = 0, tot_proper = 0;
  // V' rotations run one inner p-step late: the update of p-step k is issued
  // beside the rotation parameters of p-step k + 1 (a ~350-cycle dependent
  // chain of divisions and square roots that leaves the FP64 pipe idle), in
  // the same order per column.  A lane without a pending update applies
  // fma(0, o, v) * 1 = v (V' entries are never -0.0), so the block is
  // unconditional and the scheduler can interleave it.
  double pc1 = 0.0, pcs = 1.0;
  int ppartner = lane;
  auto v_apply = [&]() {
#pragma unroll
    for (int i = 0; i < W; i++) {
      const double o = __shfl_sync(kFull, vc[i], ppartner);
      vc[i] = fma(pc1, o, vc[i]) * pcs;
    }
    pc1 = 0.0;
    pcs = 1.0;
    ppartner = lane;
  };
  if (!status) {
    for (int sw = 0; sw < inner_limit; sw++) {
      int a_r = 0, b_r = 0;
#pragma unroll 1
      for (int si = 0; si < NSTEP; si++) {
        const int ent = S.lt[si][me], mypi = S.pi[si][me];
        const int pcol = ent & 31;           // partner column
        const bool isq = (ent >> 5) != 0;    // this lane holds the pair's q
        const int partner = S.lane_of[pcol];
        double oth[W];
#pragma unroll
        for (int i = 0; i < W; i++) oth[i] = __shfl_sync(kFull, col[i], partner);
        double own2 = 0.0, oth2 = 0.0, cross = 0.0;
#pragma unroll
        for (int i = 0; i < W; i++) {
          own2 = fma(col[i], col[i], own2);
          oth2 = fma(oth[i], oth[i], oth2);
          cross = fma(col[i], oth[i], cross);
        }
        const double hpp = isq ? oth2 : own2, hqq = isq ? own2 : oth2, hpq = cross;
        const int p = isq ? pcol : me, q = isq ? me : pcol;
        const bool hyp = S.sg[p] > 0 && S.sg[q] < 0;
        double cs, tn, sp, sq;
        bool fast_ok;
        bool rot_ok = rotation_core_fast(hpp, hqq, hpq, hyp ? -1.0 : 1.0, cs, tn, sp, sq,
                                         fast_ok);
        v_apply();  // the previous p-step's V' rotations
        if (!fast_ok) {
          sp = sqrt(hpp);
          sq = sqrt(hqq);
        }
        int fail = 0, fb = 0, act = 0;
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
            act = 1;
            if (!isq) {
              a_r++;
              if (cs != 1.0) b_r++;
            }
            if (!hyp) {
              const double h1 = fma(-tn, hpq, hpp);
              const double h2 = fma(tn, hpq, hqq);
              if ((S.sg[p] > 0 && h1 < h2) || (S.sg[p] < 0 && h1 > h2)) act = 2;
            }
          }
        }
        if (__any_sync(kFull, fail != 0)) {
          // the first failing pair in the reference's order
          const int first = __reduce_min_sync(kFull, fail ? mypi : 99);
          const unsigned who = __ballot_sync(kFull, fail && mypi == first && !isq);
          const int src = __ffs(who) - 1;
          status = __shfl_sync(kFull, fail, src);
          bad = __shfl_sync(kFull, fb, src);
          break;
        }
        if (act) {
          // gp' = fma(s, gq, gp) cs, gq' = fma(tn, gp, gq) cs with s = -tn
          // (trig) or tn (hyperbolic); the * cs is skipped when cs == 1
          const double c1 = isq ? tn : (hyp ? tn : -tn);
          const bool scale = cs != 1.0;
#pragma unroll
          for (int i = 0; i < W; i++) {
            double v = fma(c1, oth[i], col[i]);
            if (scale) v = v * cs;
            col[i] = v;
          }
          pc1 = c1;  // V' in the next p-step (v_apply)
          pcs = scale ? cs : 1.0;
          ppartner = partner;
          if (act == 2) {  // sorting swap: the lanes trade columns
            me = pcol;
            S.lane_of[me] = (uint8_t)lane;
          }
        }
        __syncwarp();
      }
      if (status) break;
      v_apply();  // the sweep's last p-step
      const int ta = __reduce_add_sync(kFull, a_r);
      const int tb = __reduce_add_sync(kFull, b_r);
      tot_rot += ta;
      tot_proper += tb;
      if (ta == 0) break;
    }
  }
  if (status) {
    if (lane == 0) {
      task_rot[task] = 0;
      atomicMin(&counters[2], err_key(pstep, task, status, bad));
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; i++) Vg[me * W + i] = vc[i];
    if (lane == 0) {
      task_rot[task] = tot_rot;
      atomicAdd(&counters[0], (unsigned long long)tot_rot);
      atomicAdd(&counters[1], (unsigned long long)tot_proper);
      if (tot_rot) atomicAdd(&counters[3], 1ull);
    }
  }
  if (done) {
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(done + task), "l"(epoch) : "memory");
      int64_t *rl = done + gridDim.x;
      const unsigned long long k = atomicAdd((unsigned long long *)rl, 1ull);
      asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(rl + 1 + k),
                   "l"((epoch << 24) | task) : "memory");
    }
  }
}

}  // namespace

bool inner8_ok(int w) { return w == kW8; }

void launch_inner8(const double *Hbuf, double *Vbuf, int64_t *trot, const int32_t *pairs,
                   int ntask, int64_t n_plus, const int32_t *inner, int inner_limit,
                   double tol_c, unsigned long long *counters, int pstep, cudaStream_t st,
                   bool from_r, int64_t *done, int64_t epoch, const int32_t *gblock) {
  k_factor_inner8<<<ntask, 32, 0, st>>>(Hbuf, Vbuf, trot, pairs, n_plus, inner, inner_limit,
                                        tol_c, counters, pstep, from_r, done, epoch, gblock);
}

}  // namespace jh
