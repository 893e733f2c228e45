// Inner Jacobi of one task, variant 7 (w <= 32): one CTA barrier per inner
// p-step instead of two.
//
// Reference: blockkernel.py:110-145 (Cholesky) and 278-334 (inner sweeps);
// the arithmetic per element is that of variant 5 (jh_inner5.cuh), so the
// results are bitwise the same.  Schedule of inner p-step t:
//  * warp 0 forms the columns of R_t = rot_{t-1}(R_{t-1}) it needs on the
//    fly from the stored R_{t-1} and the step-(t-1) parameters (lane i < w/2
//    the pair's column p, lane i + w/2 its column q; the two swap values
//    with a shuffle), runs the three dot-product chains of pair i in lane i
//    and forms the rotation and the test;
//  * meanwhile warps 1.. store R_t = rot_{t-1}(R_{t-1}) into the other R
//    buffer and apply rot_{t-1} to V';
//  * one __syncthreads, then the buffers swap.
// So the stored-R update and the V update both leave the critical path,
// which is warp 0's chains and rotation.
#pragma once

#include "jh_inner5.cuh"

namespace jh {

template <int W>
struct InnerSmem7 {
  double H[W * W];           // Cholesky scratch
  double R[2][W * (W + 1)];  // R_{t-1} / R_t
  double V[W * (W + 1)];
  StepParams5 prm[2][W / 2];
  int8_t steps[(W - 1) * W];  // (p, q) per pair per inner p-step
  int8_t own[(W - 1) * W];    // per inner p-step and column: 2 * pair + (column is q)
  int8_t sg[W];
  int fail_status, fail_bad, stop, sweep_rot, sweep_proper, chol;
};

// Rotations of one inner p-step by the NVT threads of warps 1..: element e
// = (pair e / W, row e % W); all loads of a thread before its stores.  R:
// out of place (every element written, pairs without rotation copied); V:
// in place (rotated pairs only).  Same arithmetic as rot_apply5.
template <int W, int HALF, int NVT, bool OUT_OF_PLACE>
__device__ __forceinline__ void rot_step_batch(const double *Min, double *Mout, int ld,
                                               const int8_t *pst, const StepParams5 *prm,
                                               int vt) {
  constexpr int NE = HALF * W, MP = (NE + NVT - 1) / NVT;
  constexpr int CH = 3;  // elements per batch (register budget)
#pragma unroll
  for (int u0 = 0; u0 < MP; u0 += CH) {
    double gp[CH], gq[CH], cs[CH], tn[CH];
    int cp[CH], cq[CH], act[CH];
#pragma unroll
    for (int k = 0; k < CH; k++) {
      const int e = vt + (u0 + k) * NVT;
      act[k] = 0;
      if (u0 + k < MP && e < NE) {
        const int pi = e / W, i = e - pi * W;
        act[k] = prm[pi].act;
        cs[k] = prm[pi].cs;
        tn[k] = prm[pi].tn;
        cp[k] = pst[2 * pi] * ld + i;
        cq[k] = pst[2 * pi + 1] * ld + i;
        if (OUT_OF_PLACE || act[k]) {
          gp[k] = Min[cp[k]];
          gq[k] = Min[cq[k]];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < CH; k++) {
      const int e = vt + (u0 + k) * NVT;
      if (u0 + k < MP && e < NE && (OUT_OF_PLACE || act[k])) {
        double np = gp[k], nq = gq[k];
        if (act[k]) {
          const double sn = (act[k] & 4) ? tn[k] : -tn[k];
          np = fma(sn, gq[k], gp[k]);
          nq = fma(tn[k], gp[k], gq[k]);
          if (cs[k] != 1.0) {
            np = np * cs[k];
            nq = nq * cs[k];
          }
          if ((act[k] & 3) == 2) {
            const double x = np;
            np = nq;
            nq = x;
          }
        }
        Mout[cp[k]] = np;
        Mout[cq[k]] = nq;
      }
    }
  }
}

template <int W, int NTH>
__device__ __noinline__ long long inner7_task(unsigned char *smem, const double *__restrict__ Hg,
                                              double *__restrict__ Vg, int p0, int q0,
                                              int64_t n_plus, const int32_t *__restrict__ inner,
                                              int inner_limit, double tol_c,
                                              unsigned long long *counters, int pstep,
                                              int task_key, int64_t *rot_out,
                                              bool from_r = false) {
  static_assert(W <= 32 && W % 2 == 0, "variant 7 needs w <= 32");
  constexpr int HALF = W / 2, LD = W + 1, BW = W / 2, NSTEP = W - 1;
  InnerSmem7<W> &S = *reinterpret_cast<InnerSmem7<W> *>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr unsigned FULL = 0xffffffffu;

  // ---- tables, signs, V = I
  for (int i = tid; i < W * LD; i += NTH) {
    const int col = i / LD, row = i - col * LD;
    S.V[i] = (row == col) ? 1.0 : 0.0;
  }
  for (int e = tid; e < NSTEP * HALF; e += NTH) {
    const int si = e / HALF, pi = e - si * HALF;
    const int p = inner[si * W + 2 * pi], q = inner[si * W + 2 * pi + 1];
    S.steps[si * W + 2 * pi] = (int8_t)p;
    S.steps[si * W + 2 * pi + 1] = (int8_t)q;
    S.own[si * W + p] = (int8_t)(2 * pi);
    S.own[si * W + q] = (int8_t)(2 * pi + 1);
  }
  for (int j = tid; j < W; j += NTH) {
    const int64_t gcol = (j < BW ? (int64_t)p0 * BW + j : (int64_t)q0 * BW + (j - BW)) + 1;
    S.sg[j] = gcol <= n_plus ? 1 : -1;
  }
  // parameters of "step -1": no rotation
  for (int j = tid; j < HALF; j += NTH) S.prm[1][j] = StepParams5{1.0, 0.0, 0};
  if (tid == 0) S.stop = 0;

  // ---- R_0: Cholesky of H (warp 0) or the given factor
  if (warp == 0) {
    if (from_r) {
      if (lane < W)
#pragma unroll
        for (int i = 0; i < W; i++) S.R[0][lane * LD + i] = __ldcg(Hg + lane * W + i);
      if (lane == 0) S.chol = 0;
    } else {
      const int c = chol6_warp<W>(Hg, S.R[0], S.H, lane);
      if (lane == 0) S.chol = c;
    }
  }
  __syncthreads();
  if (S.chol) {
    if (tid == 0) {
      *rot_out = 0;
      atomicMin(&counters[2], err_key(pstep, task_key, kCholesky, S.chol));
    }
    return -1;
  }

  int a_r = 0, b_r = 0;
  int64_t tot_rot = 0, tot_proper = 0;
  int sweeps = 0, status = 0, bad = -1;
  int gstep = 0;
  const int vt = tid - 32;
  constexpr int NVT = NTH - 32;
  for (int sw = 0; sw < inner_limit && !status; sw++) {
    for (int si = 0; si < NSTEP; si++, gstep++) {
      const double *Rin = S.R[gstep & 1];  // R_{t-1}
      double *Rout = S.R[(gstep + 1) & 1];  // R_t (warps 1..)
      const int spi = (si + NSTEP - 1) % NSTEP;
      const StepParams5 *prev = S.prm[(gstep + 1) & 1];  // step t-1 (or "-1")
      StepParams5 *cur = S.prm[gstep & 1];
      if (warp == 0) {
        int fail = 0, fb = 0;
        const int pi = lane < HALF ? lane : lane - HALF;  // this lane's pair
        const bool is_q = lane >= HALF;
        if (lane < 2 * HALF) {
          const int c = S.steps[si * W + 2 * pi + (is_q ? 1 : 0)];
          // column c of R_t from R_{t-1}: new = keep ? old[a]
          //                                   : fma(coef, old[b], old[a]) [* cs]
          const int o = S.own[spi * W + c], pp = o >> 1, role = o & 1;
          const StepParams5 P = prev[pp];
          const int a0 = S.steps[spi * W + 2 * pp], b0 = S.steps[spi * W + 2 * pp + 1];
          const bool keep = P.act == 0;
          const bool want_np = (role == 0) != ((P.act & 3) == 2);
          const double s = (P.act & 4) ? P.tn : -P.tn;
          const int ca = keep ? c : (want_np ? a0 : b0);
          const int cb = keep ? c : (want_np ? b0 : a0);
          const double coef = want_np ? s : P.tn, cs = P.cs;
          const double *ap = Rin + ca * LD, *bp = Rin + cb * LD;
          double hxx = 0.0, hpq = 0.0;  // hpp (lane < HALF) or hqq; hpq in lane < HALF
#pragma unroll 8
          for (int i = 0; i < W; i++) {
            const double xa = ap[i], xb = bp[i];
            double v = fma(coef, xb, xa);
            if (cs != 1.0) v = v * cs;
            v = keep ? xa : v;
            const double other = __shfl_xor_sync(FULL >> (32 - 2 * HALF), v, HALF);
            hxx = fma(v, v, hxx);
            hpq = fma(is_q ? other : v, is_q ? v : other, hpq);
          }
          const double hqq_other = __shfl_xor_sync(FULL >> (32 - 2 * HALF), hxx, HALF);
          if (!is_q) {
            const double hpp = hxx, hqq = hqq_other;
            const int p = S.steps[si * W + 2 * pi], q = S.steps[si * W + 2 * pi + 1];
            StepParams5 pr{1.0, 0.0, 0};
            const bool hyp = S.sg[p] > 0 && S.sg[q] < 0;
            double csr, tn, sp, sq;
            bool fast_ok;
            bool rot_ok = rotation_core_fast(hpp, hqq, hpq, hyp ? -1.0 : 1.0, csr, tn, sp, sq,
                                             fast_ok);
            if (!fast_ok) {
              rot_ok = rotation_core(hpp, hqq, hpq, hyp ? -1.0 : 1.0, csr, tn);
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
              if (!rot_ok) {
                fail = kHypDomain;
                fb = p + 1;
              } else {
                a_r++;
                if (csr != 1.0) b_r++;
                pr.cs = csr;
                pr.tn = tn;
                pr.act = hyp ? 5 : 1;
                if (!hyp) {
                  const double h1 = fma(-tn, hpq, hpp);
                  const double h2 = fma(tn, hpq, hqq);
                  if ((S.sg[p] > 0 && h1 < h2) || (S.sg[p] < 0 && h1 > h2)) pr.act = 2;
                }
              }
            }
            cur[pi] = pr;
          }
        }
        const unsigned fm = __ballot_sync(FULL, fail != 0);
        if (fm) {
          const int first = __ffs(fm) - 1;  // first failing pair in reference order
          const int fs = __shfl_sync(FULL, fail, first);
          const int fbb = __shfl_sync(FULL, fb, first);
          if (lane == 0) {
            S.fail_status = fs;
            S.fail_bad = fbb;
            S.stop = 1;
          }
        }
      } else {
        // warps 1..: stored R_t and V' <- V' rot_{t-1}
        const int8_t *pst = S.steps + spi * W;
        rot_step_batch<W, HALF, NVT, true>(Rin, Rout, LD, pst, prev, vt);
        if (gstep > 0) rot_step_batch<W, HALF, NVT, false>(S.V, S.V, LD, pst, prev, vt);
      }
      __syncthreads();
      if (S.stop) {
        status = S.fail_status;
        bad = S.fail_bad;
        break;
      }
    }
    if (status) break;
    // sweep end: totals of applied / proper rotations
    if (warp == 0) {
      const int ta = __reduce_add_sync(FULL, a_r);
      const int tb = __reduce_add_sync(FULL, b_r);
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
  // V' <- V' rot of the last inner p-step
  if (gstep > 0) {
    const int last = (gstep - 1) % NSTEP;
    const int8_t *pst = S.steps + last * W;
    const StepParams5 *prev = S.prm[(gstep - 1) & 1];
    for (int e = tid; e < HALF * W; e += NTH) {
      const int pi = e / W, i = e - pi * W;
      if (prev[pi].act) rot_apply5(S.V, LD, pst[2 * pi], pst[2 * pi + 1], i, prev[pi]);
    }
  }
  __syncthreads();
  for (int e = tid; e < W * W; e += NTH) {
    const int j = e / W, i = e - j * W;
    Vg[e] = S.V[j * LD + i];
  }
  if (tid == 0) {
    *rot_out = tot_rot;
    atomicAdd(&counters[0], (unsigned long long)tot_rot);
    atomicAdd(&counters[1], (unsigned long long)tot_proper);
    if (tot_rot) atomicAdd(&counters[3], 1ull);
  }
  return tot_rot;
}

}  // namespace jh
