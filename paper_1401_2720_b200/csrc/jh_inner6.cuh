// Inner Jacobi of one task, variant 6 (w <= 32): warp 0 alone carries the
// serial chain, the other warps apply the rotations to V behind it.
//
// Reference: blockkernel.py:110-145 (Cholesky) and 278-334 (inner sweeps).
// The arithmetic per element is that of variant 5 (jh_inner5.cuh), so the
// results are bitwise the same; only the schedule differs:
//  * Cholesky by warp 0 with lane x holding column x of the triangle in
//    registers: element (j, x) still receives its updates for k = 0..j-1 in
//    order, then the square root (diagonal) or the division by l_j -- the
//    right-looking element order of the reference, with shuffles instead of
//    three CTA barriers per column.
//  * Inner p-step s: lane i < w/2 owns pair i.  It forms its two columns of
//    R after step s-1 on the fly from the columns of R before step s-1 and
//    the step-(s-1) rotation parameters (double-buffered R), stores them for
//    step s+1 and runs the three dot-product chains on them; then the
//    rotation and the test.  No CTA barrier per step: warp 0 hands each
//    step's parameters to warps 1.. through a ring of mbarrier-guarded slots,
//    and those warps rotate V in step order.
#pragma once

#include "jh_common.cuh"
#include "jh_fastmath.cuh"
#include "jh_dmma.cuh"
#include "jh_inner5.cuh"

namespace jh {

constexpr int kI6Ring = 4;  // parameter slots between warp 0 and the V warps

template <int W>
struct InnerSmem6 {
  double R[2][W * (W + 1)];
  double V[W * (W + 1)];
  StepParams5 prm[kI6Ring][W / 2];
  int8_t steps[(W - 1) * W];  // (p, q) per pair per inner p-step
  int8_t own[(W - 1) * W];    // per inner p-step and column: 2 * pair + (column is q)
  int8_t sg[W];
  int sidx[kI6Ring];          // table row of the slot's p-step; -1 = no more p-steps
  uint64_t full[kI6Ring], empty[kI6Ring];
  int chol;
  long long result;
};

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Returns the task's rotation count (>= 0; V' written to Vg column-major,
// counters updated) or -1 after recording a numerical failure under key
// (pstep, task_key).  smem must hold an InnerSmem6<W>.  All NTH threads call.
template <int W, int NTH>
__device__ __forceinline__ long long inner6_task(unsigned char *smem, const double *__restrict__ Hg,
                                              double *__restrict__ Vg, int p0, int q0,
                                              int64_t n_plus, const int32_t *__restrict__ inner,
                                              int inner_limit, double tol_c,
                                              unsigned long long *counters, int pstep,
                                              int task_key, int64_t *rot_out,
                                              bool from_r = false) {
  static_assert(W <= 32 && W % 2 == 0, "variant 6 needs w <= 32");
  constexpr int HALF = W / 2, LD = W + 1, BW = W / 2, NSTEP = W - 1;
  InnerSmem6<W> &S = *reinterpret_cast<InnerSmem6<W> *>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr unsigned FULL = 0xffffffffu;
  // the chain warp rotates with the task index, so that the chain warps of
  // the CTAs sharing an SM do not all land on the same SM sub-partition
  const int cw = (int)(blockIdx.x % (NTH / 32));
  const bool chain = warp == cw;
  const int vwarp = warp < cw ? warp : warp - 1;  // index among the V warps
  // phase timing (jh_inner5_profile): thread 0 [Cholesky, empty-slot wait,
  // columns + dots, rotation + test], thread 32 [full-slot wait]
  const bool prof = g_i5_on && lane == 0 && (chain || vwarp == 0);
  long long t_task = prof ? clock64() : 0, t_mark = t_task;
  unsigned long long pc[5] = {0, 0, 0, 0, 0};
  auto lap = [&](int k) {
    if (prof) {
      const long long now = clock64();
      pc[k] += (unsigned long long)(now - t_mark);
      t_mark = now;
    }
  };

  // ---- tables, signs, V = I, barriers (all threads)
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
  for (int j = tid; j < HALF; j += NTH) S.prm[kI6Ring - 1][j] = StepParams5{1.0, 0.0, 0};
  if (tid == 0) {
    for (int s = 0; s < kI6Ring; s++) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    fence_mbar_init();
  }

  // ---- R: Cholesky of H (chain warp), or the given factor
  long long t_setup = prof ? clock64() : 0;
  if (chain) {
    const int x = lane;
    if (from_r) {
      if (x < W)
#pragma unroll
        for (int i = 0; i < W; i++) S.R[0][x * LD + i] = __ldcg(Hg + x * W + i);
      if (lane == 0) S.chol = 0;
    } else {
      const int chol = chol6_warp<W>(Hg, S.R[0], S.R[1], lane);
      if (lane == 0) S.chol = chol;
      if (prof) {
        atomicAdd(&g_i5[10], (unsigned long long)(t_setup - t_task));
        atomicAdd(&g_i5[11], (unsigned long long)(clock64() - t_setup));
      }
    }
  }
  __syncthreads();
  lap(0);
  if (S.chol) {
    if (tid == 0) {
      *rot_out = 0;
      atomicMin(&counters[2], err_key(pstep, task_key, kCholesky, S.chol));
    }
    return -1;
  }
  int prof_steps = 0, prof_sweeps = 0;

  if (chain) {
    // ---- the serial chain: dots, rotation, test per inner p-step
    int a_r = 0, b_r = 0;
    int64_t tot_rot = 0, tot_proper = 0;
    int sweeps = 0, status = 0, bad = -1;
    int gstep = 0;
    for (int sw = 0; sw < inner_limit && !status; sw++) {
      for (int si = 0; si < NSTEP; si++, gstep++) {
        const int slot = gstep % kI6Ring, pslot = (gstep + kI6Ring - 1) % kI6Ring;
        if (gstep >= kI6Ring) mbar_wait(&S.empty[slot], (uint32_t)(((gstep / kI6Ring) - 1) & 1));
        lap(1);
        const double *Rin = S.R[gstep & 1];
        double *Rout = S.R[(gstep + 1) & 1];
        const int spi = (si + NSTEP - 1) % NSTEP;
        int fail = 0, fb = 0;
        StepParams5 pr{1.0, 0.0, 0};
        if (lane < HALF) {
          const int p = S.steps[si * W + 2 * lane], q = S.steps[si * W + 2 * lane + 1];
          // sources of the new columns p and q: new = keep ? old[a]
          //                                             : fma(coef, old[b], old[a]) * cs
          int ca[2], cb[2];
          double coef[2], csv[2];
          bool keep[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int c = h ? q : p;
            const int o = S.own[spi * W + c], pp = o >> 1, role = o & 1;
            const StepParams5 P = S.prm[pslot][pp];
            const int a0 = S.steps[spi * W + 2 * pp], b0 = S.steps[spi * W + 2 * pp + 1];
            keep[h] = P.act == 0;
            // np = fma(s, gq, gp) [* cs], nq = fma(tn, gp, gq) [* cs]; a swap
            // exchanges them; s = -tn (trigonometric) or +tn (hyperbolic)
            const bool want_np = (role == 0) != ((P.act & 3) == 2);
            const double s = (P.act & 4) ? P.tn : -P.tn;
            ca[h] = keep[h] ? c : (want_np ? a0 : b0);
            cb[h] = keep[h] ? c : (want_np ? b0 : a0);
            coef[h] = want_np ? s : P.tn;
            csv[h] = P.cs;
          }
          const double *ap = Rin + ca[0] * LD, *bp = Rin + cb[0] * LD;
          const double *aq = Rin + ca[1] * LD, *bq = Rin + cb[1] * LD;
          double *op = Rout + p * LD, *oq = Rout + q * LD;
          double hpp = 0.0, hqq = 0.0, hpq = 0.0;
          // rows in chunks of 8: all loads of a chunk before its stores (the
          // compiler cannot move a load of R_in above a store to R_out)
#pragma unroll 1
          for (int i0 = 0; i0 < W; i0 += 8) {
            double xa[8], xb[8], ya[8], yb[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
              xa[u] = ap[i0 + u];
              xb[u] = bp[i0 + u];
              ya[u] = aq[i0 + u];
              yb[u] = bq[i0 + u];
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
              double gp = fma(coef[0], xb[u], xa[u]), gq = fma(coef[1], yb[u], ya[u]);
              if (csv[0] != 1.0) gp = gp * csv[0];
              if (csv[1] != 1.0) gq = gq * csv[1];
              gp = keep[0] ? xa[u] : gp;
              gq = keep[1] ? ya[u] : gq;
              op[i0 + u] = gp;
              oq[i0 + u] = gq;
              hpp = fma(gp, gp, hpp);
              hqq = fma(gq, gq, hqq);
              hpq = fma(gp, gq, hpq);
            }
          }
          if (prof) {
            asm volatile("" ::"d"(hpp), "d"(hqq), "d"(hpq));
            lap(2);
          }
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
            rot_ok = rotation_core(hpp, hqq, hpq, hyp ? -1.0 : 1.0, cs, tn);
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
          S.prm[slot][lane] = pr;
          lap(3);
        }
        const unsigned fm = __ballot_sync(FULL, fail != 0);
        if (fm) {
          const int first = __ffs(fm) - 1;  // first failing pair in reference order
          status = __shfl_sync(FULL, fail, first);
          bad = __shfl_sync(FULL, fb, first);
          break;
        }
        __syncwarp();
        if (lane == 0) {
          S.sidx[slot] = si;
          mbar_arrive(&S.full[slot]);
        }
      }
      if (status) break;
      const int ta = __reduce_add_sync(FULL, a_r);
      const int tb = __reduce_add_sync(FULL, b_r);
      a_r = b_r = 0;
      sweeps++;
      tot_rot += ta;
      tot_proper += tb;
      if (ta == 0) break;
    }
    prof_steps = gstep;
    prof_sweeps = sweeps;
    // end token for the V warps
    {
      const int slot = gstep % kI6Ring;
      if (gstep >= kI6Ring) mbar_wait(&S.empty[slot], (uint32_t)(((gstep / kI6Ring) - 1) & 1));
      __syncwarp();
      if (lane == 0) {
        S.sidx[slot] = -1;
        mbar_arrive(&S.full[slot]);
      }
    }
    if (lane == 0) {
      if (status) {
        *rot_out = 0;
        atomicMin(&counters[2], err_key(pstep, task_key, status, bad));
        S.result = -1;
      } else {
        *rot_out = tot_rot;
        atomicAdd(&counters[0], (unsigned long long)tot_rot);
        atomicAdd(&counters[1], (unsigned long long)tot_proper);
        if (tot_rot) atomicAdd(&counters[3], 1ull);
        S.result = tot_rot;
      }
    }
  } else {
    // ---- V warps: the rotations of each inner p-step, in order
    constexpr int NV = NTH - 32, VGS = NV / W;
    const int vt = vwarp * 32 + lane, vrow = vt % W, vg = vt / W;
    for (int k = 0;; k++) {
      const int slot = k % kI6Ring;
      if (prof) t_mark = clock64();
      mbar_wait(&S.full[slot], (uint32_t)((k / kI6Ring) & 1));
      lap(4);
      const int si = S.sidx[slot];
      if (si < 0) break;
      const int8_t *pst = S.steps + si * W;
      const StepParams5 *pp = S.prm[slot];
      if (vt < VGS * W) {
        // all loads of the thread's pairs first, then the stores
        constexpr int MP = (HALF + VGS - 1) / VGS;
        double vp[MP], vq[MP];
        StepParams5 P[MP];
        int cp[MP], cq[MP];
#pragma unroll
        for (int u = 0; u < MP; u++) {
          const int pi = vg + u * VGS;
          if (pi < HALF) {
            P[u] = pp[pi];
            cp[u] = pst[2 * pi];
            cq[u] = pst[2 * pi + 1];
            vp[u] = S.V[cp[u] * LD + vrow];
            vq[u] = S.V[cq[u] * LD + vrow];
          }
        }
#pragma unroll
        for (int u = 0; u < MP; u++) {
          const int pi = vg + u * VGS;
          if (pi < HALF && P[u].act) {
            const double cs = P[u].cs, tn = P[u].tn;
            const double sn = (P[u].act & 4) ? tn : -tn;
            double np = fma(sn, vq[u], vp[u]), nq = fma(tn, vp[u], vq[u]);
            if (cs != 1.0) {
              np = np * cs;
              nq = nq * cs;
            }
            const bool sw = (P[u].act & 3) == 2;
            S.V[cp[u] * LD + vrow] = sw ? nq : np;
            S.V[cq[u] * LD + vrow] = sw ? np : nq;
          }
        }
      }
      named_bar_sync(1, NV);
      if (vt == 0) mbar_arrive(&S.empty[slot]);
    }
  }
  __syncthreads();
  if (prof) {
    for (int k = 0; k < 5; k++) atomicAdd(&g_i5[k], pc[k]);
    if (chain) {
      const unsigned long long tt = (unsigned long long)(clock64() - t_task);
      atomicAdd(&g_i5[5], (unsigned long long)prof_steps);
      atomicAdd(&g_i5[6], (unsigned long long)prof_sweeps);
      atomicAdd(&g_i5[7], 1ull);
      atomicAdd(&g_i5[8], tt);
      atomicMax(&g_i5[9], tt);
    }
  }
  const long long res = S.result;
  if (res >= 0)
    for (int e = tid; e < W * W; e += NTH) {
      const int j = e / W, i = e - j * W;
      Vg[e] = S.V[j * LD + i];
    }
  return res;
}

}  // namespace jh
