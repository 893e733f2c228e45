// K3 device code: in-place post-multiplication of one task's pair columns
// of G (rows < m) or V (rows < nv) by V' for one slab of rows (reference
// blockkernel.py:407-428, driver.py:165-173), shared by the per-p-step
// update kernel (jh_tiles.cu) and the mixed G + V-pair update kernel
// (jh_vpair.cu).  See jh_tiles.cu for the design.
#pragma once

#include "jh_gram.cuh"

namespace jh {

constexpr int kUpdStages = 4;
constexpr int kUpdCons = 4;        // consumer warps
constexpr int kUpdSlab = 2048;     // rows per CTA

// the body of one CTA (task, slab_y); ring = kUpdStages x W x kLd doubles of
// shared memory, full / empty = kUpdStages mbarriers each (shared with the
// mixed update kernel of jh_vpair.cu)
template <int W, int STAGES = kUpdStages, int RCH = kRch>
__device__ __forceinline__ void update_tma_cta(double *__restrict__ G, int64_t ldg, int64_t m,
                                               double *__restrict__ V, int64_t ldv, int64_t nv,
                                               const int32_t *__restrict__ pairs,
                                               const double *__restrict__ Vbuf,
                                               const int64_t *__restrict__ trot, int nslab_g,
                                               int slab_rows,
                                               int task, int slab_y, double *ring,
                                               uint64_t *full, uint64_t *empty) {
  constexpr int NT = W / 8, NK = W / 4, BW = W / 2, LD = RCH + 4;
  constexpr int RB = RCH / (8 * kUpdCons);  // 8-row blocks per consumer warp and chunk
  static_assert(RCH % (8 * kUpdCons) == 0, "chunk rows");
  if (trot[task] == 0) return;
  const int p = pairs[2 * task], q = pairs[2 * task + 1];
  double *A;
  int64_t ld, rows, s0;
  if (slab_y < nslab_g) {
    A = G; ld = ldg; rows = m; s0 = (int64_t)slab_y * slab_rows;
  } else {
    A = V; ld = ldv; rows = nv; s0 = (int64_t)(slab_y - nslab_g) * slab_rows;
  }
  const int64_t s1 = min64(s0 + slab_rows, rows);
  const int nchunk = (int)cdiv(s1 - s0, RCH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kUpdCons);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    // producer
    for (int c = 0; c < nchunk; c++) {
      const int s = c % STAGES;
      if (c >= STAGES) mbar_wait(&empty[s], (uint32_t)(((c / STAGES) - 1) & 1));
      const int64_t r0 = s0 + (int64_t)c * RCH;
      const uint32_t bytes = (uint32_t)min64(RCH, s1 - r0) * 8u;
      if (lane == 0) mbar_expect_tx(&full[s], bytes * W);
      __syncwarp();
      for (int j = lane; j < W; j += 32) {
        const int64_t col = j < BW ? (int64_t)p * BW + j : (int64_t)q * BW + (j - BW);
        bulk_g2s(ring + ((size_t)s * W + j) * LD, A + col * ld + r0, bytes, &full[s]);
      }
    }
    return;
  }
  // consumers
  const int cw = warp - 1;
  const double *Vt = Vbuf + (size_t)task * W * W;
  double bf[NK][NT];
#pragma unroll
  for (int kk = 0; kk < NK; kk++)
#pragma unroll
    for (int Y = 0; Y < NT; Y++) bf[kk][Y] = Vt[(8 * Y + g) * W + 4 * kk + t];
  double *pout = A + ((int64_t)p * BW + 2 * t) * ld;
  double *qout = A + ((int64_t)q * BW + 2 * t) * ld;
  for (int c = 0; c < nchunk; c++) {
    const int s = c % STAGES;
    mbar_wait(&full[s], (uint32_t)((c / STAGES) & 1));
    const int64_t r0 = s0 + (int64_t)c * RCH;
    const double *buf = ring + (size_t)s * W * LD;
    // this warp's rows of the chunk start at row0; the row blocks below are
    // immediate offsets from per-chunk column pointers
    const int64_t row0 = r0 + cw * (8 * RB) + g;
    double *cp = pout + row0, *cq = qout + row0;
    const int64_t left = s1 - row0;  // rows of this warp's part still in the slab
#pragma unroll
    for (int rb = 0; rb < RB; rb++) {
      const int rl = cw * (8 * RB) + rb * 8;
      double a[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) a[kk] = buf[(4 * kk + t) * LD + rl + g];
      double acc[NT][2];
#pragma unroll
      for (int Y = 0; Y < NT; Y++) acc[Y][0] = acc[Y][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < NK; kk++)
#pragma unroll
        for (int Y = 0; Y < NT; Y++) dmma(acc[Y][0], acc[Y][1], a[kk], bf[kk][Y]);
      if (rb * 8 < left) {
#pragma unroll
        for (int Y = 0; Y < NT; Y++)
#pragma unroll
          for (int j = 0; j < 2; j++) {
            double *dst = Y < NT / 2 ? cp + (int64_t)(8 * Y + j) * ld
                                     : cq + (int64_t)(8 * Y + j - BW) * ld;
            st_f64(dst + rb * 8, acc[Y][j]);
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// ring of the stand-alone update K3 (engine 0): chunk rows x stages
#ifndef JH_E0RCH
#define JH_E0RCH 128
#endif
#ifndef JH_E0STG
#define JH_E0STG 3
#endif
constexpr int kE0Rch = JH_E0RCH, kE0Stages = JH_E0STG;

template <int W>
__global__ void __launch_bounds__(32 * (kUpdCons + 1))
k_update_tma(double *__restrict__ G, int64_t ldg, int64_t m, double *__restrict__ V,
             int64_t ldv, int64_t nv, const int32_t *__restrict__ pairs,
             const double *__restrict__ Vbuf, const int64_t *__restrict__ trot, int nslab_g) {
  extern __shared__ __align__(128) double ring[];  // [kE0Stages][W][kE0Rch + 4]
  __shared__ __align__(8) uint64_t full[kE0Stages], empty[kE0Stages];
  update_tma_cta<W, kE0Stages, kE0Rch>(G, ldg, m, V, ldv, nv, pairs, Vbuf, trot, nslab_g,
                                       kUpdSlab, blockIdx.x, blockIdx.y, ring, full, empty);
}

}  // namespace jh
