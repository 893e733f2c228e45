// FP64 tensor-core (DMMA) building blocks for the block-pair contractions.
//
// sm_100a has no FP64 tcgen05 (UMMA) kind; FP64 tensor work is the warp-level
// mma.sync m8n8k4 f64 (SASS DMMA).  Probed on B200 (profiles/r01/dmma_probe.json):
// a DMMA accumulates its 4 k terms as an in-order chain of fused multiply-adds,
// d = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0, c)))), bit for bit.  A chain
// of DMMAs over k-steps in ascending order is therefore exactly the reference's
// per-entry fma chain (_gram_kernel, _postmultiply_kernel), and the contractions
// below stay bitwise equal to the reference.
//
// Fragment layout (m8n8k4, row.col): g = lane >> 2, t = lane & 3
//   A (8 x 4, M x K): lane holds A[g][t]
//   B (4 x 8, K x N): lane holds B[t][g]
//   C/D (8 x 8)     : lane holds D[g][2t], D[g][2t + 1]
#pragma once

#include <cuda.h>

#include "jh_common.cuh"

namespace jh {

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double ldg_f64(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ double ld_f64(const double *p) {
  double v;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

#ifndef JH_STG_MODE
#define JH_STG_MODE 0
#endif
__device__ __forceinline__ void st_f64(double *p, double v) {
#if JH_STG_MODE == 1
  __stcs(p, v);  // streaming store, schedulable like any store
#elif JH_STG_MODE == 2
  *p = v;
#else
  asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v));
#endif
}

// ---- mbarrier + bulk async copy (TMA engine, SASS UBLKCP) -----------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA tensor tile load: the box at (row, col) of the 2-D tensor map into
// shared memory (128 B aligned), completion on `bar` as transaction bytes
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int row, int col,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(row), "r"(col), "r"(smem_u32(bar))
      : "memory");
}

// global -> shared bulk copy of `bytes` (multiple of 16, both 16 B aligned),
// completion signalled on `bar` as transaction bytes.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

}  // namespace jh
