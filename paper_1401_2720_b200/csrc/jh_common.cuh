// Shared device helpers for the jhsvd_b200 kernels (sm_100a, FP64).
//
// Exactness contract: every kernel reproduces the reference's IEEE operation
// sequence.  The library is compiled with -fmad=false so that nvcc never
// contracts a*b+c; the only fused operations are the explicit fma() calls
// that mirror the reference's _fp.fma (llvm.fma.f64, pkg/src/jhsvd/_fp.py:24-39).
// Division and square root are the IEEE round-to-nearest CUDA defaults.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace jh {

// rotation.py:42-45: _CT2_HUGE = 2**27, _CT2_TINY = sqrt(2**-53)
constexpr double kCt2Huge = 134217728.0;
constexpr double kCt2Tiny = 0x1.6a09e667f3bcdp-27;

// robustnorm.py:34-45 (NU is ldexp(2 - 2**-52, 1022), half the largest double)
constexpr double kMu = 0x1p-1022;
constexpr double kNu = 0x1.fffffffffffffp+1022;
constexpr int kLeaf = 256;

// error statuses reported through the sweep error key
enum Status : int {
  kOk = 0,
  kCholesky = 1,     // nonpositive Cholesky pivot (RankDeficiencyError)
  kZeroColumn = 2,   // zero column norm in the inner kernel (RankDeficiencyError)
  kHypDomain = 3,    // |coth 2phi| < 1 (JDefinitenessError)
};

// 64-bit error key: smaller = earlier in the reference's sequential order.
//   bits 38..63 p-step, 16..37 task, 13..15 status, 0..12 1-based index
__host__ __device__ inline unsigned long long err_key(int pstep, int task, int status,
                                                      int index) {
  return ((unsigned long long)pstep << 38) | ((unsigned long long)task << 16) |
         ((unsigned long long)status << 13) | (unsigned long long)(index & 0x1fff);
}

// Guarded rotation parameters, rotation.py:71-102 (_rotation_core with the
// cs2 formula of _params_from_ct2).  t = +1 trigonometric, -1 hyperbolic.
// Returns false for a hyperbolic pair with |ct2| < 1.
__device__ __forceinline__ bool rotation_core(double hpp, double hqq, double hpq, double t,
                                              double &cs, double &tn) {
  const double h = hqq - t * hpp;
  double ct2 = t * (h / (2.0 * hpq));
  if (t < 0.0) {
    if (fabs(ct2) == 1.0) {
      ct2 = ct2 > 0.0 ? 1.25 : -1.25;
    } else if (fabs(ct2) < 1.0) {
      cs = 0.0;
      tn = 0.0;
      return false;
    }
  }
  const double a = fabs(ct2);
  const double sgn = ct2 >= 0.0 ? 1.0 : -1.0;
  if (a >= kCt2Huge) {
    tn = sgn / (2.0 * a);
    cs = 1.0;
    return true;
  }
  double ct;
  if (t > 0.0 && a < kCt2Tiny)
    ct = a + 1.0;
  else
    ct = a + sqrt(fma(ct2, ct2, t));
  tn = sgn / ct;
  // (the reference also forms cs1 = 1/sqrt(fma(t*tn, tn, 1)); it is unused)
  cs = ct / sqrt(fma(ct, ct, t));
  return true;
}

// Branch-light form of rotation_core with identical results: every special
// case (hyperbolic 5/4 substitution and domain check, the sqrt(eps) and
// sqrt(2/eps) guards) becomes a select, so the two square roots and three
// divisions issue without divergence and the critical path is
// div -> sqrt -> sqrt -> div.  Values computed on a discarded branch (NaN /
// inf from sqrt of a negative or an overflowing square) never reach a result.
__device__ __forceinline__ bool rotation_core_sel(double hpp, double hqq, double hpq, double t,
                                                  double &cs, double &tn) {
  const double h = hqq - t * hpp;
  double ct2 = t * (h / (2.0 * hpq));
  bool ok = true;
  if (t < 0.0) {
    const double aa = fabs(ct2);
    ok = !(aa < 1.0);
    ct2 = (aa == 1.0) ? (ct2 > 0.0 ? 1.25 : -1.25) : ct2;
  }
  const double a = fabs(ct2);
  const double sgn = ct2 >= 0.0 ? 1.0 : -1.0;
  const double r = sqrt(fma(ct2, ct2, t));
  const bool huge = a >= kCt2Huge;
  double ct = (t > 0.0 && a < kCt2Tiny) ? a + 1.0 : a + r;
  ct = huge ? 2.0 * a : ct;
  tn = sgn / ct;
  const double c2 = ct / sqrt(fma(ct, ct, t));
  cs = huge ? 1.0 : c2;
  if (!ok) {
    cs = 0.0;
    tn = 0.0;
  }
  return ok;
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// total kernel launches issued by this library (defined in jh_runtime.cu)
extern unsigned long long g_launches;

}  // namespace jh
