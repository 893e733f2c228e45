// Scalar pieces of the robust sum of squares (DRDSSQ, reference
// pkg/src/jhsvd/robustnorm.py:116-162) shared by the column-norm kernels
// (jh_norms.cu) and the QR peel-off shortening (jh_qr.cu).
#pragma once

#include "jh_common.cuh"

namespace jh {

// -- host/device scalar helpers (robustnorm.py:116-162) ----------------------

__host__ __device__ inline int scale_exponent(double f, double t, bool up) {
  int fe, te;
  const double fy = frexp(f, &fe), ty = frexp(t, &te);
  if (up) return (te - fe) + (fy < ty ? 1 : 0);
  return (te - fe) - (fy > ty ? 1 : 0);
}

__host__ __device__ inline void common_form(int64_t j, double v, int64_t &jo, double &vo) {
  if (v == 0.0) {
    jo = 0;
    vo = 0.0;
    return;
  }
  int fe;
  const double fy = frexp(v, &fe);
  const double y = 2.0 * fy;
  const int64_t m = fe - 1;
  const int64_t mp = (m & 1) ? -1 : 0;
  jo = j + m - mp;
  vo = ldexp(y, (int)mp);
}

__host__ __device__ inline void add_scaled(int64_t ja, double va, int64_t jb, double vb,
                                           int64_t &jo, double &vo) {
  if (va == 0.0) {
    jo = jb;
    vo = vb;
    return;
  }
  if (vb == 0.0) {
    jo = ja;
    vo = va;
    return;
  }
  int64_t js, jbig;
  double vs, vbig;
  if (ja < jb || (ja == jb && va <= vb)) {
    js = ja; vs = va; jbig = jb; vbig = vb;
  } else {
    js = jb; vs = vb; jbig = ja; vbig = va;
  }
  const double shifted = ldexp(vs, (int)(js - jbig));
  jo = jbig;
  vo = shifted + vbig;
}

}  // namespace jh
