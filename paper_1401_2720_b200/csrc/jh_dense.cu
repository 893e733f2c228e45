// Back substitution of the solve-for-V path (driver.py:203-211): every
// entry's fma chain in the reference's order (k descending from i + 1), then
// the division.  The dense contractions are in jh_outer.cu.
#include "jh_common.cuh"

namespace jh {

// R V = W by back substitution, one column per thread (driver.py:203-211).
__global__ void k_back_substitute(const double *__restrict__ R, int n, const double *__restrict__ W,
                                  int nc, double *__restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nc) return;
  const double *w = W + (int64_t)j * n;
  double *o = out + (int64_t)j * n;
  for (int i = n - 1; i >= 0; i--) {
    double acc = w[i];
    for (int k = i + 1; k < n; k++) acc = fma(-R[(int64_t)k * n + i], o[k], acc);
    o[i] = acc / R[(int64_t)i * n + i];
  }
}

}  // namespace jh

using namespace jh;

extern "C" {

// solve_for_v back substitution (driver.py:203-211), R n x n upper, W n x nc.
int jh_back_substitute(const double *R, int n, const double *W, int nc, double *out,
                       void *stream) {
  g_launches++;
  k_back_substitute<<<(unsigned)cdiv(nc, 128), 128, 0, (cudaStream_t)stream>>>(R, n, W, nc, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // extern "C"
