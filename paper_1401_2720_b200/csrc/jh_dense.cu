// Exact-order dense FP64 kernels of arbitrary shape, used by the kernel-level
// API (gram / postmultiply / solve_for_v of blockkernel.py and driver.py) and
// by the outer (multi-GPU) level, where the shortened factor is 2n/g wide.
//
// "Exact order" = every output entry is one chain of fused multiply-adds in
// the reference's order (rows ascending for the Gram matrix,
// blockkernel.py:76-96; k ascending from +0.0 for products,
// blockkernel.py:407-417), so results are bitwise the reference's.  No
// split-K, no reassociation.
#include "jh_common.cuh"

namespace jh {

constexpr int kSyrkT = 32;  // output tile edge
constexpr int kSyrkK = 32;  // rows per staged chunk

// H = A^T A for A (m x c, ld lda); lower-triangle tiles, mirrored.
__global__ void __launch_bounds__(256)
k_syrk_exact(const double *__restrict__ A, int64_t lda, int64_t m, int c, double *__restrict__ H) {
  // map blockIdx.x to a lower-triangle tile (X >= Y)
  int t = blockIdx.x, Y = 0;
  const int nt = (int)cdiv(c, kSyrkT);
  while (t >= nt - Y) {
    t -= nt - Y;
    Y++;
  }
  const int X = Y + t;
  __shared__ double As[kSyrkK][kSyrkT + 1];
  __shared__ double Bs[kSyrkK][kSyrkT + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty 0..7
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int x = X * kSyrkT + tx;
  for (int64_t r0 = 0; r0 < m; r0 += kSyrkK) {
    const int nr = (int)min64(kSyrkK, m - r0);
    for (int idx = threadIdx.x; idx < kSyrkK * kSyrkT; idx += 256) {
      const int i = idx & 31, j = idx >> 5;
      const int cx = X * kSyrkT + j, cy = Y * kSyrkT + j;
      As[i][j] = (i < nr && cx < c) ? A[(int64_t)cx * lda + r0 + i] : 0.0;
      Bs[i][j] = (i < nr && cy < c) ? A[(int64_t)cy * lda + r0 + i] : 0.0;
    }
    __syncthreads();
    for (int i = 0; i < nr; i++) {
      const double a = As[i][tx];
#pragma unroll
      for (int k = 0; k < 4; k++) acc[k] = fma(a, Bs[i][ty + 8 * k], acc[k]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int y = Y * kSyrkT + ty + 8 * k;
    if (x < c && y < c && x >= y) {
      H[(int64_t)y * c + x] = acc[k];
      H[(int64_t)x * c + y] = acc[k];
    }
  }
}

// C = A B (A: m x k, B: k x n2, C: m x n2; column-major, no aliasing);
// entry chains over k ascending from +0.0.
__global__ void __launch_bounds__(256)
k_gemm_exact(const double *__restrict__ A, int64_t lda, int64_t m, int kdim,
             const double *__restrict__ B, int64_t ldb, int n2, double *__restrict__ C,
             int64_t ldc) {
  __shared__ double As[32][65];  // [k][row]
  __shared__ double Bs[32][33];  // [k][col]
  const int64_t row0 = (int64_t)blockIdx.x * 64;
  const int col0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // ty 0..3
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; k++) acc[k] = 0.0;
  for (int k0 = 0; k0 < kdim; k0 += 32) {
    const int nk = min(32, kdim - k0);
    for (int idx = threadIdx.x; idx < 32 * 64; idx += 256) {
      const int i = idx & 63, kk = idx >> 6;
      As[kk][i] = (kk < nk && row0 + i < m) ? A[(int64_t)(k0 + kk) * lda + row0 + i] : 0.0;
    }
    for (int idx = threadIdx.x; idx < 32 * 32; idx += 256) {
      const int kk = idx & 31, j = idx >> 5;
      Bs[kk][j] = (kk < nk && col0 + j < n2) ? B[(int64_t)(col0 + j) * ldb + k0 + kk] : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < nk; kk++) {
      const double a = As[kk][tx];
#pragma unroll
      for (int k = 0; k < 8; k++) acc[k] = fma(a, Bs[kk][ty + 4 * k], acc[k]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const int j = col0 + ty + 4 * k;
    if (row0 + tx < m && j < n2) C[(int64_t)j * ldc + row0 + tx] = acc[k];
  }
}

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

// gram (blockkernel.py:99-107): H (c x c) = A^T A, A m x c (ld lda).
int jh_gram(const double *A, int64_t lda, int64_t m, int c, double *H, void *stream) {
  const int nt = (int)cdiv(c, kSyrkT);
  g_launches++;
  k_syrk_exact<<<nt * (nt + 1) / 2, 256, 0, (cudaStream_t)stream>>>(A, lda, m, c, H);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// postmultiply (blockkernel.py:420-428): C = A B, A m x k, B k x n2.
int jh_gemm(const double *A, int64_t lda, int64_t m, int k, const double *B, int64_t ldb, int n2,
            double *C, int64_t ldc, void *stream) {
  dim3 grid((unsigned)cdiv(m, 64), (unsigned)cdiv(n2, 32));
  g_launches++;
  k_gemm_exact<<<grid, 256, 0, (cudaStream_t)stream>>>(A, lda, m, k, B, ldb, n2, C, ldc);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// solve_for_v back substitution (driver.py:203-211), R n x n upper, W n x nc.
int jh_back_substitute(const double *R, int n, const double *W, int nc, double *out,
                       void *stream) {
  g_launches++;
  k_back_substitute<<<(unsigned)cdiv(nc, 128), 128, 0, (cudaStream_t)stream>>>(R, n, W, nc, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // extern "C"
