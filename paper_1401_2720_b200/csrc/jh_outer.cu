// Dense FP64 contractions of any shape on the DMMA tensor pipe, in the
// reference's per-entry operation order: the kernel-level API (gram /
// postmultiply / cholesky_in_place of blockkernel.py) and the outer
// (multi-GPU) level of distsim.py, where one worker's shortened factor is
// 2n/g wide (DSYRK, DPOTRF, 2 x DGEMM).
//
//   jh_gram   H = A^T A                 every entry one fma chain over the
//                                       rows, ascending (blockkernel.py:76-96)
//   jh_gemm   C = A B                   one chain over k ascending from +0.0
//                                       (blockkernel.py:407-417)
//   jh_cholesky H = L L^T, R = L^T      blocked right-looking Cholesky whose
//                                       every entry sees the reference's
//                                       sequence (blockkernel.py:110-127)
//
// A DMMA (mma.sync m8n8k4 f64) adds its four k terms as an in-order chain of
// fused multiply-adds (jh_dmma.cuh, profiles/r01/dmma_probe.json), so a
// chain of DMMAs over ascending k-steps is the reference's chain; nothing is
// split over k.  One CTA = 4 warps computes a 64 x 64 output tile, each warp
// a 32 x 32 quadrant (16 independent 8 x 8 accumulators); operands stream
// through a 3-stage cp.async ring of 32-deep k slices with padded strides
// (= 4 mod 16 doubles: conflict-free fragment loads in either orientation).
//
// Cholesky (jh_cholesky): for each 64-wide panel K0 --
//   k_chol_diag   the 64 x 64 diagonal block, right-looking in shared memory
//                 (the reference loop restricted to the block);
//   k_chol_trsm   every row below: L[x][j] = (h[x][j] - sum_k L[x][k] L[j][k])
//                 / L[j][j], the sum an ascending fma chain (one thread per row);
//   trailing      C -= L_p L_p^T on the lower tiles of the trailing matrix,
//                 a DMMA chain over the panel's k in ascending order added to
//                 the entry's running value.
// Per entry that is exactly the reference's order: updates k = 0, 1, ... in
// ascending order, then the division by the pivot.
#include "jh_common.cuh"
#include "jh_dmma.cuh"
#include "jh_kernels.h"

namespace jh {

namespace {

constexpr int kT = 64;        // output tile edge
constexpr int kKc = 32;       // k slice per stage
constexpr int kStg = 3;       // ring stages
constexpr int kOpElems = 64 * (kKc + 4) > kKc * (64 + 4) ? 64 * (kKc + 4) : kKc * (64 + 4);
constexpr int kOuterThreads = 128;
constexpr int kNb = 64;       // Cholesky panel width

// 8-byte async copy; invalid elements are zero-filled (src-size 0, the
// source address -- a valid one -- is not read)
__device__ __forceinline__ void cp_async8(double *dst, const double *src, const double *safe,
                                          bool valid) {
  const uint32_t d = smem_u32(dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(valid ? src : safe),
               "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One operand of a tile: element (i, k) (i = tile row/column index, k =
// contraction index) lives at g[i * gi + k * gk] in global memory; exactly
// one of gi, gk is 1.  In shared memory the contiguous direction is kept
// contiguous: KMAJ (gk != 1, i contiguous) -> s[k * (64 + 4) + i], else
// s[i * (kKc + 4) + k].
struct Operand {
  const double *g;
  int64_t gi, gk;
  int64_t ilim, klim;  // valid i < ilim, k < klim (relative to the tile origin)
  bool kmaj;
};

__device__ __forceinline__ void load_slice(double *s, const Operand &o, int64_t k0) {
  if (o.kmaj) {
    for (int e = threadIdx.x; e < kKc * 64; e += kOuterThreads) {
      const int i = e & 63, k = e >> 6;
      const bool ok = i < o.ilim && k0 + k < o.klim;
      cp_async8(s + k * (64 + 4) + i, o.g + (int64_t)i * o.gi + (k0 + k) * o.gk, o.g, ok);
    }
  } else {
    for (int e = threadIdx.x; e < kKc * 64; e += kOuterThreads) {
      const int k = e & (kKc - 1), i = e / kKc;
      const bool ok = i < o.ilim && k0 + k < o.klim;
      cp_async8(s + i * (kKc + 4) + k, o.g + (int64_t)i * o.gi + (k0 + k) * o.gk, o.g, ok);
    }
  }
}

__device__ __forceinline__ double frag(const double *s, bool kmaj, int i, int k) {
  return kmaj ? s[k * (64 + 4) + i] : s[i * (kKc + 4) + k];
}

// acc[a][b] (+)= sum_k A(i0 + 8a + g, k) B(j0 + 8b + g, k) over k in
// [0, K), one DMMA chain per 8 x 8 tile in ascending k.  NEG negates A.
template <bool NEG>
__device__ __forceinline__ void tile_chain(double (&acc)[4][4][2], const Operand &A,
                                           const Operand &B, int64_t K, double *smem) {
  double *sa = smem, *sb = smem + kStg * kOpElems;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int i0 = 32 * (warp & 1), j0 = 32 * (warp >> 1);
  const int64_t nslice = cdiv(K, kKc);
#pragma unroll
  for (int s = 0; s < kStg - 1; s++) {
    if (s < nslice) {
      load_slice(sa + s * kOpElems, A, (int64_t)s * kKc);
      load_slice(sb + s * kOpElems, B, (int64_t)s * kKc);
    }
    cp_commit();
  }
  for (int64_t sl = 0; sl < nslice; sl++) {
    cp_wait<kStg - 2>();
    __syncthreads();
    {  // refill the stage consumed one iteration ago
      const int64_t nx = sl + kStg - 1;
      if (nx < nslice) {
        load_slice(sa + (nx % kStg) * kOpElems, A, nx * kKc);
        load_slice(sb + (nx % kStg) * kOpElems, B, nx * kKc);
      }
      cp_commit();
    }
    const double *ca = sa + (sl % kStg) * kOpElems, *cb = sb + (sl % kStg) * kOpElems;
#pragma unroll 2
    for (int kk = 0; kk < kKc; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int a = 0; a < 4; a++) {
        const double v = frag(ca, A.kmaj, i0 + 8 * a + g, kk + t);
        fa[a] = NEG ? -v : v;
      }
#pragma unroll
      for (int b = 0; b < 4; b++) fb[b] = frag(cb, B.kmaj, j0 + 8 * b + g, kk + t);
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
  }
  cp_wait<0>();
  __syncthreads();
}

// lower tile (X, Y), X >= Y, of an nt x nt tile grid from a linear index
__device__ __forceinline__ void lower_tile(int64_t t, int nt, int &X, int &Y) {
  int y = 0;
  while (t >= nt - y) {
    t -= nt - y;
    y++;
  }
  X = y + (int)t;
  Y = y;
}

// H (c x c) = A^T A, A m x c (ld lda): lower tiles, each written to both
// triangles (an fma's product is commutative, so the mirrored entry of a
// diagonal tile is the same chain bit for bit)
__global__ void __launch_bounds__(kOuterThreads, 2)
k_syrk_dmma(const double *__restrict__ A, int64_t lda, int64_t m, int c, double *__restrict__ H) {
  extern __shared__ __align__(16) double smem[];
  const int nt = (int)cdiv(c, kT);
  int X, Y;
  lower_tile(blockIdx.x, nt, X, Y);
  const int64_t x0 = (int64_t)X * kT, y0 = (int64_t)Y * kT;
  // operand (i = column of A, k = row of A): g[i * lda + k]
  Operand oa{A + x0 * lda, lda, 1, c - x0, m, false};
  Operand ob{A + y0 * lda, lda, 1, c - y0, m, false};
  double acc[4][4][2] = {};
  tile_chain<false>(acc, oa, ob, m, smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t x = x0 + 32 * (warp & 1) + 8 * a + g;
        const int64_t y = y0 + 32 * (warp >> 1) + 8 * b + 2 * t + h;
        if (x < c && y < c) {
          H[y * c + x] = acc[a][b][h];
          H[x * c + y] = acc[a][b][h];
        }
      }
}

// C (m x n2, ld ldc) = A (m x kd, ld lda) B (kd x n2, ld ldb)
__global__ void __launch_bounds__(kOuterThreads, 2)
k_gemm_dmma(const double *__restrict__ A, int64_t lda, int64_t m, int kd,
            const double *__restrict__ B, int64_t ldb, int n2, double *__restrict__ C,
            int64_t ldc) {
  extern __shared__ __align__(16) double smem[];
  const int64_t x0 = (int64_t)blockIdx.x * kT, y0 = (int64_t)blockIdx.y * kT;
  // A operand (i = row, k): A[k * lda + i] (rows contiguous: k-major slices)
  Operand oa{A + x0, 1, lda, m - x0, kd, true};
  // B operand (i = column j, k): B[j * ldb + k]
  Operand ob{B + y0 * ldb, ldb, 1, n2 - y0, kd, false};
  double acc[4][4][2] = {};
  tile_chain<false>(acc, oa, ob, kd, smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t x = x0 + 32 * (warp & 1) + 8 * a + g;
        const int64_t y = y0 + 32 * (warp >> 1) + 8 * b + 2 * t + h;
        if (x < m && y < n2) C[y * ldc + x] = acc[a][b][h];
      }
}

// ---- blocked Cholesky -------------------------------------------------------

// diagonal block [K0, K0 + kb) of H (c x c, column-major, lower triangle),
// the reference's right-looking loop in shared memory
__global__ void __launch_bounds__(256)
k_chol_diag(double *__restrict__ H, int c, int K0, int kb, int *info) {
  __shared__ double S[kNb][kNb + 1];  // S[col][row]
  __shared__ int s_bad;
  if (*info) return;
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int j = e / kb, x = e - j * kb;
    if (x >= j) S[j][x] = H[(int64_t)(K0 + j) * c + K0 + x];
  }
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int k = 0; k < kb; k++) {
    if (threadIdx.x == 0) {
      const double d = S[k][k];
      if (!(d > 0.0) || !isfinite(d))
        s_bad = K0 + k + 1;
      else
        S[k][k] = sqrt(d);
    }
    __syncthreads();
    if (s_bad) break;
    const double l = S[k][k];
    for (int x = k + 1 + threadIdx.x; x < kb; x += blockDim.x) S[k][x] = S[k][x] / l;
    __syncthreads();
    // h[x][j] = fma(-h[x][k], h[j][k], h[x][j]) for k < j <= x
    const int nrem = kb - k - 1;
    for (int e = threadIdx.x; e < nrem * nrem; e += blockDim.x) {
      const int j = k + 1 + e / nrem, x = k + 1 + e % nrem;
      if (x >= j) S[j][x] = fma(-S[k][x], S[k][j], S[j][x]);
    }
    __syncthreads();
  }
  if (s_bad) {
    if (threadIdx.x == 0) *info = s_bad;
    return;
  }
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int j = e / kb, x = e - j * kb;
    if (x >= j) H[(int64_t)(K0 + j) * c + K0 + x] = S[j][x];
  }
}

// rows x >= K0 + 64 of the panel: L[x][K0 + j], one thread per row
__global__ void __launch_bounds__(128)
k_chol_trsm(double *__restrict__ H, int c, int K0, const int *info) {
  __shared__ double Ld[kNb][kNb + 1];  // Ld[k][j] = L[K0 + j][K0 + k]
  if (*info) return;
  for (int e = threadIdx.x; e < kNb * kNb; e += blockDim.x) {
    const int k = e / kNb, j = e - k * kNb;
    Ld[k][j] = (j >= k) ? H[(int64_t)(K0 + k) * c + K0 + j] : 0.0;
  }
  __syncthreads();
  const int64_t x = (int64_t)K0 + kNb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= c) return;
  double row[kNb];
#pragma unroll
  for (int j = 0; j < kNb; j++) row[j] = H[(int64_t)(K0 + j) * c + x];
#pragma unroll
  for (int j = 0; j < kNb; j++) {
    double acc = row[j];
#pragma unroll
    for (int k = 0; k < j; k++) acc = fma(-row[k], Ld[k][j], acc);
    row[j] = acc / Ld[j][j];
  }
#pragma unroll
  for (int j = 0; j < kNb; j++) H[(int64_t)(K0 + j) * c + x] = row[j];
}

// trailing update of the lower tiles of [T0, c): C[x][y] -= sum over the
// panel's k (ascending) of L[x][k] L[y][k], added to the running entry
__global__ void __launch_bounds__(kOuterThreads, 2)
k_chol_update(double *__restrict__ H, int c, int K0, int T0, const int *info) {
  extern __shared__ __align__(16) double smem[];
  if (*info) return;
  const int nt = (int)cdiv(c - T0, kT);
  int X, Y;
  lower_tile(blockIdx.x, nt, X, Y);
  const int64_t x0 = T0 + (int64_t)X * kT, y0 = T0 + (int64_t)Y * kT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t x = x0 + 32 * (warp & 1) + 8 * a + g;
        const int64_t y = y0 + 32 * (warp >> 1) + 8 * b + 2 * t + h;
        acc[a][b][h] = (x < c && y < c && x >= y) ? H[y * c + x] : 0.0;
      }
  // operand (i = row x, k = panel column): H[(K0 + k) * c + x]
  Operand oa{H + (int64_t)K0 * c + x0, 1, c, c - x0, kNb, true};
  Operand ob{H + (int64_t)K0 * c + y0, 1, c, c - y0, kNb, true};
  tile_chain<true>(acc, oa, ob, kNb, smem);
#pragma unroll
  for (int a = 0; a < 4; a++)
#pragma unroll
    for (int b = 0; b < 4; b++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t x = x0 + 32 * (warp & 1) + 8 * a + g;
        const int64_t y = y0 + 32 * (warp >> 1) + 8 * b + 2 * t + h;
        if (x < c && y < c && x >= y) H[y * c + x] = acc[a][b][h];
      }
}

// R = L^T (upper triangle), zero strict lower
__global__ void k_chol_to_r(const double *__restrict__ H, int c, double *__restrict__ R,
                            const int *info) {
  if (*info) return;
  const int64_t total = (int64_t)c * c;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / c, i = e - j * c;  // R[i][j] at e = j * c + i
    R[e] = (i <= j) ? H[i * c + j] : 0.0;
  }
}

constexpr size_t kTileSmem = sizeof(double) * 2 * kStg * kOpElems;

}  // namespace

}  // namespace jh

using namespace jh;

static int finish_outer() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" {

// gram (blockkernel.py:99-107): H (c x c) = A^T A, A m x c (ld lda).
int jh_gram(const double *A, int64_t lda, int64_t m, int c, double *H, void *stream) {
  if (c < 1 || m < 0 || lda < m) return -1000;
  const int64_t nt = cdiv(c, kT);
  ensure_smem((const void *)k_syrk_dmma, (int)kTileSmem);
  g_launches++;
  k_syrk_dmma<<<(unsigned)(nt * (nt + 1) / 2), kOuterThreads, kTileSmem, (cudaStream_t)stream>>>(
      A, lda, m, c, H);
  return finish_outer();
}

// postmultiply (blockkernel.py:420-428): C = A B, A m x k, B k x n2.
int jh_gemm(const double *A, int64_t lda, int64_t m, int k, const double *B, int64_t ldb, int n2,
            double *C, int64_t ldc, void *stream) {
  if (m < 0 || k < 0 || n2 < 0 || lda < m || ldb < k || ldc < m) return -1000;
  if (m == 0 || n2 == 0) return 0;
  ensure_smem((const void *)k_gemm_dmma, (int)kTileSmem);
  dim3 grid((unsigned)cdiv(m, kT), (unsigned)cdiv(n2, kT));
  g_launches++;
  k_gemm_dmma<<<grid, kOuterThreads, kTileSmem, (cudaStream_t)stream>>>(A, lda, m, k, B, ldb, n2,
                                                                        C, ldc);
  return finish_outer();
}

// cholesky_in_place (blockkernel.py:130-145) of any order c: H (c x c,
// device, lower triangle read, overwritten by L), R = L^T with a zero strict
// lower triangle; *info (device int, must be 0 on entry) = 0 or the 1-based
// first nonpositive pivot (then R is not written).
int jh_cholesky(double *H, int c, double *R, int *info, void *stream) {
  if (c < 1) return -1000;
  cudaStream_t st = (cudaStream_t)stream;
  ensure_smem((const void *)k_chol_update, (int)kTileSmem);
  for (int K0 = 0; K0 < c; K0 += kNb) {
    const int kb = c - K0 < kNb ? c - K0 : kNb;
    k_chol_diag<<<1, 256, 0, st>>>(H, c, K0, kb, info);
    g_launches++;
    const int T0 = K0 + kb;
    if (T0 < c) {
      k_chol_trsm<<<(unsigned)cdiv(c - T0, 128), 128, 0, st>>>(H, c, K0, info);
      const int64_t nt = cdiv(c - T0, kT);
      k_chol_update<<<(unsigned)(nt * (nt + 1) / 2), kOuterThreads, kTileSmem, st>>>(H, c, K0, T0,
                                                                                    info);
      g_launches += 2;
    }
  }
  const int64_t total = (int64_t)c * c;
  k_chol_to_r<<<(unsigned)min64(cdiv(total, 256), 148 * 32), 256, 0, st>>>(H, c, R, info);
  g_launches++;
  return finish_outer();
}

}  // extern "C"
