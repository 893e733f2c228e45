// QR peel-off shortening (reference qr_peeloff, pkg/src/jhsvd/blockkernel.py:148-244,
// selected by SolverConfig.shortening == "qr"): the upper-triangular factor R
// of a task's block pair [Gp Gq] (m x w) without forming the Gram matrix,
// for inputs whose column scaling makes the Gram formation unsafe.
//
// The pair is cut into m / w chunks of w rows.  Every chunk is reduced by
// Householder QR (_householder_qr) and merged into the running R by the
// Givens peel-off stages (_peel_combine), in chunk order.  One CTA per task:
// its warps factor consecutive chunks concurrently (lane j owns column j of
// the column updates, so each entry's fma chain runs in the reference's
// order), then warp 0 merges them one by one (lane x owns the row pair
// (x, x - k) of stage k -- the row pairs of a stage are disjoint, and the
// stages are sequential as in the reference).  The sub-column norm of each
// Householder step is the reference's robust norm (norm2_unscaled: one
// 256-element leaf, with the scaled three-partition fallback).  Results
// are bitwise the reference's.
#include "jh_kernels.h"
#include "jh_robust.cuh"
#include "jhsvd_b200.h"

#include <cmath>

namespace jh {

constexpr int kQrThreads = 128;
constexpr int kQrWarps = kQrThreads / 32;
constexpr int kQrMaxW = 32;

// safe bounds (robustnorm.safe_bounds) for vector lengths 0..kQrMaxW, a
// kernel parameter (no per-device state)
struct QrBounds {
  double mu[kQrMaxW + 1], nu[kQrMaxW + 1];
};

static const QrBounds &qr_bounds() {
  static const QrBounds b = [] {
    QrBounds t{};
    for (int n = 1; n <= kQrMaxW; n++) jh_safe_bounds(n, &t.mu[n], &t.nu[n]);
    return t;
  }();
  return b;
}

// sum of squares of one leaf restricted to lo <= |x| <= hi, scaled by 2**j
// (_tree_sumsq_selected with a single leaf)
__device__ __forceinline__ double qr_selected(const double *x, int n, double lo, double hi, int j) {
  double acc = 0.0;
  for (int i = 0; i < n; i++) {
    const double a = fabs(x[i]);
    if (a > 0.0 && lo <= a && a <= hi) {
      const double v = ldexp(x[i], j);
      acc = fma(v, v, acc);
    }
  }
  return acc;
}

// norm2_unscaled (robustnorm.py:303-308) of a vector of n <= 256 entries
// (one leaf), by one thread: _sum_squares_core (robustnorm.py:242-292) then
// norm2 (:295-300)
template <class Bounds>
__device__ double qr_norm2(const double *x, int n, const Bounds &bd) {
  if (n == 0) return 0.0;
  double big = 0.0, small = kNu;
  for (int i = 0; i < n; i++) {
    const double a = fabs(x[i]);
    if (a > big) big = a;
    if (0.0 < a && a < small) small = a;
  }
  if (big == 0.0) return 0.0;
  int64_t jr;
  double vr;
  double plain = 0.0;
  for (int i = 0; i < n; i++) plain = fma(x[i], x[i], plain);
  if (isfinite(plain) && small * small >= kMu) {
    common_form(0, plain, jr, vr);
  } else {
    const double mu_tilde = bd.mu[n], nu_hat = bd.nu[n];
    int64_t js[3] = {0, 0, 0};
    double vs[3] = {0.0, 0.0, 0.0};
    int count = 0;
    if (small <= nu_hat && big >= mu_tilde) {
      const double s1 = qr_selected(x, n, mu_tilde, nu_hat, 0);
      if (s1 != 0.0) {
        common_form(0, s1, js[count], vs[count]);
        count++;
      }
    }
    if (big > nu_hat) {
      const int j2 = scale_exponent(big, nu_hat, false);
      const double s2 = qr_selected(x, n, nextafter(nu_hat, kNu), kNu, j2);
      if (s2 != 0.0) {
        common_form(-2 * (int64_t)j2, s2, js[count], vs[count]);
        count++;
      }
    }
    if (small < mu_tilde) {
      const int j0 = scale_exponent(small, mu_tilde, true);
      const double s0 = qr_selected(x, n, 0.0, nextafter(mu_tilde, 0.0), j0);
      if (s0 != 0.0) {
        common_form(-2 * (int64_t)j0, s0, js[count], vs[count]);
        count++;
      }
    }
    if (count == 0) return 0.0;
    for (int a = 0; a < count - 1; a++)
      for (int b = a + 1; b < count; b++)
        if (js[a] > js[b] || (js[a] == js[b] && vs[a] > vs[b])) {
          const int64_t tj = js[a];
          js[a] = js[b];
          js[b] = tj;
          const double tv = vs[a];
          vs[a] = vs[b];
          vs[b] = tv;
        }
    int64_t ja = js[0];
    double va = vs[0];
    for (int k = 1; k < count; k++) {
      common_form(ja, va, ja, va);
      add_scaled(ja, va, js[k], vs[k], ja, va);
    }
    common_form(ja, va, jr, vr);
  }
  if (vr == 0.0) return 0.0;
  // norm = sqrt(v) / 2**js with js = -(jr // 2) (Python floor division)
  int64_t q = jr / 2;
  if ((jr % 2) && jr < 0) q -= 1;
  return ldexp(sqrt(vr), (int)q);
}

// _hypot2 (blockkernel.py:148-158)
__device__ __forceinline__ double qr_hypot2(double a, double b) {
  const double aa = fabs(a), ab = fabs(b);
  const double big = aa >= ab ? aa : ab;
  if (big == 0.0) return 0.0;
  int e;
  frexp(big, &e);
  const double as = ldexp(aa, -e), bs = ldexp(ab, -e);
  return ldexp(sqrt(fma(as, as, bs * bs)), e);
}

// _givens (blockkernel.py:191-201)
__device__ __forceinline__ void qr_givens(double a, double b, double &cc, double &ss) {
  const double aa = fabs(a), ab = fabs(b);
  const double big = aa >= ab ? aa : ab;
  int e;
  frexp(big, &e);
  const double as = ldexp(a, -e), bs = ldexp(b, -e);
  const double d = sqrt(fma(as, as, bs * bs));
  cc = as / d;
  ss = bs / d;
}

// _householder_qr (blockkernel.py:161-188) of a W x W block (column-major,
// ld W + 1) by one warp; sc: 4 doubles of per-warp scratch
template <int W>
__device__ void qr_householder_warp(double *a, double *sc, int lane, const QrBounds &bd) {
  constexpr int LD = W + 1;
  for (int k = 0; k < W - 1; k++) {
    if (lane == 0) {
      const double alpha = a[k * LD + k];
      const double xnorm = qr_norm2(a + k * LD + k + 1, W - k - 1, bd);
      double skip = 1.0, tau = 0.0, denom = 1.0, beta = 0.0;
      if (xnorm != 0.0) {
        const double nr = qr_hypot2(alpha, xnorm);
        beta = alpha >= 0.0 ? -nr : nr;
        tau = (beta - alpha) / beta;
        denom = alpha - beta;
        skip = 0.0;
      }
      sc[0] = skip;
      sc[1] = tau;
      sc[2] = denom;
      sc[3] = beta;
    }
    __syncwarp();
    if (sc[0] != 0.0) {
      __syncwarp();
      continue;
    }
    const double tau = sc[1], denom = sc[2], beta = sc[3];
    if (lane > k && lane < W) a[k * LD + lane] = a[k * LD + lane] / denom;
    __syncwarp();
    if (lane == 0) a[k * LD + k] = beta;
    const int j = lane;
    if (j > k && j < W) {
      double *cj = a + j * LD;
      const double *ck = a + k * LD;
      double z = cj[k];
      for (int i = k + 1; i < W; i++) z = fma(ck[i], cj[i], z);
      const double tz = tau * z;
      cj[k] = cj[k] - tz;
      for (int i = k + 1; i < W; i++) cj[i] = fma(-tz, ck[i], cj[i]);
    }
    __syncwarp();
  }
  for (int j = lane; j < W; j += 32)
    for (int i = j + 1; i < W; i++) a[j * LD + i] = 0.0;
  __syncwarp();
}

// _peel_combine (blockkernel.py:204-220) of r1 into r0 by one warp
template <int W>
__device__ void qr_peel_warp(double *r0, double *r1, int lane) {
  constexpr int LD = W + 1;
  for (int k = 0; k < W; k++) {
    const int x = lane;
    if (x >= k && x < W) {
      const int xr = x - k;
      const double b = r1[x * LD + xr];
      if (b != 0.0) {
        double cc, ss;
        qr_givens(r0[x * LD + x], b, cc, ss);
        for (int j = x; j < W; j++) {
          const double v0 = r0[j * LD + x];
          const double v1 = r1[j * LD + xr];
          r0[j * LD + x] = fma(ss, v1, cc * v0);
          r1[j * LD + xr] = fma(cc, v1, -(ss * v0));
        }
      }
    }
    __syncwarp();
  }
}

template <int W>
__global__ void __launch_bounds__(kQrThreads)
k_qr_peeloff(const double *__restrict__ G, int64_t ldg, int64_t m,
             const int32_t *__restrict__ pairs, double *__restrict__ Rbuf,
             const __grid_constant__ QrBounds bd) {
  constexpr int LD = W + 1, BW = W / 2;
  __shared__ double r0[W * LD];
  __shared__ double blk[kQrWarps][W * LD];
  __shared__ double sc[kQrWarps][4];
  const int task = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // pairs == nullptr: the single pair (0, 1) of jh_qr_peeloff
  const int64_t p = pairs ? pairs[2 * task] : 0, q = pairs ? pairs[2 * task + 1] : 1;
  const int64_t nchunk = m / W;
  for (int64_t g0 = 0; g0 < nchunk; g0 += kQrWarps) {
    const int64_t c = g0 + warp;
    if (c < nchunk) {
      double *a = blk[warp];
      for (int e = lane; e < W * W; e += 32) {
        const int j = e / W, i = e - j * W;
        const int64_t col = j < BW ? p * BW + j : q * BW + (j - BW);
        a[j * LD + i] = G[col * ldg + c * W + i];
      }
      __syncwarp();
      qr_householder_warp<W>(a, sc[warp], lane, bd);
    }
    __syncthreads();
    if (warp == 0) {
      for (int w2 = 0; w2 < kQrWarps && g0 + w2 < nchunk; w2++) {
        if (g0 + w2 == 0) {
          for (int e = lane; e < W * LD; e += 32) r0[e] = blk[0][e];
          __syncwarp();
        } else {
          qr_peel_warp<W>(r0, blk[w2], lane);
        }
      }
    }
    __syncthreads();
  }
  // nonnegative diagonal (row sign flips go into the discarded Q)
  if (warp == 0 && lane < W && r0[lane * LD + lane] < 0.0)
    for (int j = lane; j < W; j++) r0[j * LD + lane] = -r0[j * LD + lane];
  __syncthreads();
  double *R = Rbuf + (size_t)task * W * W;
  for (int e = threadIdx.x; e < W * W; e += kQrThreads) {
    const int j = e / W, i = e - j * W;
    R[e] = r0[j * LD + i];
  }
}

// ---- any even width up to kQrWideMax: the same algorithm with the blocks in
// global memory (L2-resident scratch, one CTA of kQrWideThreads per task):
// thread j owns column j in the Householder updates, thread x row x of a
// peel-off stage.  Column norms of up to kQrWideMax - 1 entries are one leaf
// of the reference's robust norm (robustnorm.py:242-308): qr_norm2 with a
// bounds table for lengths up to kQrWideMax.
constexpr int kQrWideMax = 256;
constexpr int kQrWideThreads = 256;

struct QrBoundsWide {
  double mu[kQrWideMax + 1], nu[kQrWideMax + 1];
};

static const QrBoundsWide &qr_bounds_wide() {
  static const QrBoundsWide b = [] {
    QrBoundsWide t{};
    for (int n = 1; n <= kQrWideMax; n++) jh_safe_bounds(n, &t.mu[n], &t.nu[n]);
    return t;
  }();
  return b;
}

// _householder_qr of a c x c block (column-major, ld c) by the CTA
__device__ void qr_householder_cta(double *a, int c, const QrBoundsWide &bd, double *sc) {
  const int tid = threadIdx.x;
  for (int k = 0; k < c - 1; k++) {
    if (tid == 0) {
      const double alpha = a[(int64_t)k * c + k];
      const double xnorm = qr_norm2(a + (int64_t)k * c + k + 1, c - k - 1, bd);
      double skip = 1.0, tau = 0.0, denom = 1.0, beta = 0.0;
      if (xnorm != 0.0) {
        const double nr = qr_hypot2(alpha, xnorm);
        beta = alpha >= 0.0 ? -nr : nr;
        tau = (beta - alpha) / beta;
        denom = alpha - beta;
        skip = 0.0;
      }
      sc[0] = skip;
      sc[1] = tau;
      sc[2] = denom;
      sc[3] = beta;
    }
    __syncthreads();
    const bool skip = sc[0] != 0.0;
    const double tau = sc[1], denom = sc[2], beta = sc[3];
    if (!skip) {
      for (int i = k + 1 + tid; i < c; i += blockDim.x)
        a[(int64_t)k * c + i] = a[(int64_t)k * c + i] / denom;
    }
    __syncthreads();
    if (!skip) {
      if (tid == 0) a[(int64_t)k * c + k] = beta;
      const double *ck = a + (int64_t)k * c;
      for (int j = k + 1 + tid; j < c; j += blockDim.x) {
        double *cj = a + (int64_t)j * c;
        double z = cj[k];
        for (int i = k + 1; i < c; i++) z = fma(ck[i], cj[i], z);
        const double tz = tau * z;
        cj[k] = cj[k] - tz;
        for (int i = k + 1; i < c; i++) cj[i] = fma(-tz, ck[i], cj[i]);
      }
    }
    __syncthreads();
  }
  for (int j = tid; j < c; j += blockDim.x)
    for (int i = j + 1; i < c; i++) a[(int64_t)j * c + i] = 0.0;
  __syncthreads();
}

// _peel_combine of r1 into r0 (both c x c, ld c) by the CTA
__device__ void qr_peel_cta(double *r0, double *r1, int c) {
  for (int k = 0; k < c; k++) {
    for (int x = k + threadIdx.x; x < c; x += blockDim.x) {
      const int xr = x - k;
      const double b = r1[(int64_t)x * c + xr];
      if (b != 0.0) {
        double cc, ss;
        qr_givens(r0[(int64_t)x * c + x], b, cc, ss);
        for (int j = x; j < c; j++) {
          const double v0 = r0[(int64_t)j * c + x];
          const double v1 = r1[(int64_t)j * c + xr];
          r0[(int64_t)j * c + x] = fma(ss, v1, cc * v0);
          r1[(int64_t)j * c + xr] = fma(cc, v1, -(ss * v0));
        }
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kQrWideThreads)
k_qr_wide(const double *__restrict__ G, int64_t ldg, int64_t m, int c,
          const int32_t *__restrict__ pairs, double *__restrict__ Rbuf, double *__restrict__ scr,
          const __grid_constant__ QrBoundsWide bd) {
  __shared__ double sc[4];
  const int task = blockIdx.x, bw = c / 2;
  const int64_t p = pairs ? pairs[2 * task] : 0, q = pairs ? pairs[2 * task + 1] : 1;
  const int64_t cc2 = (int64_t)c * c;
  double *r0 = Rbuf + (int64_t)task * cc2;   // the running factor, in place in Rbuf
  double *r1 = scr + (int64_t)task * cc2;
  const int64_t nchunk = m / c;
  for (int64_t ch = 0; ch < nchunk; ch++) {
    double *a = ch == 0 ? r0 : r1;
    for (int64_t e = threadIdx.x; e < cc2; e += blockDim.x) {
      const int j = (int)(e / c), i = (int)(e - (int64_t)j * c);
      const int64_t col = j < bw ? p * bw + j : q * bw + (j - bw);
      a[e] = G[col * ldg + ch * c + i];
    }
    __syncthreads();
    qr_householder_cta(a, c, bd, sc);
    if (ch > 0) qr_peel_cta(r0, r1, c);
  }
  // nonnegative diagonal
  for (int i = threadIdx.x; i < c; i += blockDim.x)
    if (r0[(int64_t)i * c + i] < 0.0)
      for (int j = i; j < c; j++) r0[(int64_t)j * c + i] = -r0[(int64_t)j * c + i];
}

static int launch_qr_wide(const double *G, int64_t ldg, int64_t m, const int32_t *pairs,
                          int ntask, int w, double *Rbuf, cudaStream_t st) {
  double *scr = nullptr;
  if (cudaMallocAsync((void **)&scr, sizeof(double) * (size_t)ntask * w * w, st) != cudaSuccess)
    return -(int)cudaErrorMemoryAllocation;
  k_qr_wide<<<ntask, kQrWideThreads, 0, st>>>(G, ldg, m, w, pairs, Rbuf, scr, qr_bounds_wide());
  cudaFreeAsync(scr, st);
  return 0;
}

// widths of the GPU QR path (the inner Jacobi that takes R is the v5 kernel)
bool qr_ok(int w, int64_t m) {
  return (w == 16 || w == 32 || w == 64) && m % w == 0 && m >= w;
}

template <int W>
static void launch_qr_t(const double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                        double *Rbuf, cudaStream_t st) {
  k_qr_peeloff<W><<<ntask, kQrThreads, 0, st>>>(G, ldg, m, pairs, Rbuf, qr_bounds());
}

void launch_qr_peeloff(const double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                       int w, double *Rbuf, cudaStream_t st) {
  switch (w) {
#define JH_QR_CASE(W) \
  case W:             \
    launch_qr_t<W>(G, ldg, m, pairs, ntask, Rbuf, st); \
    break;
    JH_QR_CASE(2) JH_QR_CASE(4) JH_QR_CASE(6) JH_QR_CASE(8) JH_QR_CASE(10) JH_QR_CASE(12)
    JH_QR_CASE(14) JH_QR_CASE(16) JH_QR_CASE(18) JH_QR_CASE(20) JH_QR_CASE(22)
    JH_QR_CASE(24) JH_QR_CASE(26) JH_QR_CASE(28) JH_QR_CASE(30) JH_QR_CASE(32)
#undef JH_QR_CASE
    default:
      if (w <= kQrWideMax) launch_qr_wide(G, ldg, m, pairs, ntask, w, Rbuf, st);
      break;
  }
}

}  // namespace jh

// qr_peeloff (blockkernel.py:223-244) of one m x c pair (c even <= 256, m a
// positive multiple of c): R (c x c, column-major, nonnegative diagonal);
// widths above 32 run the global-memory kernel k_qr_wide.
extern "C" int jh_qr_peeloff(const double *A, int64_t lda, int64_t m, int c, double *R,
                             void *stream) {
  if (c < 2 || c > jh::kQrWideMax || c % 2 || m < c || m % c) return -1000;
  if (c > jh::kQrMaxW) {
    jh::g_launches++;
    const int rc = jh::launch_qr_wide(A, lda, m, nullptr, 1, c, R, (cudaStream_t)stream);
    if (rc) return rc;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : -(int)e;
  }
  jh::launch_qr_peeloff(A, lda, m, nullptr, 1, c, R, (cudaStream_t)stream);
  jh::g_launches++;
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}
