// Robust column norms (DRDSSQ, reference Appendix A / pkg/src/jhsvd/robustnorm.py)
// for the sigma extraction (driver.py:230-238), U = G / sigma (driver.py:294-297)
// and the input scaling check (driver.py:99-112).
//
// One CTA per column.  The sum of squares follows the reference's fixed
// reduction layout exactly: 256-element leaves, each one in-order fma chain
// from +0.0, combined along the fixed binary tree of _tree_combine, with the
// scaled three-partition fallback of _sum_squares_core when the plain sum
// over/underflows.  The result is therefore bitwise the reference's.
#include "jh_common.cuh"
#include "jh_kernels.h"
#include "jh_robust.cuh"

#include <cmath>

namespace jh {

constexpr int kNormThreads = 256;

// -- device reduction pieces ---------------------------------------------------

// leaves of 256 in-order fma chains, optionally restricted to lo <= |x| <= hi
// and scaled by 2**j (_tree_sumsq_plain / _tree_sumsq_selected), then the
// fixed-tree combine (_tree_combine) by thread 0.  Result valid in thread 0.
__device__ double cta_tree_sumsq(const double *__restrict__ x, int64_t m, bool selected,
                                 double lo, double hi, int j, double *part, int leaf) {
  const int64_t nleaf = cdiv(m, leaf);
  for (int64_t c = threadIdx.x; c < nleaf; c += blockDim.x) {
    double acc = 0.0;
    const int64_t end = min64((c + 1) * leaf, m);
    if (!selected) {
      for (int64_t i = c * leaf; i < end; i++) acc = fma(x[i], x[i], acc);
    } else {
      for (int64_t i = c * leaf; i < end; i++) {
        const double a = fabs(x[i]);
        if (a > 0.0 && lo <= a && a <= hi) {
          const double v = ldexp(x[i], j);
          acc = fma(v, v, acc);
        }
      }
    }
    part[c] = acc;
  }
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    int64_t k = nleaf;
    while (k > 1) {
      const int64_t half = (k + 1) / 2;
      for (int64_t i = 0; i < k / 2; i++) part[i] = part[2 * i] + part[2 * i + 1];
      if (k % 2) part[half - 1] = part[k - 1];
      k = half;
    }
    r = part[0];
  }
  __syncthreads();
  return r;
}

// norm2 of one column (robustnorm.py:242-300): (js, sigma), ||x|| = sigma / 2**js,
// and the sum of squares in common form (j, v) = v * 2**-j (_sum_squares_core).
// leaf = the reference's chunk (256 by default); force_scaled skips the plain
// fast path (robustnorm.sum_squares(force_scaled=True)).  Valid in thread 0.
__device__ void cta_norm2(const double *__restrict__ x, int64_t m, double mu_tilde,
                          double nu_hat, double *part, int64_t &js_out, double &s_out,
                          int leaf = kLeaf, bool force_scaled = false,
                          int64_t *jsq_out = nullptr, double *vsq_out = nullptr) {
  __shared__ double s_big[kNormThreads / 32], s_small[kNormThreads / 32];
  __shared__ double s_plain;
  __shared__ int s_done;
  double big = 0.0, small = kNu;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double a = fabs(x[i]);
    if (a > big) big = a;
    if (0.0 < a && a < small) small = a;
  }
  for (int off = 16; off; off >>= 1) {
    big = fmax(big, __shfl_xor_sync(0xffffffffu, big, off));
    small = fmin(small, __shfl_xor_sync(0xffffffffu, small, off));
  }
  if ((threadIdx.x & 31) == 0) {
    s_big[threadIdx.x >> 5] = big;
    s_small[threadIdx.x >> 5] = small;
  }
  __syncthreads();
  big = 0.0;
  small = kNu;
  for (int k = 0; k < (int)(blockDim.x >> 5); k++) {
    big = fmax(big, s_big[k]);
    small = fmin(small, s_small[k]);
  }
  js_out = 0;
  s_out = 0.0;
  if (jsq_out) *jsq_out = 0;
  if (vsq_out) *vsq_out = 0.0;
  if (m == 0 || big == 0.0) return;
  const double plain = force_scaled ? 0.0 : cta_tree_sumsq(x, m, false, 0.0, 0.0, 0, part, leaf);
  if (threadIdx.x == 0) {
    s_plain = plain;
    s_done = (!force_scaled && isfinite(plain) && small * small >= kMu) ? 1 : 0;
  }
  __syncthreads();
  int64_t jres = 0;
  double vres = 0.0;
  if (s_done) {
    if (threadIdx.x == 0) common_form(0, s_plain, jres, vres);
  } else {
    int64_t jsv[3] = {0, 0, 0};
    double vsv[3] = {0.0, 0.0, 0.0};
    int count = 0;
    if (small <= nu_hat && big >= mu_tilde) {
      const double s1 = cta_tree_sumsq(x, m, true, mu_tilde, nu_hat, 0, part, leaf);
      if (threadIdx.x == 0 && s1 != 0.0) common_form(0, s1, jsv[count], vsv[count]);
      if (threadIdx.x == 0 && s1 != 0.0) count++;
    }
    if (big > nu_hat) {
      const int j2 = scale_exponent(big, nu_hat, false);
      const double s2 = cta_tree_sumsq(x, m, true, nextafter(nu_hat, kNu), kNu, j2, part, leaf);
      if (threadIdx.x == 0 && s2 != 0.0) {
        common_form(-2 * (int64_t)j2, s2, jsv[count], vsv[count]);
        count++;
      }
    }
    if (small < mu_tilde) {
      const int j0 = scale_exponent(small, mu_tilde, true);
      const double s0 = cta_tree_sumsq(x, m, true, 0.0, nextafter(mu_tilde, 0.0), j0, part, leaf);
      if (threadIdx.x == 0 && s0 != 0.0) {
        common_form(-2 * (int64_t)j0, s0, jsv[count], vsv[count]);
        count++;
      }
    }
    if (threadIdx.x == 0 && count) {
      for (int a = 0; a < count - 1; a++)
        for (int b = a + 1; b < count; b++)
          if (jsv[a] > jsv[b] || (jsv[a] == jsv[b] && vsv[a] > vsv[b])) {
            const int64_t tj = jsv[a];
            jsv[a] = jsv[b];
            jsv[b] = tj;
            const double tv = vsv[a];
            vsv[a] = vsv[b];
            vsv[b] = tv;
          }
      int64_t ja = jsv[0];
      double va = vsv[0];
      for (int k = 1; k < count; k++) {
        common_form(ja, va, ja, va);
        add_scaled(ja, va, jsv[k], vsv[k], ja, va);
      }
      common_form(ja, va, jres, vres);
    }
  }
  if (threadIdx.x == 0) {
    if (jsq_out) *jsq_out = jres;
    if (vsq_out) *vsq_out = vres;
  }
  if (threadIdx.x == 0 && vres != 0.0) {
    js_out = -(jres / 2);  // jres is even in common form
    s_out = sqrt(vres);
  }
}

// robustnorm.sum_squares / norm2 with the reference's chunk and
// force_scaled options, one CTA per column; any output may be null
__global__ void __launch_bounds__(kNormThreads)
k_robust_norms(const double *__restrict__ G, int64_t ldg, int64_t m, double mu_tilde,
               double nu_hat, int leaf, int force_scaled, int64_t *jsq, double *vsq,
               int64_t *js, double *s) {
  extern __shared__ double part[];
  const int64_t col = blockIdx.x;
  int64_t a, jq;
  double b, vq;
  cta_norm2(G + col * ldg, m, mu_tilde, nu_hat, part, a, b, leaf, force_scaled != 0, &jq, &vq);
  if (threadIdx.x == 0) {
    if (jsq) jsq[col] = jq;
    if (vsq) vsq[col] = vq;
    if (js) js[col] = a;
    if (s) s[col] = b;
  }
}

// batch rotation parameters (rotation.py:90-124): in[i] = (h_pp, h_qq, h_pq),
// t[i] = +1 trigonometric / -1 hyperbolic; out[i] = (cs, tn, ok)
__global__ void k_rotations(const double *__restrict__ in, const double *__restrict__ t,
                            int64_t n, double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double cs = 1.0, tn = 0.0;
    const bool ok = rotation_core(in[3 * i], in[3 * i + 1], in[3 * i + 2], t[i], cs, tn);
    out[3 * i] = cs;
    out[3 * i + 1] = tn;
    out[3 * i + 2] = ok ? 1.0 : 0.0;
  }
}

// mode 0: raw (js, sigma) per column
// mode 1: scaling check, atomicMin(bad, 1-based column) outside [mu_lo, hi_lim]
// mode 2: sigma_i = ldexp(s, -js) and U[:, i] = G[:, i] / sigma_i;
//         atomicMin(bad, i + 1) for a zero column
__global__ void __launch_bounds__(kNormThreads)
k_colnorm(const double *__restrict__ G, int64_t ldg, int64_t m, int64_t n, double mu_tilde,
          double nu_hat, int mode, double lo_lim, double hi_lim, int64_t *js_out,
          double *s_out, double *U, int64_t ldu, unsigned long long *bad) {
  extern __shared__ double part[];
  __shared__ double s_sigma;
  const int64_t col = blockIdx.x;
  const double *x = G + col * ldg;
  int64_t js;
  double s;
  cta_norm2(x, m, mu_tilde, nu_hat, part, js, s);
  if (threadIdx.x == 0) {
    if (mode == 0) {
      js_out[col] = js;
      s_out[col] = s;
    } else if (mode == 1) {
      const double nrm = (s != 0.0) ? ldexp(s, (int)(-js)) : 0.0;
      if (nrm < lo_lim || nrm > hi_lim) atomicMin(bad, (unsigned long long)(col + 1));
    } else {
      const double sig = (s != 0.0) ? ldexp(s, (int)(-js)) : 0.0;
      s_out[col] = sig;
      if (s == 0.0) atomicMin(bad, (unsigned long long)(col + 1));
    }
    s_sigma = (s != 0.0) ? ldexp(s, (int)(-js)) : 0.0;
  }
  __syncthreads();
  if (mode == 2) {
    const double sig = s_sigma;
    double *u = U + col * ldu;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) u[i] = x[i] / sig;
  }
}

// -- host double-double (for safe_bounds; _fp.py:46-157, robustnorm.py:90-101)

static void h_two_sum(double a, double b, double &s, double &e) {
  s = a + b;
  const double v = s - a;
  e = (a - (s - v)) + (b - v);
}
static void h_quick_two_sum(double a, double b, double &s, double &e) {
  s = a + b;
  e = b - (s - a);
}
static void h_dd_add(double ah, double al, double bh, double bl, double &rh, double &rl) {
  double s1, s2, t1, t2;
  h_two_sum(ah, bh, s1, s2);
  h_two_sum(al, bl, t1, t2);
  s2 += t1;
  h_quick_two_sum(s1, s2, s1, s2);
  s2 += t2;
  h_quick_two_sum(s1, s2, rh, rl);
}
static void h_dd_add_d(double ah, double al, double b, double &rh, double &rl) {
  double s1, s2;
  h_two_sum(ah, b, s1, s2);
  s2 += al;
  h_quick_two_sum(s1, s2, rh, rl);
}
static void h_dd_mul(double ah, double al, double bh, double bl, double &rh, double &rl) {
  double p1 = ah * bh;
  double p2 = std::fma(ah, bh, -p1);
  p2 += ah * bl + al * bh;
  h_quick_two_sum(p1, p2, rh, rl);
}
static void h_dd_mul_d(double ah, double al, double b, double &rh, double &rl) {
  double p1 = ah * b;
  double p2 = std::fma(ah, b, -p1);
  p2 += al * b;
  h_quick_two_sum(p1, p2, rh, rl);
}
static void h_dd_div(double ah, double al, double bh, double bl, double &rh, double &rl) {
  double q1 = ah / bh, th, tl, xh, xl;
  h_dd_mul_d(bh, bl, q1, th, tl);
  h_dd_add(ah, al, -th, -tl, xh, xl);
  double q2 = xh / bh;
  h_dd_mul_d(bh, bl, q2, th, tl);
  h_dd_add(xh, xl, -th, -tl, xh, xl);
  const double q3 = xh / bh;
  h_quick_two_sum(q1, q2, q1, q2);
  h_dd_add_d(q1, q2, q3, rh, rl);
}
static void h_dd_sqrt(double ah, double al, double &rh, double &rl) {
  if (ah == 0.0) {
    rh = rl = 0.0;
    return;
  }
  const double s = std::sqrt(ah);
  const double ph = s * s;
  const double pl = std::fma(s, s, -ph);
  double xh, xl;
  h_dd_add(ah, al, -ph, -pl, xh, xl);
  const double e = xh / (2.0 * s);
  h_quick_two_sum(s, e, rh, rl);
}

}  // namespace jh

using namespace jh;

extern "C" {

// safe_bounds(n) (robustnorm.py:90-113): inclusive magnitudes [mu_tilde,
// nu_hat] whose squares and tree sums of n terms cannot over/underflow.
void jh_safe_bounds(int64_t n, double *mu_tilde, double *nu_hat) {
  int d = 0;
  for (int64_t m = n - 1; m > 0; m >>= 1) d++;
  if (d < 1) d = 1;
  const double gamma = 1.0 - 0x1p-53;
  volatile double one = 1.0, eps = 0x1p-53;
  const double delta = one + eps;  // rounds to 1.0, as in the reference
  double h, l, sh, sl;
  h_dd_div(kMu, 0.0, gamma, 0.0, h, l);
  h_dd_sqrt(h, l, sh, sl);
  *mu_tilde = (sl > 0.0) ? std::nextafter(sh, INFINITY) : sh;
  double dh = 1.0, dl = 0.0;
  for (int i = 0; i < d + 1; i++) h_dd_mul(dh, dl, delta, 0.0, dh, dl);
  dh = std::ldexp(dh, d);
  dl = std::ldexp(dl, d);
  h_dd_div(kNu, 0.0, dh, dl, h, l);
  h_dd_sqrt(h, l, sh, sl);
  *nu_hat = (sl < 0.0) ? std::nextafter(sh, 0.0) : sh;
}

static size_t norm_smem(int64_t m, int leaf = kLeaf) {
  return sizeof(double) * (size_t)(cdiv(m, leaf) + 1);
}

static int prep_norm(int64_t m) {
  const size_t need = norm_smem(m);
  if (need > 48 * 1024) ensure_smem((const void *)k_colnorm, (int)need);
  return 0;
}

// Raw robust norms of the n columns of G (m x n, ld ldg): ||G[:, i]|| =
// s[i] / 2**js[i] (robustnorm.norm2, chunk 256).
int jh_column_norms(const double *G, int64_t ldg, int64_t m, int64_t n, int64_t *js,
                    double *s, void *stream) {
  double mu, nu;
  jh_safe_bounds(m, &mu, &nu);
  prep_norm(m);
  g_launches++;
  k_colnorm<<<(unsigned)n, kNormThreads, norm_smem(m), (cudaStream_t)stream>>>(
      G, ldg, m, n, mu, nu, 0, 0.0, 0.0, js, s, nullptr, 0, nullptr);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// check_column_scaling (driver.py:99-112): *bad (device, init ULLONG_MAX)
// receives the smallest 1-based column whose norm lies outside
// [mu_tilde, sqrt(nu_hat)] for vectors of length m.
int jh_check_scaling(const double *G, int64_t ldg, int64_t m, int64_t n,
                     unsigned long long *bad, void *stream) {
  double mu, nu;
  jh_safe_bounds(m, &mu, &nu);
  prep_norm(m);
  g_launches++;
  k_colnorm<<<(unsigned)n, kNormThreads, norm_smem(m), (cudaStream_t)stream>>>(
      G, ldg, m, n, mu, nu, 1, mu, std::sqrt(nu), nullptr, nullptr, nullptr, 0, bad);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// extract_sigma + U (driver.py:230-238, 294-297): sigma[i] = ||G[:, i]||,
// U[:, i] = G[:, i] / sigma[i]; *bad gets the smallest 1-based zero column.
int jh_sigma_u(const double *G, int64_t ldg, int64_t m, int64_t n, double *sigma, double *U,
               int64_t ldu, unsigned long long *bad, void *stream) {
  double mu, nu;
  jh_safe_bounds(m, &mu, &nu);
  prep_norm(m);
  g_launches++;
  k_colnorm<<<(unsigned)n, kNormThreads, norm_smem(m), (cudaStream_t)stream>>>(
      G, ldg, m, n, mu, nu, 2, 0.0, 0.0, nullptr, sigma, U, ldu, bad);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// robustnorm.sum_squares / norm2 (robustnorm.py:324-334) of the n columns
// of G (m x n, ld ldg) with the reference's chunk (leaf length) and
// force_scaled options: sum of squares v * 2**-j in common form (jsq, vsq)
// and the norm s / 2**js; each output may be NULL.
int jh_robust_norms(const double *G, int64_t ldg, int64_t m, int64_t n, int chunk,
                    int force_scaled, int64_t *jsq, double *vsq, int64_t *js, double *s,
                    void *stream) {
  if (chunk < 1 || m < 0 || n < 0) return -1000;
  if (n == 0) return 0;
  double mu, nu;
  jh_safe_bounds(m > 0 ? m : 1, &mu, &nu);
  const size_t smem = norm_smem(m, chunk);
  if (smem > 227 * 1024) return -1000;
  if (smem > 48 * 1024) ensure_smem((const void *)k_robust_norms, (int)smem);
  g_launches++;
  k_robust_norms<<<(unsigned)n, kNormThreads, smem, (cudaStream_t)stream>>>(
      G, ldg, m, mu, nu, chunk, force_scaled, jsq, vsq, js, s);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// rotation parameters of n pivot Grams (rotation.py:90-124 _rotation_core):
// in (device, n x 3: h_pp, h_qq, h_pq), t (device, n: +1 / -1),
// out (device, n x 3: cs, tn, 1 = ok / 0 = hyperbolic domain failure).
int jh_rotations(const double *in, const double *t, int64_t n, double *out, void *stream) {
  if (n < 0) return -1000;
  if (n == 0) return 0;
  g_launches++;
  const int64_t blocks = (n + 255) / 256;
  k_rotations<<<(unsigned)(blocks < 1024 ? blocks : 1024), 256, 0, (cudaStream_t)stream>>>(
      in, t, n, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// Scalar DRDSSQ helpers of robustnorm.py:116-162 on the host (the same code
// the kernels inline): common_form, add_scaled, scale_exponent.
void jh_common_form(int64_t j, double v, int64_t *jo, double *vo) {
  int64_t a;
  double b;
  common_form(j, v, a, b);
  *jo = a;
  *vo = b;
}

void jh_add_scaled(int64_t ja, double va, int64_t jb, double vb, int64_t *jo, double *vo) {
  int64_t a;
  double b;
  add_scaled(ja, va, jb, vb, a, b);
  *jo = a;
  *vo = b;
}

int jh_scale_exponent(double f, double t, int up) { return scale_exponent(f, t, up != 0); }

}  // extern "C"
