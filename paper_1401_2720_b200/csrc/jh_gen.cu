// Synthetic inputs for the BASELINE workloads: G = Q [diag(sigma); 0] W^T
// with Q, W products of random Givens butterflies (plus J-orthogonal
// hyperbolic layers for the HSVD workload), generated in HBM.
//
// Why not a QR of a Gaussian matrix: the whole-solve oracle goldens of the
// 16384^2 / 8192^2 / 131072 x 8192 workloads are computed offline on the
// host (tools/oracle_offline.py), so the device generator has to produce the
// same bytes as its host twin (oracle/gen_butterfly.c).  Every rotation
// parameter comes from a counter hash of (seed, layer, pair) through
// correctly rounded + - * / sqrt only, and every element sees the same
// sequence of layers, so both sides agree bit for bit.  Layer schedule,
// hash and formulas: see oracle/gen_butterfly.c (the two are pinned against
// each other by tests/test_gen.py).
//
// Work: passes * (log2 n + 1) column layers on the top n rows and
// passes * log2 m row layers, each one read + write of the touched block:
// ~0.25 TB of HBM traffic at 16384^2 (tens of milliseconds).
#include "jh_common.cuh"

#include <cstdint>

namespace jh {

__device__ __forceinline__ uint64_t gen_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double gen_draw_t(uint64_t seed, uint64_t layer, uint64_t pair) {
  const uint64_t h = gen_mix64(gen_mix64(seed * 0x9E3779B97F4A7C15ULL + layer) ^
                               (pair * 0xD1B54A32D192ED03ULL));
  const double u = __dmul_rn((double)(h >> 11), 0x1p-53);
  return __dsub_rn(__dmul_rn(2.0, u), 1.0);
}

// tables[layer][pair] = (c, s) (trig) or (ch, sh) (hyperbolic)
__global__ void k_gen_tables(double2 *__restrict__ tab, int nlayers, int64_t npairs,
                             uint64_t seed, uint64_t layer0, const int *__restrict__ kind,
                             double tanh_max) {
  const int64_t total = (int64_t)nlayers * npairs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(e / npairs);
    const int64_t k = e - (int64_t)l * npairs;
    const double t = gen_draw_t(seed, layer0 + l, (uint64_t)k);
    double a, b;
    if (kind && kind[l] < 0) {
      const double th = __dmul_rn(tanh_max, t);
      a = __ddiv_rn(1.0, __dsqrt_rn(__dsub_rn(1.0, __dmul_rn(th, th))));
      b = __dmul_rn(th, a);
    } else {
      const double t2 = __dmul_rn(t, t);
      const double d = __dadd_rn(1.0, t2);
      a = __ddiv_rn(__dsub_rn(1.0, t2), d);
      b = __ddiv_rn(__dmul_rn(2.0, t), d);
    }
    tab[e] = make_double2(a, b);
  }
}

__global__ void k_gen_init(double *__restrict__ G, int64_t ldg, int64_t m, int64_t n,
                           const double *__restrict__ sigma) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    G[j * ldg + i] = (i == j) ? sigma[j] : 0.0;
  }
}

// One column layer on rows [0, n): l >= 0 butterflies (j, j + 2^l) inside
// classes of width cls; l < 0 the hyperbolic layer (k, k + n/2).
__global__ void k_gen_col_layer(double *__restrict__ G, int64_t ldg, int64_t n, int64_t cls,
                                int l, const double2 *__restrict__ cs) {
  const int64_t total = (n / 2) * n;  // (pair, row), rows fastest
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kk = e / n, i = e - kk * n;
    int64_t j, j2;
    const double2 p = cs[kk];
    double x, y, xn, yn;
    if (l < 0) {
      j = kk;
      j2 = kk + n / 2;
      x = G[j * ldg + i];
      y = G[j2 * ldg + i];
      xn = __dadd_rn(__dmul_rn(p.x, x), __dmul_rn(p.y, y));
      yn = __dadd_rn(__dmul_rn(p.y, x), __dmul_rn(p.x, y));
    } else {
      const int64_t h = (int64_t)1 << l;
      const int64_t base = (kk / (cls / 2)) * cls, k = kk % (cls / 2);
      j = base + (((k >> l) << (l + 1)) | (k & (h - 1)));
      j2 = j + h;
      x = G[j * ldg + i];
      y = G[j2 * ldg + i];
      xn = __dsub_rn(__dmul_rn(p.x, x), __dmul_rn(p.y, y));
      yn = __dadd_rn(__dmul_rn(p.y, x), __dmul_rn(p.x, y));
    }
    G[j * ldg + i] = xn;
    G[j2 * ldg + i] = yn;
  }
}

// One row layer over all m rows of every column: pairs (i, i + 2^l).
__global__ void k_gen_row_layer(double *__restrict__ G, int64_t ldg, int64_t m, int64_t n, int l,
                                const double2 *__restrict__ cs) {
  const int64_t half = m / 2, total = half * n;
  const int64_t h = (int64_t)1 << l;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / half, k = e - j * half;
    const int64_t i = ((k >> l) << (l + 1)) | (k & (h - 1));
    const double2 p = cs[k];
    double *col = G + j * ldg;
    const double x = col[i], y = col[i + h];
    col[i] = __dsub_rn(__dmul_rn(p.x, x), __dmul_rn(p.y, y));
    col[i + h] = __dadd_rn(__dmul_rn(p.y, x), __dmul_rn(p.x, y));
  }
}

static int ilog2_i64(int64_t x) {
  int k = 0;
  while (((int64_t)1 << (k + 1)) <= x) k++;
  return k;
}

struct GenPlan {
  int64_t cls;
  int lc, lr, hyp, ncl, nrl;
  int64_t col_tab, row_tab, kinds;  // byte offsets in the workspace
  int64_t bytes;
};

static bool gen_plan(int64_t m, int64_t n, int64_t n_plus, int passes, GenPlan *p) {
  if (m < n || n < 2 || (m & (m - 1)) || (n & (n - 1)) || passes < 1) return false;
  if (n_plus != n && n_plus != n / 2) return false;
  p->cls = (n_plus == n) ? n : n / 2;
  p->lc = ilog2_i64(p->cls);
  p->lr = ilog2_i64(m);
  p->hyp = p->cls != n;
  p->ncl = passes * (p->lc + p->hyp);
  p->nrl = passes * p->lr;
  p->col_tab = 0;
  p->row_tab = p->col_tab + (int64_t)p->ncl * (n / 2) * 16;
  p->kinds = p->row_tab + (int64_t)p->nrl * (m / 2) * 16;
  p->bytes = p->kinds + 4 * (int64_t)(p->ncl + 1) + 256;
  return true;
}

static int grid_for(int64_t total) {
  const int64_t b = (total + 255) / 256;
  return (int)(b < 148 * 64 ? (b > 0 ? b : 1) : 148 * 64);
}

}  // namespace jh

namespace jh {
extern unsigned long long g_launches;
}
using namespace jh;

extern "C" {

int64_t jh_gen_workspace_bytes(int64_t m, int64_t n, int64_t n_plus, int passes) {
  GenPlan p;
  return gen_plan(m, n, n_plus, passes, &p) ? p.bytes : -1;
}

int jh_gen_butterfly(double *G, int64_t ldg, int64_t m, int64_t n, const double *sigma,
                     int64_t n_plus, unsigned long long seed, int passes, double tanh_max,
                     void *workspace, int64_t ws_bytes, void *stream) {
  GenPlan p;
  if (!gen_plan(m, n, n_plus, passes, &p) || ldg < m) return -1000;
  if (ws_bytes < p.bytes) return -1001;
  cudaStream_t st = (cudaStream_t)stream;
  char *ws = (char *)workspace;
  double2 *ctab = (double2 *)(ws + p.col_tab);
  double2 *rtab = (double2 *)(ws + p.row_tab);
  int *kinds = (int *)(ws + p.kinds);
  // column-layer kinds (host -> device): log2 h per butterfly layer, -1 hyperbolic
  int hk[4096];
  if (p.ncl > 4096) return -1000;
  for (int c = 0, q = 0; q < passes; q++) {
    for (int l = 0; l < p.lc; l++) hk[c++] = l;
    if (p.hyp) hk[c++] = -1;
  }
  cudaMemcpyAsync(kinds, hk, sizeof(int) * p.ncl, cudaMemcpyHostToDevice, st);
  // draws: column layers take layer ids [0, ncl), row layers [ncl, ncl + nrl)
  k_gen_tables<<<grid_for((int64_t)p.ncl * (n / 2)), 256, 0, st>>>(ctab, p.ncl, n / 2, seed, 0,
                                                                     kinds, tanh_max);
  k_gen_tables<<<grid_for((int64_t)p.nrl * (m / 2)), 256, 0, st>>>(rtab, p.nrl, m / 2, seed,
                                                                     p.ncl, nullptr, tanh_max);
  k_gen_init<<<grid_for(m * n), 256, 0, st>>>(G, ldg, m, n, sigma);
  for (int c = 0; c < p.ncl; c++)
    k_gen_col_layer<<<grid_for((n / 2) * n), 256, 0, st>>>(G, ldg, n, p.cls, hk[c],
                                                            ctab + (int64_t)c * (n / 2));
  for (int r = 0; r < p.nrl; r++)
    k_gen_row_layer<<<grid_for((m / 2) * n), 256, 0, st>>>(G, ldg, m, n, r % p.lr,
                                                            rtab + (int64_t)r * (m / 2));
  g_launches += 3 + p.ncl + p.nrl;
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // extern "C"
