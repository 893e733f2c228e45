// Diagnostic probe: rounding semantics of the FP64 tensor-core MMA
// (mma.sync m8n8k4 f64, SASS DMMA) against an in-order fma chain over k.
// If DMMA rounds after every k term in ascending order, the Gram and update
// contractions can run on DMMA tiles and stay bitwise equal to the reference
// (hard part H1).  Dev-only library (tools/dev):
// used by tests/ and the probe scripts, never by the solver.
#include "jh_common.cuh"
#include "jh_fastmath.cuh"

namespace jh {

// test t: A 8x4 row-major, B 4x8 row-major, C 8x8 row-major.
__global__ void k_probe_dmma(const double *__restrict__ A, const double *__restrict__ B,
                             const double *__restrict__ C, double *__restrict__ Dm,
                             double *__restrict__ Df, int ntests) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ntests) return;
  const double *a = A + warp * 32, *b = B + warp * 32, *c = C + warp * 64;
  const int g = lane >> 2, tq = lane & 3;
  const double ra = a[g * 4 + tq];
  const double rb = b[tq * 8 + g];
  const double c0 = c[g * 8 + 2 * tq], c1 = c[g * 8 + 2 * tq + 1];
  double d0, d1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(ra), "d"(rb), "d"(c0), "d"(c1));
  Dm[warp * 64 + g * 8 + 2 * tq] = d0;
  Dm[warp * 64 + g * 8 + 2 * tq + 1] = d1;
  for (int j = 0; j < 2; j++) {
    const int col = 2 * tq + j;
    double acc = c[g * 8 + col];
    for (int k = 0; k < 4; k++) acc = fma(a[g * 4 + k], b[k * 8 + col], acc);
    Df[warp * 64 + g * 8 + col] = acc;
  }
}

}  // namespace jh

extern "C" int jh_probe_dmma(const double *A, const double *B, const double *C, double *Dm,
                             double *Df, int ntests, void *stream) {
  const int threads = 256;
  const int blocks = (ntests * 32 + threads - 1) / threads;
  jh::k_probe_dmma<<<blocks, threads, 0, (cudaStream_t)stream>>>(A, B, C, Dm, Df, ntests);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// Diagnostic: sustained DMMA / DFMA issue rate.  Each warp runs 8 independent
// accumulator chains for `iters` iterations (8 DMMA or 8x? DFMA per
// iteration); the host times the launch to get FMA/s.
namespace jh {
__global__ void k_rate_dmma(int iters, double *out) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_rate_dfma(int iters, double *out) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; i++) d[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) d[i] = fma(a, b, d[i]);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += d[i];
  if (s == 12345.0) out[0] = s;
}
// DMMA with C independent chains per warp (latency probe)
template <int C>
__global__ void k_rate_dmma_c(int iters, double *out) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double d[C][2];
#pragma unroll
  for (int i = 0; i < C; i++) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < iters * 8 / C; it++) {
#pragma unroll
    for (int i = 0; i < C; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < C; i++) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

// warps 0-3 (mod 8) DMMA, 4-7 DFMA: with 8 warps per CTA every SMSP runs
// one of each (do the two FP64 paths add up?)
__global__ void k_rate_mixed(int iters, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double s = 0.0;
  if (((warp >> 2) & 1) == 0) {
    double d[8][2];
#pragma unroll
    for (int i = 0; i < 8; i++) d[i][0] = d[i][1] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
      for (int i = 0; i < 8; i++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d[i][0]), "+d"(d[i][1])
                     : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; i++) s += d[i][0] + d[i][1];
  } else {
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; i++) d[i] = i;
    // 8x the DFMA iterations so both halves run about as long
    for (int it = 0; it < 8 * iters; it++) {
#pragma unroll
      for (int i = 0; i < 8; i++) d[i] = fma(a, b, d[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; i++) s += d[i];
  }
  if (s == 12345.0) out[0] = s;
}
}  // namespace jh

// FMAs executed = ctas * threads/32 * iters * 8 * (256 for DMMA, 32 for DFMA)
// kind 2 (mixed): half the warps DMMA (iters * 8 * 256), half DFMA
// (8 iters * 8 * 32): the same FMA count per warp.  kind 10 + C: DMMA with C
// chains per warp (C in 1, 2, 4, 8, 16), same FMA count as kind 0.
extern "C" int jh_probe_rate(int kind, int ctas, int threads, int iters, double *out,
                             void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (kind == 0)
    jh::k_rate_dmma<<<ctas, threads, 0, st>>>(iters, out);
  else if (kind == 1)
    jh::k_rate_dfma<<<ctas, threads, 0, st>>>(iters, out);
  else if (kind == 2)
    jh::k_rate_mixed<<<ctas, threads, 0, st>>>(iters, out);
  else if (kind == 11)
    jh::k_rate_dmma_c<1><<<ctas, threads, 0, st>>>(iters, out);
  else if (kind == 12)
    jh::k_rate_dmma_c<2><<<ctas, threads, 0, st>>>(iters, out);
  else if (kind == 14)
    jh::k_rate_dmma_c<4><<<ctas, threads, 0, st>>>(iters, out);
  else if (kind == 18)
    jh::k_rate_dmma_c<8><<<ctas, threads, 0, st>>>(iters, out);
  else if (kind == 26)
    jh::k_rate_dmma_c<16><<<ctas, threads, 0, st>>>(iters, out);
  else
    return -1000;
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// Diagnostic: single-thread dependent-chain latencies in cycles per op:
// out[0] DFMA, out[1] DMUL, out[2] division, out[3] sqrt, out[4] rotation_core
// (trig), out[5] shared-memory load (pointer chase).
namespace jh {
__global__ void k_latency(double seed, double *out) {
  __shared__ int chase[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) chase[i] = (i * 37 + 11) & 255;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int N = 1024;
  double x = seed, y = 1.0000001, z = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < N; i++) x = fma(x, y, z);
  long long t1 = clock64();
  out[0] = (double)(t1 - t0) / N + 0.0 * x;
  double w = seed;
  t0 = clock64();
  for (int i = 0; i < N; i++) w = w * y;
  t1 = clock64();
  out[1] = (double)(t1 - t0) / N + 0.0 * w;
  double d = seed + 2.0;
  t0 = clock64();
  for (int i = 0; i < N; i++) d = 3.0 / d;
  t1 = clock64();
  out[2] = (double)(t1 - t0) / N + 0.0 * d;
  double s = seed + 3.0;
  t0 = clock64();
  for (int i = 0; i < N; i++) s = sqrt(s) + 1.0;
  t1 = clock64();
  out[3] = (double)(t1 - t0) / N + 0.0 * s;
  double hpq = 0.3 + seed, cs, tn;
  t0 = clock64();
  for (int i = 0; i < N; i++) {
    rotation_core(1.5, 1.0, hpq, 1.0, cs, tn);
    hpq = 0.3 + tn * 1e-9;
  }
  t1 = clock64();
  out[4] = (double)(t1 - t0) / N + 0.0 * cs;
  int idx = (int)seed & 255;
  t0 = clock64();
  for (int i = 0; i < N; i++) idx = chase[idx];
  t1 = clock64();
  out[5] = (double)(t1 - t0) / N + 0.0 * idx;
  bool ok = true;
  double d2 = seed + 2.0;
  t0 = clock64();
  for (int i = 0; i < N; i++) d2 = div_fp(3.0, d2, ok);
  t1 = clock64();
  out[6] = (double)(t1 - t0) / N + 0.0 * d2;
  double s2 = seed + 3.0;
  t0 = clock64();
  for (int i = 0; i < N; i++) s2 = sqrt_fp(s2, ok) + 1.0;
  t1 = clock64();
  out[7] = (double)(t1 - t0) / N + 0.0 * s2;
  double h2 = 0.3 + seed, c2, tn2, sp, sq;
  bool okf;
  t0 = clock64();
  for (int i = 0; i < N; i++) {
    rotation_core_fast(1.5, 1.0, h2, 1.0, c2, tn2, sp, sq, okf);
    h2 = 0.3 + tn2 * 1e-9;
  }
  t1 = clock64();
  out[8] = (double)(t1 - t0) / N + 0.0 * c2 + (ok && okf ? 0.0 : 1e9);
}
}  // namespace jh

extern "C" int jh_probe_latency(double *out, void *stream) {
  jh::k_latency<<<1, 32, 0, (cudaStream_t)stream>>>(0.5, out);  // out[0..8]
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}

// Diagnostic / test: the branch-free fast paths (jh_fastmath.cuh) against the
// IEEE operators.  cnt[0] = division mismatches on fast-ok lanes, cnt[1] =
// division fast-path rejections, cnt[2] / cnt[3] the same for sqrt (of |a|).
#include "jh_fastmath.cuh"
namespace jh {
__global__ void k_probe_fastmath(const double *__restrict__ a, const double *__restrict__ b,
                                 int64_t n, unsigned long long *cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    const double q = div_fp(a[i], b[i], ok);
    const double qi = a[i] / b[i];
    if (!ok)
      atomicAdd(&cnt[1], 1ull);
    else if (__double_as_longlong(q) != __double_as_longlong(qi))
      atomicAdd(&cnt[0], 1ull);
    bool ok2 = true;
    const double x = fabs(a[i]);
    const double s = sqrt_fp(x, ok2);
    const double si = sqrt(x);
    if (!ok2)
      atomicAdd(&cnt[3], 1ull);
    else if (__double_as_longlong(s) != __double_as_longlong(si))
      atomicAdd(&cnt[2], 1ull);
  }
}
}  // namespace jh

extern "C" int jh_probe_fastmath(const double *a, const double *b, int64_t n,
                                 unsigned long long *cnt, void *stream) {
  jh::k_probe_fastmath<<<1184, 256, 0, (cudaStream_t)stream>>>(a, b, n, cnt);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}
