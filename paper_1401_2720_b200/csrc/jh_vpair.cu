#include <atomic>
// V update of a pair of p-steps in one pass over V (engine 1).
//
// V is read by nothing else until the sweep ends, so the post-multiplication
// of V by the transforms of p-steps a and a+1 (reference driver.py:165-172,
// blockkernel.py:407-428) can run as one pass: for the rrow tables, the pairs
// of two consecutive p-steps form 4-cycles over four block-columns (the
// cycle plan, jh_plan.cu), so the 64 V columns of a cycle go through shared
// memory once, get the two step-a transforms and then the two step-(a+1)
// transforms, and go back -- V moves through HBM once per two p-steps.
// Every V row still receives the same transformations in the same order
// with the same in-order DMMA chains, so the result is bitwise that of two
// per-p-step updates.
//
// CTA = TMA producer warp + 4 DMMA warps, the layout of the per-p-step
// update kernel (each transform's V' held in registers): warps 1 and 2
// apply t1 / t2 of p-step a to all 64 rows of a chunk (slot columns 0-31 /
// 32-63), in place; warps 3 and 4 then apply u1 / u2 of p-step a+1 to their
// block pairs and store the final values straight from the accumulators.
// The two phases are pipelined over a 3-stage ring (chunk c's second phase
// overlaps chunk c+1's first).  Grid: (cycles, row slabs).
#include "jh_gram.cuh"
#include "jh_kernels.h"
#include "jh_update.cuh"

namespace jh {

namespace {

__device__ __forceinline__ void fence_async_smem_cta() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// thread 0 spins until flag == epoch (acquire), then the CTA proceeds
__device__ __forceinline__ void wait_flag_cta(const int64_t *flag, int64_t epoch) {
  if (threadIdx.x == 0) {
    for (;;) {
      int64_t v;
      asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
      if (v == epoch) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
}

constexpr int kVW = 32;
constexpr int kVCols = 64;
#ifndef JH_VRCH
#define JH_VRCH 64
#endif
#ifndef JH_VSTG
#define JH_VSTG 3
#endif
constexpr int kVStages = JH_VSTG;    // ring stages of the V items
constexpr int kVRch = JH_VRCH;       // rows per V-item chunk
constexpr int kVLd = kVRch + 4;      // = 4 (mod 16): conflict-free 64-bit shared accesses
// Row slabs of the mixed launch: from 256 tasks per p-step on, longer G and
// V slabs (fewer CTAs, less pipeline fill and drain per CTA); below that the
// short ones keep enough CTAs for the SMs.  A/B at n = 16384 (ms per
// p-step, G/V slab rows): 2048/512 1.952, 2048/1024 1.915, 4096/1024 1.89,
// 4096/1536 1.882, 8192/2048 1.891; n = 4096: 4096/1536 is 8 % slower.
constexpr int kMixBigTasks = 256;
#ifndef JH_MGST
#define JH_MGST 3
#endif
constexpr int kMixGStages = JH_MGST;  // ring stages of the G items (inside the union with the V ring)
#ifndef JH_MGRCH
#define JH_MGRCH 128
#endif
constexpr int kMixGRch = JH_MGRCH;  // rows per G-item chunk
#ifndef JH_VORDER
#define JH_VORDER 0
#endif
constexpr int kMixVOrder = JH_VORDER;  // ring stages of the G items (the union with the V ring)
#ifndef JH_GBIG
#define JH_GBIG 4096
#endif
#ifndef JH_VBIG
#define JH_VBIG 1536
#endif
constexpr int kMixGSlab[2] = {2048, JH_GBIG};
constexpr int kMixVSlab[2] = {512, JH_VBIG};

struct VpSmem {
  double ring[kVStages][kVCols][kVLd];
  uint64_t full[kVStages], adone[kVStages], empty[kVStages];
};

struct VpArgs {
  double *V;
  int64_t ldv, nv;
  const int32_t *outer, *cyc;
  int S, T, ncyc;
  int sa;
  bool second;
  const double *VpA, *VpB;
  const int64_t *rotA, *rotB;
  const int64_t *doneA;  // non-null: the step-a tasks may still be running
  const int64_t *doneB;  // non-null: the step-(a+1) tasks may still be running
  int64_t epoch;
  int vslab;             // V rows per CTA
};

// rows 0..kVRch-1 of the 32 slot columns col(k) = cb0 + k (k < 16),
// cb1 + k - 16 (k >= 16) times V' (fragments in registers); each result
// entry goes to the slot in place when keep[block] and to HBM when
// fin[block] (block = slot block of its column, 0..3)
// Addressing of one transform within a V item, set up once per item (it
// does not change from chunk to chunk): the shared-memory offsets of the 8
// A fragments, and per output tile Y the slot column and the global column
// pointer of value 0 at row g (value 1 sits 1 - 2 sw columns away), and
// whether the tile's block stays in the slot (keep) or goes to HBM (fin).
//
// Lanes with t >= 2 (sw = 1) store their two values in the opposite order
// (conflict-free 64-bit shared stores).  Their V' fragments carry the tile's
// columns 4 <-> 5 and 6 <-> 7 swapped (vp_load_bfrag), so the accumulator
// acc[j] already holds column 2t + (j ^ sw): no value select.
struct VpAddr {
  int aoff[8];
  int soff[4];
  const double *gp[4];  // at row r0 + g of the item's slab
  int dsj;
  int64_t dgj;
  bool kp[4], tg[4];
};

__device__ __forceinline__ VpAddr vp_addr(int cb0, int cb1, unsigned keep, unsigned fin,
                                          const double *V, int64_t ldv, const int64_t (&gcol)[4],
                                          int64_t r0, int g, int t) {
  VpAddr d;
  const int sw = (t >> 1) & 1;
#pragma unroll
  for (int kk = 0; kk < 8; kk++)
    d.aoff[kk] = ((kk < 4 ? cb0 + 4 * kk : cb1 + 4 * kk - 16) + t) * kVLd + g;
  d.dsj = (1 - 2 * sw) * kVLd;
  d.dgj = (1 - 2 * sw) * ldv;
#pragma unroll
  for (int Y = 0; Y < 4; Y++) {
    const int cbase = Y < 2 ? cb0 : cb1, blk = cbase >> 4;
    d.kp[Y] = (keep >> blk) & 1;
    d.tg[Y] = (fin >> blk) & 1;
    const int64_t gc = blk == 0 ? gcol[0] : blk == 1 ? gcol[1] : blk == 2 ? gcol[2] : gcol[3];
    const int n = 8 * (Y & 1) + 2 * t + sw;
    d.soff[Y] = (cbase + n) * kVLd + g;
    d.gp[Y] = V + (gc + n) * ldv + r0 + g;
  }
  return d;
}

// rows 0..kVRch-1 of a staged chunk (rows dr.. of the slab) times V'
// (fragments in registers); each result goes to the slot in place (kp) and
// / or to HBM (tg)
__device__ __forceinline__ void vp_transform(double *buf, const double (&bf)[8][4],
                                             const VpAddr &d, int64_t dr, int nr, int g) {
#pragma unroll 1
  for (int rb = 0; rb < kVRch / 8; rb += 2) {
    double a[2][8];
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int kk = 0; kk < 8; kk++) a[h][kk] = buf[d.aoff[kk] + 8 * (rb + h)];
    double acc[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int Y = 0; Y < 4; Y++) acc[h][Y][0] = acc[h][Y][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; kk++)
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int Y = 0; Y < 4; Y++) dmma(acc[h][Y][0], acc[h][Y][1], a[h][kk], bf[kk][Y]);
    const int ro = 8 * rb;
    const int64_t go = dr + ro;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const bool in = ro + 8 * h + g < nr;
#pragma unroll
      for (int Y = 0; Y < 4; Y++) {
#pragma unroll
        for (int j = 0; j < 2; j++) {
          if (d.kp[Y]) buf[d.soff[Y] + (j ? d.dsj : 0) + ro + 8 * h] = acc[h][Y][j];
          if (d.tg[Y] && in)
            st_f64(const_cast<double *>(d.gp[Y]) + (j ? d.dgj : 0) + go + 8 * h, acc[h][Y][j]);
        }
      }
    }
  }
}

// B fragments of V' (lane: row 4kk + t, column 8Y + g), with columns
// 4 <-> 5 and 6 <-> 7 of every 8-column tile swapped (see vp_transform)
__device__ __forceinline__ void vp_load_bfrag(double (&bf)[8][4], const double *Vt, int g, int t) {
  const int gs = g >= 4 ? g ^ 1 : g;
#pragma unroll
  for (int kk = 0; kk < 8; kk++)
#pragma unroll
    for (int Y = 0; Y < 4; Y++) bf[kk][Y] = Vt[(8 * Y + gs) * kVW + 4 * kk + t];
}

// one CTA: cycle c, V row slab k
__device__ __forceinline__ void vpair_cta(const VpArgs &a, int c, int k, VpSmem &S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int32_t *cy = a.cyc + ((int64_t)((a.sa + 1) % a.S) * a.ncyc + c) * 8;
  const int tk[2] = {cy[0], cy[1]}, uk[2] = {cy[2], cy[3]};
  if (a.doneA) {
    wait_flag_cta(a.doneA + tk[0], a.epoch);
    wait_flag_cta(a.doneA + tk[1], a.epoch);
  }
  if (a.second && a.doneB) {
    wait_flag_cta(a.doneB + uk[0], a.epoch);
    wait_flag_cta(a.doneB + uk[1], a.epoch);
  }
  const int32_t *pa = a.outer + ((int64_t)a.sa * a.T + tk[0]) * 2;
  const int32_t *pb = a.outer + ((int64_t)a.sa * a.T + tk[1]) * 2;
  int64_t gcol[4] = {(int64_t)pa[0] * 16, (int64_t)pa[1] * 16, (int64_t)pb[0] * 16,
                     (int64_t)pb[1] * 16};
  const bool updA[2] = {a.rotA[tk[0]] > 0, a.rotA[tk[1]] > 0};
  const bool updB[2] = {a.second && a.rotB[uk[0]] > 0, a.second && a.rotB[uk[1]] > 0};
  if (!(updA[0] || updA[1] || updB[0] || updB[1])) return;
  const int ib[2][2] = {{cy[4], cy[5]}, {cy[6], cy[7]}};
  // blocks a transform B rewrites: their transform-A values stay in the slot
  unsigned touchedB = 0;
  for (int h = 0; h < 2; h++)
    if (updB[h]) touchedB |= (1u << ib[h][0]) | (1u << ib[h][1]);
  const int64_t r0 = (int64_t)k * a.vslab, r1 = min64(r0 + a.vslab, a.nv);
  const int nchunk = (int)cdiv(r1 - r0, kVRch);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kVStages; i++) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.adone[i], 2);
      mbar_init(&S.empty[i], 2);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    // only the blocks some transform reads (late sweeps rotate few tasks)
    const unsigned need = (updA[0] ? 0x3u : 0u) | (updA[1] ? 0xCu : 0u) | touchedB;
    const uint32_t nneed = (uint32_t)__popc(need);
    for (int cc = 0; cc < nchunk; cc++) {
      const int st = cc % kVStages;
      if (cc >= kVStages) mbar_wait(&S.empty[st], (uint32_t)(((cc / kVStages) - 1) & 1));
      const int64_t r = r0 + (int64_t)cc * kVRch;
      const uint32_t bytes = (uint32_t)min64(kVRch, r1 - r) * 8u;
      if (lane == 0) mbar_expect_tx(&S.full[st], bytes * 16u * nneed);
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = lane + 32 * h;
        if ((need >> (j >> 4)) & 1u)
          bulk_g2s(&S.ring[st][j][0], a.V + (gcol[j >> 4] + (j & 15)) * a.ldv + r, bytes,
                   &S.full[st]);
      }
    }
    return;
  }
  const int role = warp - 1;  // 0, 1: transform A of t1 / t2; 2, 3: transform B of u1 / u2
  const int h = role & 1;
  const bool phaseA = role < 2;
  const bool mine = phaseA ? updA[h] : updB[h];
  double bf[8][4];
  if (mine) vp_load_bfrag(bf, (phaseA ? a.VpA + (int64_t)tk[h] * kVW * kVW
                                      : a.VpB + (int64_t)uk[h] * kVW * kVW), g, t);
  const int cb0 = phaseA ? 32 * h : 16 * ib[h][0];
  const int cb1 = phaseA ? 32 * h + 16 : 16 * ib[h][1];
  const unsigned keep = phaseA ? touchedB : 0u;
  const unsigned fin = phaseA ? (0xFu & ~touchedB) : 0xFu;
  const VpAddr d = vp_addr(cb0, cb1, keep, fin, a.V, a.ldv, gcol, r0, g, t);
  for (int cc = 0; cc < nchunk; cc++) {
    const int st = cc % kVStages;
    const uint32_t par = (uint32_t)((cc / kVStages) & 1);
    mbar_wait(phaseA ? &S.full[st] : &S.adone[st], par);
    double *buf = &S.ring[st][0][0];
    const int64_t dr = (int64_t)cc * kVRch;
    const int nr = (int)min64(kVRch, r1 - r0 - dr);
    if (mine) vp_transform(buf, bf, d, dr, nr, g);
    if (phaseA && mine && keep) fence_async_smem_cta();  // before the slot's next TMA fill
    __syncwarp();
    if (lane == 0) mbar_arrive(phaseA ? &S.adone[st] : &S.empty[st]);
  }
}

// ---- Gram of one task of the next p-step inside the update launch -----------------
//
// The K1 body (jh_tiles.cu, k_gram_tma<32, 2>) as a device function for the
// mixed launch: warp 0 streams the pair through a 3-stage TMA ring, warps 1
// and 2 own 5 lower 8x8 tiles each (one in-order DMMA chain per tile over
// the rows), warps 3 and 4 have nothing to do.  It runs after the G-update
// CTAs of the two tasks that last wrote its block-columns (per-task slab
// counters), i.e. in the tail of the update launch instead of after it.

// Increments an epoch-tagged counter ((epoch << 16) | count; a value with an
// older epoch counts as 0) and returns the new count.
__device__ __forceinline__ int tagged_inc(int64_t *p, int64_t epoch) {
  unsigned long long *c = (unsigned long long *)p;
  unsigned long long old = atomicAdd(c, 0ull);
  for (;;) {
    const unsigned long long nw = ((int64_t)(old >> 16) == epoch)
                                      ? old + 1
                                      : (((unsigned long long)epoch << 16) | 1ull);
    const unsigned long long seen = atomicCAS(c, old, nw);
    if (seen == old) return (int)(nw & 0xffff);
    old = seen;
  }
}

__device__ __forceinline__ void gram_cta32(const double *G, int64_t ldg, int64_t m, int p, int q,
                                           double *H, double *sm, uint64_t *full,
                                           uint64_t *empty) {
  // the G-item ring of the launch: kMixGStages x 32 columns x (kMixGRch + 4)
  constexpr int W = 32, NW = 4, BW = 16, MY = GramTiles<W, NW>::MY;
  constexpr int RCH = kMixGRch, LD = kMixGRch + 4, STG = kMixGStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t nchunk = cdiv(m, RCH);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STG; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp > NW) return;
  if (warp == 0) {
    fence_async_global();  // the block-columns were just written by generic stores
    for (int64_t c = 0; c < nchunk; c++) {
      const int s = (int)(c % STG);
      if (c >= STG) mbar_wait(&empty[s], (uint32_t)(((c / STG) - 1) & 1));
      const int64_t r0 = c * RCH;
      const uint32_t bytes = (uint32_t)min64(RCH, m - r0) * 8u;
      if (lane == 0) mbar_expect_tx(&full[s], bytes * W);
      __syncwarp();
      const int64_t col = lane < BW ? (int64_t)p * BW + lane : (int64_t)q * BW + (lane - BW);
      bulk_g2s(sm + ((size_t)s * W + lane) * LD, G + col * ldg + r0, bytes, &full[s]);
    }
    return;
  }
  const int cw = warp - 1;
  double acc[MY][2];
#pragma unroll
  for (int i = 0; i < MY; i++) acc[i][0] = acc[i][1] = 0.0;
  for (int64_t c = 0; c < nchunk; c++) {
    const int s = (int)(c % STG);
    mbar_wait(&full[s], (uint32_t)((c / STG) & 1));
    const double *buf = sm + (size_t)s * W * LD + (size_t)g * LD + t;
    const int nr = (int)min64(RCH, m - c * RCH);
    switch (cw) {
      case 0: gram_chunk<W, NW, 0, RCH>(buf, nr, acc, t); break;
      case 1: gram_chunk<W, NW, 1, RCH>(buf, nr, acc, t); break;
      case 2: gram_chunk<W, NW, 2, RCH>(buf, nr, acc, t); break;
      default: gram_chunk<W, NW, 3, RCH>(buf, nr, acc, t); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  switch (cw) {
    case 0: gram_store<W, NW, 0>(H, acc, g, t); break;
    case 1: gram_store<W, NW, 1>(H, acc, g, t); break;
    case 2: gram_store<W, NW, 2>(H, acc, g, t); break;
    default: gram_store<W, NW, 3>(H, acc, g, t); break;
  }
}

__global__ void k_colpos(const int32_t *__restrict__ outer, int nsteps, int T, int b,
                         int32_t *__restrict__ colpos) {
  const int64_t n = (int64_t)nsteps * T;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / T;
    const int t = (int)(i - s * T);
    colpos[s * b + outer[2 * i]] = t;
    colpos[s * b + outer[2 * i + 1]] = t;
  }
}

// ---- one launch: the G update of p-step s (per-task CTAs of the per-p-step
// kernel) and V-pair row slabs (vpair_cta), interleaved over the grid so
// that HBM-bound G slabs and DMMA-bound V slabs share the SMs

struct MixArgs {
  double *G;
  int64_t ldg, m;
  const int32_t *pairs;
  const double *Vbuf;
  const int64_t *trot;
  const int64_t *done;  // non-null: launched programmatically after the inner kernel
  int64_t epoch;
  int ntask, nslab_g, nG, gslab;
  VpArgs vp[2];
  int k0[2], kstep[2], nk[2];
  int nsrc, nV;
  int vfirst;  // V items placed before the interleaved G / V items
  // Gram items of the next p-step at the end of the grid (nGr of them)
  int nGr;
  const int32_t *pairs_next;  // pair table row of p-step s+1
  const int32_t *colpos;      // [b]: task of p-step s holding block-column c
  int64_t *gcnt;              // [ntask]: (gepoch << 16) | G slabs done
  int64_t gepoch;
  double *Hn;
};

union MixSmem {
  struct {
    double ring[kMixGStages][kVW][kMixGRch + 4];
    uint64_t full[kMixGStages], empty[kMixGStages];
  } g;
  VpSmem v;
};

#ifndef JH_MIX_MINB
#define JH_MIX_MINB 2
#endif
__global__ void __launch_bounds__(160, JH_MIX_MINB) k_update_mix(MixArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  MixSmem &S = *reinterpret_cast<MixSmem *>(smraw);
  const int N = a.nG + a.nV, bid = blockIdx.x;
  if (bid >= N) {
    // Gram of task u of the next p-step, once its two block-columns are
    // final (the G updates of the tasks holding them now, colpos, are done;
    // a queue in completion order was slower: most Grams need a late task)
    const int u = bid - N;
    const int p = a.pairs_next[2 * u], q = a.pairs_next[2 * u + 1];
    if (threadIdx.x == 0) {
      const int64_t want = (a.gepoch << 16) | a.nslab_g;
      const int src[2] = {a.colpos[p], a.colpos[q]};
      for (int k = 0; k < 2; k++)
        for (;;) {
          int64_t v;
          asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(a.gcnt + src[k])
                       : "memory");
          if (v == want) break;
          __nanosleep(64);
        }
    }
    __syncthreads();
    gram_cta32(a.G, a.ldg, a.m, p, q, a.Hn + (int64_t)u * kVW * kVW, &S.g.ring[0][0][0],
               S.g.full, S.g.empty);
    return;
  }
  // item order: the first a.vfirst CTAs are V items -- they do not wait for
  // the inner kernel, so in a programmatic launch they run beside its
  // CTAs -- then the remaining V items spread evenly among the G items
  int64_t v0, v1;
  if (bid < a.vfirst) {
    v0 = bid;
    v1 = bid + 1;
  } else {
    const int64_t b2 = bid - a.vfirst, n2 = N - a.vfirst, nv2 = a.nV - a.vfirst;
    v0 = a.vfirst + b2 * nv2 / n2;
    v1 = a.vfirst + (b2 + 1) * nv2 / n2;
  }
  if (v1 == v0) {
    const int i = bid - (int)v0;
    int task = i % a.ntask, slab = i / a.ntask;
    if (a.done) {
      // tasks in the order the inner kernel finishes them (its ready list):
      // G item i is slab i % nslab of the (i / nslab)-th finished task
      __shared__ int s_task;
      const int64_t *rl = a.done + a.ntask;
      const int k = i / a.nslab_g;
      slab = i % a.nslab_g;
      if (threadIdx.x == 0) {
        int64_t v;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(rl + 1 + k) : "memory");
          if ((v >> 24) == a.epoch) break;
          __nanosleep(64);
        }
        s_task = (int)(v & 0xffffff);
      }
      __syncthreads();
      task = s_task;
    }
    update_tma_cta<kVW, kMixGStages, kMixGRch>(a.G, a.ldg, a.m, nullptr, 0, 0, a.pairs, a.Vbuf,
                                               a.trot,
                                     a.nslab_g, a.gslab,
                        task, slab, &S.g.ring[0][0][0], S.g.full, S.g.empty);
    if (a.nGr) {
      // count this slab of the task as final (for the next p-step's Grams)
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        tagged_inc(a.gcnt + task, a.gepoch);
      }
    }
    return;
  }
  int i = (int)v0, q = 0;
  const int ncyc = a.vp[0].ncyc;
  if (a.nsrc > 1 && i >= ncyc * a.nk[0]) {
    i -= ncyc * a.nk[0];
    q = 1;
  }
  vpair_cta(a.vp[q], i % ncyc, a.k0[q] + (i / ncyc) * a.kstep[q], S.v);
}

}  // namespace

void launch_colpos(const int32_t *outer, int nsteps, int T, int b, int32_t *colpos,
                   cudaStream_t st) {
  k_colpos<<<256, 256, 0, st>>>(outer, nsteps, T, b, colpos);
}

void launch_update_mix(double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                       const double *Vbuf, const int64_t *trot, double *V, int64_t ldv,
                       int64_t nv, const int32_t *outer, const int32_t *plan, int b, int steps,
                       int nsrc, const int *sa, const bool *second, const double *const *VpA,
                       const int64_t *const *rotA, const double *const *VpB,
                       const int64_t *const *rotB, const int *k0, const int *kstep,
                       cudaStream_t st, const int64_t *done, int64_t epoch, int cur_step,
                       const int32_t *pairs_next, const int32_t *colpos, int64_t *gcnt,
                       double *Hgram) {
  MixArgs a{};
  a.done = done;
  a.epoch = epoch;
  a.G = G;
  a.ldg = ldg;
  a.m = m;
  a.pairs = pairs;
  a.Vbuf = Vbuf;
  a.trot = trot;
  a.ntask = ntask;
  const int big = ntask >= kMixBigTasks ? 1 : 0;  // a function of ntask only: the
  // flush launches (m = 0) must cut V into the same slabs as the others
  a.gslab = kMixGSlab[big];
  const int vslab = kMixVSlab[big];
  a.nslab_g = (int)cdiv(m, a.gslab);
  a.nG = ntask * a.nslab_g;
  const int nslab_v = (int)cdiv(nv, vslab);
  for (int q = 0; q < nsrc && V; q++) {
    VpArgs &v = a.vp[a.nsrc];
    v.vslab = vslab;
    v.V = V;
    v.ldv = ldv;
    v.nv = nv;
    v.outer = outer;
    v.cyc = plan;
    v.S = steps;
    v.T = b / 2;
    v.ncyc = v.T / 2;
    v.sa = sa[q];
    v.second = second[q];
    v.VpA = VpA[q];
    v.VpB = VpB[q] ? VpB[q] : VpA[q];
    v.rotA = rotA[q];
    v.rotB = rotB[q] ? rotB[q] : rotA[q];
    v.doneA = (done && sa[q] == cur_step) ? done : nullptr;
    v.doneB = (done && second[q] && sa[q] + 1 == cur_step) ? done : nullptr;
    v.epoch = epoch;
    a.k0[a.nsrc] = k0[q];
    a.kstep[a.nsrc] = kstep[q];
    a.nk[a.nsrc] = k0[q] < nslab_v ? (int)cdiv(nslab_v - k0[q], kstep[q]) : 0;
    if (a.nk[a.nsrc] == 0) continue;
    a.nV += v.ncyc * a.nk[a.nsrc];
    a.nsrc++;
  }
  if (pairs_next && m > 0) {
    static std::atomic<int64_t> gepoch{0};
    a.nGr = ntask;
    a.pairs_next = pairs_next;
    a.colpos = colpos;
    a.gcnt = gcnt;
    a.gepoch = ++gepoch;
    a.Hn = Hgram;
  }
  if (a.nG + a.nV + a.nGr == 0) return;
#ifndef JH_VFIRST_PCT
#define JH_VFIRST_PCT 0
#endif
  a.vfirst = kMixVOrder == 1 ? a.nV : (done ? (int)((int64_t)a.nV * JH_VFIRST_PCT / 100) : 0);
  const size_t smem = sizeof(MixSmem);
  ensure_smem((const void *)k_update_mix, (int)smem);
  if (!done) {
    k_update_mix<<<a.nG + a.nV + a.nGr, 160, smem, st>>>(a);
    return;
  }
  // programmatic dependent launch: may start while the inner kernel runs
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(a.nG + a.nV + a.nGr);
  cfg.blockDim = dim3(160);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_update_mix, a);
}

}  // namespace jh
