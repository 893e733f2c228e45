// DMMA-tiled, bitwise-exact Gram and post-multiply kernels of the p-step
// (the streaming, HBM-bound part of the hot path).
//
//   K1  k_gram_tma<W>     H = [Gp Gq]^T [Gp Gq]       (blockkernel.py:76-107)
//   K3  k_update_dmma<W>  [Gp Gq] <- [Gp Gq] V'       (blockkernel.py:407-428)
//                          and [Vp Vq] <- [Vp Vq] V'  (driver.py:165-173)
//
// Exactness: every output entry is one chain of DMMA k-steps in ascending k,
// each DMMA being four in-order fmas (see jh_dmma.cuh), from +0.0 -- the
// reference's per-entry fma chain.  Rows past the end of a column are fed as
// zeros: fma(0, x, acc) leaves any accumulator that started at +0.0 unchanged
// (finite data; such a chain never holds -0.0), so padding is bit-neutral.
#include "jh_gram.cuh"
#include "jh_kernels.h"
#include "jh_update.cuh"

#include <cstdlib>

namespace jh {

// ---------------------------------------------------------------------------
// K1: Gram matrix of one block-column pair per CTA (one warp).
//
// Row chunks of the pair (64 rows x W columns) stream into a 3-stage shared
// memory ring through the TMA engine (cp.async.bulk, one 512 B copy per
// column, completion on an mbarrier).  Columns are stored with a padded
// stride of 68 doubles so that the DMMA fragment loads (lane = (column
// 8X + g, row 4kk + t)) are bank-conflict free.  The warp owns all
// (W/8)(W/8+1)/2 lower 8x8 tiles; per k-step it loads W/8 fragments (one
// LDS.64 each) and issues one DMMA per tile: fragment X serves as the A
// operand (A^T rows) and the B operand alike.

// Consumer warp cw of CTA part `part` (of SPLIT CTAs per task) acts as warp
// vw = cw + NW * part of NW * SPLIT virtual warps: it owns the tiles
// i == vw (mod NW * SPLIT).  SPLIT > 1 spreads one task's tile chains over
// several SMs (few tasks per p-step: the sharded solve), each CTA streaming
// the whole pair (the second read of a chunk is an L2 hit).
template <int W, int VW, int RCH, int LD>
__device__ __forceinline__ void gram_chunk_dispatch(int vw, const double *buf, int nr,
                                                    double (&acc)[GramTiles<W, VW>::MY][2],
                                                    int t) {
  switch (vw) {
#define JH_GC(k) \
  case k:        \
    if constexpr (k < VW) gram_chunk<W, VW, (k < VW ? k : 0), RCH, LD>(buf, nr, acc, t); \
    break;
    JH_GC(0) JH_GC(1) JH_GC(2) JH_GC(3) JH_GC(4) JH_GC(5) JH_GC(6) JH_GC(7) JH_GC(8) JH_GC(9)
#undef JH_GC
    default: break;
  }
}

template <int W, int VW>
__device__ __forceinline__ void gram_store_dispatch(int vw, double *H,
                                                    const double (&acc)[GramTiles<W, VW>::MY][2],
                                                    int g, int t) {
  switch (vw) {
#define JH_GS(k) \
  case k:        \
    if constexpr (k < VW) gram_store<W, VW, (k < VW ? k : 0)>(H, acc, g, t); \
    break;
    JH_GS(0) JH_GS(1) JH_GS(2) JH_GS(3) JH_GS(4) JH_GS(5) JH_GS(6) JH_GS(7) JH_GS(8) JH_GS(9)
#undef JH_GS
    default: break;
  }
}

// The producer loads each chunk as two TMA tensor tiles (rows x W/2 columns
// of block p and of block q, `tmap` over G) into a dense [W][kGramRch]
// stage; kGramRch = 4 (mod 16) keeps the fragment loads conflict free.
// Rows past m arrive as zeros (the consumers stop at m anyway).  Without a
// tensor map (use_tmap false) one bulk copy per column, padded stride.
template <int W, int NW, int kGramRch, int kGramStages, int SPLIT = 1>
__global__ void __launch_bounds__(32 * (NW + 1))
k_gram_tma(const double *__restrict__ G, int64_t ldg, int64_t m,
           const int32_t *__restrict__ pairs, double *__restrict__ Hbuf,
           const __grid_constant__ CUtensorMap tmap, bool use_tmap) {
  // warp 0 produces (TMA), warps 1..NW consume (DMMA)
  static_assert(kGramRch % 16 == 4, "dense tensor-tile stage: column stride 4 (mod 16)");
  constexpr int BW = W / 2, VW = NW * SPLIT, MY = GramTiles<W, VW>::MY, kGramLd = kGramRch;
  static_assert(VW <= 10, "at most one virtual warp per tile of w = 32");
  extern __shared__ __align__(128) double sm[];  // [kGramStages][W][kGramLd]
  __shared__ __align__(8) uint64_t full[kGramStages], empty[kGramStages];
  const int task = blockIdx.x / SPLIT, part = blockIdx.x % SPLIT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int p = pairs[2 * task], q = pairs[2 * task + 1];
  const int64_t nchunk = cdiv(m, kGramRch);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGramStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    for (int64_t c = 0; c < nchunk; c++) {
      const int s = (int)(c % kGramStages);
      if (c >= kGramStages) mbar_wait(&empty[s], (uint32_t)(((c / kGramStages) - 1) & 1));
      const int64_t r0 = c * kGramRch;
      if (use_tmap) {
        if (lane == 0) {
          mbar_expect_tx(&full[s], (uint32_t)(W * kGramRch * 8));  // whole boxes
          tma_load_2d(sm + (size_t)s * W * kGramLd, &tmap, (int)r0, p * BW, &full[s]);
          tma_load_2d(sm + ((size_t)s * W + BW) * kGramLd, &tmap, (int)r0, q * BW, &full[s]);
        }
        continue;
      }
      const uint32_t bytes = (uint32_t)min64(kGramRch, m - r0) * 8u;
      if (lane == 0) mbar_expect_tx(&full[s], bytes * W);
      __syncwarp();
      for (int j = lane; j < W; j += 32) {
        const int64_t col = j < BW ? (int64_t)p * BW + j : (int64_t)q * BW + (j - BW);
        bulk_g2s(sm + ((size_t)s * W + j) * kGramLd, G + col * ldg + r0, bytes, &full[s]);
      }
    }
    return;
  }
  const int vw = (warp - 1) + NW * part;
  double acc[MY][2];
#pragma unroll
  for (int i = 0; i < MY; i++) acc[i][0] = acc[i][1] = 0.0;

  for (int64_t c = 0; c < nchunk; c++) {
    const int s = (int)(c % kGramStages);
    mbar_wait(&full[s], (uint32_t)((c / kGramStages) & 1));
    const double *buf = sm + (size_t)s * W * kGramLd + (size_t)g * kGramLd + t;
    const int nr = (int)min64(kGramRch, m - c * kGramRch);
    gram_chunk_dispatch<W, VW, kGramRch, kGramLd>(vw, buf, nr, acc, t);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  double *H = Hbuf + (size_t)task * W * W;  // column-major: H[y * W + x] = h[x][y]
  gram_store_dispatch<W, VW>(vw, H, acc, g, t);
}

// ---------------------------------------------------------------------------
// K3: in-place post-multiplication of the pair columns of G (rows < m) and V
// (rows < nv) by the task's V' (W x W).  A CTA of 8 warps owns a slab of
// 8 * kUpdRpw rows of one matrix for one task; V' sits in shared memory in
// fragment order (conflict-free LDS.64 of the DMMA B operand).  Each warp
// streams 8-row blocks: W/4 A fragments (LDG.64, rows r0+g, columns 4kk+t),
// W/4 x W/8 DMMAs and W/4 STG.64 of the result (rows r0+g, columns 8Y+2t+j:
// every 32 B sector is written whole).  Loads run two blocks ahead.  Every
// row is read completely before it is written, by the same warp.

constexpr int kUpdWarps = 8;
constexpr int kUpdRpw = 256;  // rows per warp

template <int W>
__global__ void __launch_bounds__(32 * kUpdWarps, W == 64 ? 2 : 1)
k_update_dmma(double *__restrict__ G, int64_t ldg, int64_t m, double *__restrict__ V,
              int64_t ldv, int64_t nv, const int32_t *__restrict__ pairs,
              const double *__restrict__ Vbuf, const int64_t *__restrict__ trot, int nslab_g) {
  constexpr int NT = W / 8, NK = W / 4, BW = W / 2;
  __shared__ double vfrag[NK * NT * 32];
  const int task = blockIdx.x;
  if (trot[task] == 0) return;
  const int p = pairs[2 * task], q = pairs[2 * task + 1];
  double *A;
  int64_t ld, rows, slab0;
  if ((int)blockIdx.y < nslab_g) {
    A = G; ld = ldg; rows = m; slab0 = (int64_t)blockIdx.y * kUpdWarps * kUpdRpw;
  } else {
    A = V; ld = ldv; rows = nv; slab0 = (int64_t)(blockIdx.y - nslab_g) * kUpdWarps * kUpdRpw;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  // V' fragments: B[k][n] = v'[4kk + t][8Y + g]; Vbuf is column-major (v'[k][n] at n*W + k)
  const double *Vt = Vbuf + (size_t)task * W * W;
  for (int e = threadIdx.x; e < NK * NT * 32; e += blockDim.x) {
    const int l = e & 31, f = e >> 5, kk = f / NT, Y = f % NT;
    vfrag[e] = Vt[(8 * Y + (l >> 2)) * W + 4 * kk + (l & 3)];
  }
  __syncthreads();
  const int64_t r_begin = slab0 + (int64_t)warp * kUpdRpw;
  if (r_begin >= rows) return;
  const int64_t r_end = min64(r_begin + kUpdRpw, rows);

  // column c of the pair: block p for c < BW, block q otherwise
  const double *pin = A + ((int64_t)p * BW + t) * ld;
  const double *qin = A + ((int64_t)q * BW + t) * ld;
  double *pout = A + ((int64_t)p * BW + 2 * t) * ld;
  double *qout = A + ((int64_t)q * BW + 2 * t) * ld;
  auto ain = [&](int kk) -> const double * {
    return kk < NK / 2 ? pin + (int64_t)(4 * kk) * ld : qin + (int64_t)(4 * kk - BW) * ld;
  };
  auto aout = [&](int Y, int j) -> double * {
    return Y < NT / 2 ? pout + (int64_t)(8 * Y + j) * ld : qout + (int64_t)(8 * Y + j - BW) * ld;
  };
  auto load_block = [&](int64_t r0, double (&f)[NK]) {
    const int64_t row = r0 + g;
    const bool ok = row < r_end;
#pragma unroll
    for (int kk = 0; kk < NK; kk++) f[kk] = ok ? ld_f64(ain(kk) + row) : 0.0;
  };
  auto compute_store = [&](int64_t r0, const double (&f)[NK]) {
    double acc[NT][2];
#pragma unroll
    for (int Y = 0; Y < NT; Y++) acc[Y][0] = acc[Y][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < NK; kk++)
#pragma unroll
      for (int Y = 0; Y < NT; Y++)
        dmma(acc[Y][0], acc[Y][1], f[kk], vfrag[(kk * NT + Y) * 32 + lane]);
    const int64_t row = r0 + g;
    if (row < r_end) {
#pragma unroll
      for (int Y = 0; Y < NT; Y++)
#pragma unroll
        for (int j = 0; j < 2; j++) st_f64(aout(Y, j) + row, acc[Y][j]);
    }
  };
  if constexpr (W == 64) {
    // (B fragments re-read from shared memory per use: kept loop-invariant,
    // all 128 of them would not fit in registers)
    auto lds_f64 = [](const double *a) {
      double v;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(a)));
      return v;
    };
    // 16 A fragments per 8-row block; the 8 output tiles in two halves of
    // 4 accumulators; column addresses formed on the fly (no per-column
    // pointer registers); latency hidden by the 16 warps per SM -- no spills
    const double *pb = A + (int64_t)p * BW * ld, *qb = A + (int64_t)q * BW * ld;
    // the stride is re-read through an opaque move per use, so the compiler
    // does not hoist 64 per-column pointers out of the row loop (spills)
    auto col = [&](int c) -> double * {
      int64_t l;
      asm volatile("mov.b64 %0, %1;" : "=l"(l) : "l"(ld));
      return const_cast<double *>(c < BW ? pb + (int64_t)c * l : qb + (int64_t)(c - BW) * l);
    };
    auto load64 = [&](int64_t r0, double (&f)[NK]) {
      const int64_t row = r0 + g;
      const bool ok = row < r_end;
#pragma unroll
      for (int kk = 0; kk < NK; kk++) f[kk] = ok ? __ldcs(col(4 * kk + t) + row) : 0.0;
    };
    auto half = [&](int64_t r0, const double (&f)[NK], int y0) {
      double acc[4][2];
#pragma unroll
      for (int Y = 0; Y < 4; Y++) acc[Y][0] = acc[Y][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        double b[4];
#pragma unroll
        for (int Y = 0; Y < 4; Y++) b[Y] = lds_f64(&vfrag[(kk * NT + y0 + Y) * 32 + lane]);
#pragma unroll
        for (int Y = 0; Y < 4; Y++)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[Y][0]), "+d"(acc[Y][1]) : "d"(f[kk]), "d"(b[Y]));
      }
      const int64_t row = r0 + g;
      if (row < r_end) {
#pragma unroll
        for (int Y = 0; Y < 4; Y++)
#pragma unroll
          for (int j = 0; j < 2; j++) st_f64(col(8 * (y0 + Y) + 2 * t + j) + row, acc[Y][j]);
      }
    };
    double fa[NK];
#pragma unroll 1
    for (int64_t r0 = r_begin; r0 < r_end; r0 += 8) {
      load64(r0, fa);
#pragma unroll 1
      for (int h = 0; h < 2; h++) half(r0, fa, 4 * h);
    }
  } else {
  double f0[NK], f1[NK], f2[NK];
  load_block(r_begin, f0);
  load_block(r_begin + 8, f1);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += 24) {
    load_block(r0 + 16, f2);
    compute_store(r0, f0);
    if (r0 + 8 >= r_end) break;
    load_block(r0 + 24, f0);
    compute_store(r0 + 8, f1);
    if (r0 + 16 >= r_end) break;
    load_block(r0 + 32, f1);
    compute_store(r0 + 16, f2);
  }
  }
}

// K3 (TMA variant): the same post-multiplication with the pair rows streamed
// through a 4-stage shared-memory ring by the TMA engine, so the bytes in
// flight do not cost registers.  Warp 0 produces (one 512 B bulk copy per
// column and chunk of 64 rows); warps 1..4 consume 16 rows each per chunk
// (two 8-row DMMA blocks, A fragments by conflict-free LDS.64 from the
// padded ring, V' fragments in registers) and store the results straight to
// global memory (whole 32 B sectors).  A CTA owns a slab of kUpdSlab rows of
// one matrix for one task.

// ---------------------------------------------------------------------------
// host launchers

bool gram_tma_ok(int w, int64_t m, int64_t ldg) {
  return (w == 16 || w == 32 || w == 64) && m % 2 == 0 && ldg % 2 == 0;
}

// consumer warps per Gram CTA: 2 (tiles 5 + 5 for w = 32), or 4 when few
// tasks meet long columns (tall factors: one CTA per task leaves SMs short
// of DMMA warps while every tile is a chain over all m rows)
template <int W, int NW, int RCH, int STG, int SPLIT = 1>
static void launch_gram_nw(const double *G, int64_t ldg, int64_t m, const int32_t *pairs,
                           int ntask, double *Hbuf, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)STG * W * RCH;
  ensure_smem((const void *)k_gram_tma<W, NW, RCH, STG, SPLIT>, (int)smem);
  // the table's block-columns span ntask * W columns of G
  CUtensorMap tmap;
  const bool ok = make_col_tmap(&tmap, G, m, (int64_t)ntask * W, ldg, RCH, W / 2);
  k_gram_tma<W, NW, RCH, STG, SPLIT><<<ntask * SPLIT, 32 * (NW + 1), smem, st>>>(
      G, ldg, m, pairs, Hbuf, tmap, ok);
}

// Ring shape by the CTAs an SM must hold for one wave: longer chunks (one
// bulk copy of 8 * rows bytes per column) pay while the ring still fits
// (w = 32: 192 rows x 2 stages = 100 KB up to 2 CTAs per SM, 128 x 2 up
// to 3, 104 x 2 = 55 KB up to 4).  K1 us per launch, 64 x 3 before:
// n = 16384 390.5 -> 376.4, 131072 x 8192 2079 -> 1766, n = 4096 72 -> 61.
template <int W, int NW>
static void launch_gram_shape(const double *G, int64_t ldg, int64_t m, const int32_t *pairs,
                              int ntask, int sms, double *Hbuf, cudaStream_t st) {
  const int per_sm = (ntask + sms - 1) / sms;
  if (per_sm <= 2)
    launch_gram_nw<W, NW, 196, 2>(G, ldg, m, pairs, ntask, Hbuf, st);
  else if (per_sm == 3)
    launch_gram_nw<W, NW, 132, 2>(G, ldg, m, pairs, ntask, Hbuf, st);
  else
    launch_gram_nw<W, NW, 100, 2>(G, ldg, m, pairs, ntask, Hbuf, st);
}

template <int W>
static void launch_gram_t(const double *G, int64_t ldg, int64_t m, const int32_t *pairs,
                          int ntask, double *Hbuf, cudaStream_t st) {
  // Few tasks per p-step (the sharded solve) leave the Gram latency-bound:
  // every tile is one chain over all m rows.  Up to half an SM per task, two
  // CTAs of 5 consumer warps split a task's 10 tiles (one chain per warp);
  // up to one SM per task, one CTA of 10 (profiles/r02/README.md: Gram per
  // p-step at 64 tasks 0.187 -> 0.118 ms, at 128 tasks 0.188 -> 0.144 ms).
#ifndef JH_GS2_DIV
#define JH_GS2_DIV 2
#endif
#ifndef JH_G10_MUL
#define JH_G10_MUL 1
#endif
  const int sms = sm_count();
  if constexpr (W == 32) {
    if (ntask <= sms / JH_GS2_DIV) {
      launch_gram_nw<W, 5, 196, 2, 2>(G, ldg, m, pairs, ntask, Hbuf, st);
      return;
    }
    if (ntask <= sms * JH_G10_MUL) {
      launch_gram_nw<W, 10, 196, 2, 1>(G, ldg, m, pairs, ntask, Hbuf, st);
      return;
    }
  }
  if (ntask < 3 * sms)
    launch_gram_shape<W, 4>(G, ldg, m, pairs, ntask, sms, Hbuf, st);
  else
    launch_gram_shape<W, 2>(G, ldg, m, pairs, ntask, sms, Hbuf, st);
}

void launch_gram_tma(const double *G, int64_t ldg, int64_t m, const int32_t *pairs, int ntask,
                     int w, double *Hbuf, cudaStream_t st) {
  if (w == 16)
    launch_gram_t<16>(G, ldg, m, pairs, ntask, Hbuf, st);
  else if (w == 32)
    launch_gram_t<32>(G, ldg, m, pairs, ntask, Hbuf, st);
  else  // w = 64: 36 lower tiles over 4 consumer warps (9 chains each), 3 x 64-row ring (104 KB)
    launch_gram_nw<64, 4, 68, 3>(G, ldg, m, pairs, ntask, Hbuf, st);
}

bool update_dmma_ok(int w) { return w == 16 || w == 32 || w == 64; }

template <int W>
static void launch_update_tma_t(double *G, int64_t ldg, int64_t m, double *V, int64_t ldv,
                                int64_t nv, const int32_t *pairs, int ntask, const double *Vbuf,
                                const int64_t *trot, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)kE0Stages * W * (kE0Rch + 4);
  ensure_smem((const void *)k_update_tma<W>, (int)smem);
  const int nsg = (int)cdiv(m, kUpdSlab);
  const int nsv = V ? (int)cdiv(nv, kUpdSlab) : 0;
  dim3 grid(ntask, nsg + nsv);
  k_update_tma<W><<<grid, 32 * (kUpdCons + 1), smem, st>>>(G, ldg, m, V, ldv, nv, pairs, Vbuf,
                                                          trot, nsg);
}

void launch_update_dmma(double *G, int64_t ldg, int64_t m, double *V, int64_t ldv, int64_t nv,
                        const int32_t *pairs, int ntask, int w, const double *Vbuf,
                        const int64_t *trot, cudaStream_t st) {
  // the TMA ring needs 16-byte aligned columns; the LDG variant takes the rest
  // (w = 64: the V' fragments of a warp would not fit in registers -- the LDG
  // variant keeps them in shared memory)
  const bool tma = w != 64 && m % 2 == 0 && ldg % 2 == 0 &&
                   (!V || (nv % 2 == 0 && ldv % 2 == 0));
  if (tma) {
    if (w == 16)
      launch_update_tma_t<16>(G, ldg, m, V, ldv, nv, pairs, ntask, Vbuf, trot, st);
    else
      launch_update_tma_t<32>(G, ldg, m, V, ldv, nv, pairs, ntask, Vbuf, trot, st);
    return;
  }
  const int64_t slab = (int64_t)kUpdWarps * kUpdRpw;
  const int nsg = (int)cdiv(m, slab);
  const int nsv = V ? (int)cdiv(nv, slab) : 0;
  dim3 grid(ntask, nsg + nsv);
  if (w == 16)
    k_update_dmma<16><<<grid, 32 * kUpdWarps, 0, st>>>(G, ldg, m, V, ldv, nv, pairs, Vbuf, trot,
                                                        nsg);
  else if (w == 32)
    k_update_dmma<32><<<grid, 32 * kUpdWarps, 0, st>>>(G, ldg, m, V, ldv, nv, pairs, Vbuf, trot,
                                                        nsg);
  else
    k_update_dmma<64><<<grid, 32 * kUpdWarps, 0, st>>>(G, ldg, m, V, ldv, nv, pairs, Vbuf, trot,
                                                        nsg);
}

}  // namespace jh
