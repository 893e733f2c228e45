// Cycle engine: a block sweep as one persistent dataflow kernel in which the
// post-multiplication of p-step s-1 and the Gram formation of p-step s are a
// single streaming pass over the G block-columns, and the V updates of two
// consecutive p-steps are a single pass over V.
//
// Structure it relies on (checked on the host by cycle_plan): the union of
// the pairings of two consecutive p-steps is a set of 4-cycles.  For the
// reversed row-closest strategy ("rrow", the Mantharam-Eberlein equivalent,
// SURVEY.md section 8) this holds for every step pair, including the wrap from
// the last step of a sweep to the first.  A cycle c of boundary s joins tasks
// t1 = (p1, q1), t2 = (p2, q2) of p-step s-1 with tasks u1, u2 of p-step s,
// each u taking one block-column from t1 and one from t2.  Work items:
//   B(s, c)   one 2-CTA cluster.  Both CTAs receive the four block-columns
//             [p1 q1 p2 q2] (64 columns of G) chunk by chunk through TMA
//             multicast (each CTA loads half and broadcasts it).  CTA r
//             computes the two block-columns of u_r from their p-step s-1
//             pairs (post-multiplication, reference blockkernel.py:407-428,
//             skipped for a task that did not rotate, driver.py:165), stores
//             them, and accumulates u_r's Gram matrix (blockkernel.py:76-107)
//             from the updated rows in shared memory -- G is read once per
//             p-step.  Then the same CTA runs the Cholesky + inner Jacobi of
//             u_r (blockkernel.py:110-145, 278-400; the v5 device code).
//   V(j, c, k) row slab k of the four V block-columns of cycle c of the step
//             pair (a, a+1), a = s_begin + 2j, halves per CTA: the step-a
//             transforms, then the step-(a+1) transforms, in one pass (V is
//             read by nothing else until the sweep ends).
// Dependencies: B(s, c) after the inner Jacobi of t1 and t2 (which ran after
// the B items that wrote their columns); V(j, c, *) after the inner Jacobi of
// its four tasks and after every V item of pair j-1 (a barrier per pair).
// Two queues: B items first, V items fill what the critical path leaves.
// Per entry every fma chain runs in the reference's order (a Gram entry over
// rows 0..m-1 in one CTA; an update entry over k per row), so results are
// bitwise those of the per-p-step kernels and of the reference.
//
// CTA: warp 0 = TMA producer, warps 1..4 = DMMA consumers; results go back
// to HBM with cp.async.bulk stores from the ring slot.  Two CTAs per SM.
#include "jh_gram.cuh"
#include "jh_inner5.cuh"
#include "jh_kernels.h"

#include <cstdlib>
#include <vector>

namespace jh {

constexpr int kCyW = 32;              // block width (shortened order)
constexpr int kCyThreads = 128;       // 4 DMMA warps; warp 0 also issues the TMA loads
constexpr int kCyStages = 4;          // B ring (multicast)
constexpr int kBR = 48;               // rows per B chunk
constexpr int kBLd = kBR + 4;         // padded slot column stride (== 4 mod 16: conflict-free)
constexpr int kCyVStages = 2;         // V ring (local) + the four V'
constexpr int kCyCols = 64;           // four block-columns of 16
constexpr int kCyVpLd = kCyW + 4;     // padded V' column stride (conflict-free B loads)
constexpr int kCyQCap = 1 << 18;      // queue slots (per queue)
constexpr int64_t kCyVSlab = 2048;    // rows of V per V item (a cluster)

enum CyItem : int { kCyB = 0, kCyV = 2 };

__host__ __device__ inline long long cy_pack(int type, int a, int c, int k) {
  return ((long long)type << 60) | ((long long)a << 40) | ((long long)c << 16) | (long long)k;
}

// two FIFO queues: 0 = critical path (B items), 1 = V items
struct CySched {
  unsigned long long head[2], tail[2], done;
};

struct CyArgs {
  double *G;
  int64_t ldg, m;
  double *V;
  int64_t ldv, nv;
  const int32_t *outer;  // [S][T][2] block-column pairs
  const int32_t *cyc;    // [S][ncyc][8]: t1 t2 u1 u2 iu1 ju1 iu2 ju2 (boundary s)
  const int32_t *tpos;   // [S][T]: 2 c + side of task (s, t) at boundary s + 1
  const int32_t *upos;   // [S][T]: 2 c + side of task (s, u) at boundary s
  const int32_t *inner;
  int64_t n_plus;
  int inner_limit;
  double tol_c;
  unsigned long long *counters;
  int S, T, ncyc, s_begin, nsteps, npairs, nslab_v;
  unsigned long long total;
  double *H, *Vp;   // [nsteps][T][W*W]
  int64_t *rot;     // [nsteps][T]
  int *bready;      // [nsteps + 1][ncyc]
  int *vready;      // [npairs][ncyc]
  int *vdone;       // [npairs]
  CySched *sched;
  long long *qitem, *qseq;  // [2][kCyQCap]
  long long *trace;         // optional: [0] = count, then {item, smid, t0, t1}
  long long trace_cap;
};

struct CySmem {
  union {
    double ring[kCyStages][kCyCols][kBLd]; // B items
    struct {
      double ring[kCyVStages][kCyCols][kLd];
      double vp[4][kCyW][kCyVpLd];         // V' of t1, t2, u1, u2 (column-major)
    } v;                                   // V items
    InnerSmem5<kCyW> inner;                // inner Jacobi after a B item
  } u;
  uint64_t full[kCyStages], empty[kCyStages];     // B ring (empty: 4 local + 4 peer warps)
  uint64_t updb[kCyStages];                       // B ring: chunk updated by the 4 warps
  uint64_t vfull[kCyVStages], vempty[kCyVStages]; // V ring
  long long item;
  unsigned chunk, vchunk;  // chunks streamed so far (ring phases)
  int last;
};

// ---- PTX helpers ---------------------------------------------------------------

__device__ __forceinline__ long long cy_ld_acquire(const long long *p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long cy_ld_acquire_u(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cy_st_release(long long *p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void compute_bar() {
  asm volatile("bar.sync 1, 128;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_map(const void *p, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// arrive on the peer CTA's mbarrier (default .release.cta semantics, as
// CUTLASS's ClusterBarrier::arrive(cta_id); the slot reads it releases have
// completed -- their values were consumed by earlier DMMAs)
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy delivered to the same offset in both CTAs of
// the cluster, completing on each CTA's mbarrier at `bar`'s offset
__device__ __forceinline__ void bulk_g2s_mc(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ unsigned long long cy_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- queues --------------------------------------------------------------------

__device__ void cy_push(const CyArgs &a, int q, const long long *items, int cnt) {
  const unsigned long long j0 = atomicAdd(&a.sched->tail[q], (unsigned long long)cnt);
  long long *qi = a.qitem + (size_t)q * kCyQCap, *qs = a.qseq + (size_t)q * kCyQCap;
  for (int i = 0; i < cnt; i++) {
    const unsigned long long j = j0 + i;
    const size_t slot = j & (kCyQCap - 1);
    qi[slot] = items[i];
    __threadfence();
    cy_st_release(&qs[slot], (long long)j);
  }
}

// push the nslab_v row slabs of V item (j, c)
__device__ void cy_push_vslabs(const CyArgs &a, int j, int c) {
  long long items[16];
  for (int k0 = 0; k0 < a.nslab_v; k0 += 16) {
    const int cnt = a.nslab_v - k0 < 16 ? a.nslab_v - k0 : 16;
    for (int i = 0; i < cnt; i++) items[i] = cy_pack(kCyV, j, c, k0 + i);
    cy_push(a, 1, items, cnt);
  }
}

// next item (critical-path queue first); -1 once all work is done
__device__ long long cy_pop(const CyArgs &a) {
  for (;;) {
    for (int q = 0; q < 2; q++) {
      unsigned long long h = cy_ld_acquire_u(&a.sched->head[q]);
      const unsigned long long t = cy_ld_acquire_u(&a.sched->tail[q]);
      while (h < t) {
        const unsigned long long old = atomicCAS(&a.sched->head[q], h, h + 1);
        if (old == h) {
          const size_t slot = h & (kCyQCap - 1);
          const long long *qs = a.qseq + (size_t)q * kCyQCap;
          while (cy_ld_acquire(&qs[slot]) != (long long)h) __nanosleep(20);
          return __ldcg(a.qitem + (size_t)q * kCyQCap + slot);
        }
        h = old;
      }
    }
    if (cy_ld_acquire_u(&a.sched->done) >= a.total) return -1;
    __nanosleep(32);
  }
}

__device__ __forceinline__ int cy_vtarget(const CyArgs &a, int j) {
  return (2 * j + 1 < a.nsteps ? 4 : 2) + 1;
}

__device__ __forceinline__ const int32_t *cy_cycle(const CyArgs &a, int s, int c) {
  return a.cyc + ((int64_t)(s % a.S) * a.ncyc + c) * 8;
}
__device__ __forceinline__ const int32_t *cy_pair(const CyArgs &a, int s, int t) {
  return a.outer + ((int64_t)(s % a.S) * a.T + t) * 2;
}

// ---- B items: update (s-1) + Gram (s) of one cycle, 2-CTA cluster -------------------

struct CyB {
  int blk[4];          // block-columns in slot order [p1 q1 p2 q2]
  bool upd[2];         // t1 / t2 rotated at p-step s-1
  const double *VA[2]; // their V'
  int ob[2];           // slot blocks of this CTA's u (first, second column block)
  bool gram;
  double *H;           // Gram of this CTA's u
};

// post-multiply rows row0..row0+23 (3 row tiles) of the output block at slot
// columns ocol..ocol+15 from the 32 slot columns icol.. of its p-step s-1
// pair; results go in place into the slot (for the Gram) and straight from
// the accumulators to HBM (out = the block's first column in G at this
// chunk's first row; nr valid rows).  B fragments (the block's 16 columns of
// V') in registers.  Per output entry the DMMA chain runs over k ascending
// (blockkernel.py:407-418).  Lanes with t >= 2 store their two columns in
// the opposite order, which makes the 64-bit shared stores conflict-free.
__device__ __forceinline__ void cy_update_block(double *buf, int row0, int icol, int ocol,
                                                const double (&bf)[8][2], double *out,
                                                int64_t ld, int nr, int g, int t) {
  const int sw = (t >> 1) & 1;
  double *o0 = out + (2 * t + sw) * ld, *o1 = out + (2 * t + 1 - sw) * ld;
  const int64_t l8 = 8 * ld;
#pragma unroll 1
  for (int rt = 0; rt < 3; rt++) {
    const int row = row0 + 8 * rt + g;
    double acc[2][2];
    acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.0;
    const double *col = buf + (icol + t) * kBLd + row;
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
      const double av = col[4 * kk * kBLd];
      dmma(acc[0][0], acc[0][1], av, bf[kk][0]);
      dmma(acc[1][0], acc[1][1], av, bf[kk][1]);
    }
    const double v00 = sw ? acc[0][1] : acc[0][0], v01 = sw ? acc[0][0] : acc[0][1];
    const double v10 = sw ? acc[1][1] : acc[1][0], v11 = sw ? acc[1][0] : acc[1][1];
    double *ob = buf + (ocol + 2 * t + sw) * kBLd + row;
    const int d = (1 - 2 * sw) * kBLd;  // to the other column of the pair
    ob[0] = v00;
    ob[d] = v01;
    ob[8 * kBLd] = v10;
    ob[8 * kBLd + d] = v11;
    if (row < nr) {
      st_f64(o0 + row, v00);
      st_f64(o1 + row, v01);
      st_f64(o0 + l8 + row, v10);
      st_f64(o1 + l8 + row, v11);
    }
  }
}

// Gram tiles of compute warp CW: tiles CW, CW+4, CW+8 of the 10 lower 8x8
// tiles (X, Y), Y <= X, enumerated row-major; column tile X of the task sits
// at slot column cb[X].  One in-order DMMA chain per tile over the rows.
template <int CW>
struct CyTiles {
  static constexpr int N = CW < 2 ? 3 : 2;
  __device__ static constexpr int X(int i) {
    constexpr int xs[10] = {0, 1, 1, 2, 2, 2, 3, 3, 3, 3};
    return xs[CW + 4 * i];
  }
  __device__ static constexpr int Y(int i) {
    constexpr int ys[10] = {0, 0, 1, 0, 1, 2, 0, 1, 2, 3};
    return ys[CW + 4 * i];
  }
};

template <int CW>
__device__ __forceinline__ void cy_gram_chunk(const double *buf, int nr, const int (&cb)[4],
                                              double (&acc)[3][2], int g, int t) {
  using TL = CyTiles<CW>;
  const double *c[4];
#pragma unroll
  for (int X = 0; X < 4; X++) c[X] = buf + (cb[X] + g) * kBLd + t;
  auto step = [&](int kk, bool ok) {
    double f[4];
#pragma unroll
    for (int X = 0; X < 4; X++) f[X] = ok ? c[X][4 * kk] : 0.0;
#pragma unroll
    for (int i = 0; i < TL::N; i++) dmma(acc[i][0], acc[i][1], f[TL::X(i)], f[TL::Y(i)]);
  };
  if (nr == kBR) {
#pragma unroll 2
    for (int kk = 0; kk < kBR / 4; kk++) step(kk, true);
  } else {
    const int nks = (nr + 3) / 4;
    for (int kk = 0; kk < nks; kk++) step(kk, 4 * kk + t < nr);
  }
}

template <int CW>
__device__ __forceinline__ void cy_gram_store(double *H, const double (&acc)[3][2], int g, int t) {
  using TL = CyTiles<CW>;
#pragma unroll
  for (int i = 0; i < TL::N; i++) {
    const int X = TL::X(i), Y = TL::Y(i);
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const int x = 8 * X + g, y = 8 * Y + 2 * t + j;
      H[y * kCyW + x] = acc[i][j];
      if (X != Y) H[x * kCyW + y] = acc[i][j];
    }
  }
}

// warp 0: issue chunk c of a B item (this CTA's half of the 64 columns,
// multicast to both CTAs) once the slot's previous chunk was released by all
// eight compute warps of the cluster.  Multicast is what makes the in-place
// update safe: a chunk is in both CTAs before either overwrites it in HBM.
__device__ __forceinline__ void cy_issue_b(CySmem &S, const double *G, int64_t ldg, int64_t m,
                                           const int64_t (&gcol)[4], unsigned rank,
                                           unsigned base, int c) {
  const int lane = threadIdx.x & 31;
  const unsigned gc = base + c;
  const int st = (int)(gc % kCyStages);
  if (gc >= (unsigned)kCyStages) mbar_wait_cluster(&S.empty[st], ((gc / kCyStages) - 1) & 1);
  const int64_t r = (int64_t)c * kBR;
  const uint32_t bytes = (uint32_t)min64(kBR, m - r) * 8u;
  if (lane == 0) mbar_expect_tx(&S.full[st], bytes * kCyCols);
  __syncwarp();
  const int j = 32 * (int)rank + lane;  // this CTA loads slot columns 32 rank ..
  bulk_g2s_mc(&S.u.ring[st][j][0], G + (gcol[j >> 4] + (j & 15)) * ldg + r, bytes, &S.full[st]);
}

// Compute warp CW of a B item: (side, rs) = (CW / 2, CW % 2) produces rows
// 24 rs .. +24 of every chunk of this CTA's block ob[side] and accumulates
// Gram tiles CW, CW+4, CW+8.  The Gram of chunk c runs after the update of
// chunk c+1 (per-stage `upd` mbarriers instead of a CTA barrier per chunk).
template <int CW>
__device__ __forceinline__ void cy_b_consume(CySmem &S, const CyArgs &a, const CyB &J,
                                             unsigned rank, unsigned base, int nchunk,
                                             uint32_t peer_empty0) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  constexpr int side = CW >> 1, rs = CW & 1;
  const int ob = J.ob[side];   // slot block this warp produces
  const int tside = ob >> 1;   // its p-step s-1 task: 0 = t1 (slot cols 0..31), 1 = t2
  const bool upd = J.upd[tside];
  const bool gram = J.gram;
  const bool lag = gram && (J.upd[0] || J.upd[1]);  // Gram waits for other warps' updates
  double *G = a.G;
  const int64_t ldg = a.ldg, m = a.m;
  int64_t gcol[4];
#pragma unroll
  for (int b = 0; b < 4; b++) gcol[b] = (int64_t)J.blk[b] * 16;
  if (CW == 0) {
    fence_async_global();
    fence_async_smem();  // the ring may last have been used by generic code
    for (int c = 0; c < kCyStages - 2 && c < nchunk; c++) cy_issue_b(S, G, ldg, m, gcol, rank, base, c);
  }
  double bf[8][2];
  if (upd) {
    const double *Vt = J.VA[tside];
    const int n0 = 16 * (ob & 1);
#pragma unroll
    for (int kk = 0; kk < 8; kk++)
#pragma unroll
      for (int Y = 0; Y < 2; Y++) bf[kk][Y] = __ldcg(Vt + (n0 + 8 * Y + g) * kCyW + 4 * kk + t);
  }
  int cb[4];
  cb[0] = 16 * J.ob[0];
  cb[1] = 16 * J.ob[0] + 8;
  cb[2] = 16 * J.ob[1];
  cb[3] = 16 * J.ob[1] + 8;
  double acc[3][2];
#pragma unroll
  for (int i = 0; i < 3; i++) acc[i][0] = acc[i][1] = 0.0;
  double *gout = G + gcol[ob] * ldg;
  auto release = [&](int st) {
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&S.empty[st]);
      mbar_arrive_remote(peer_empty0 + st * 8);
    }
  };
  for (int c = 0; c < nchunk; c++) {
    if (CW == 0 && c + kCyStages - 2 < nchunk)
      cy_issue_b(S, G, ldg, m, gcol, rank, base, c + kCyStages - 2);
    const unsigned gc = base + c;
    const int st = (int)(gc % kCyStages);
    mbar_wait(&S.full[st], (gc / kCyStages) & 1);
    double *buf = &S.u.ring[st][0][0];
    const int64_t r = (int64_t)c * kBR;
    const int nr = (int)min64(kBR, m - r);
    if (upd) {
      cy_update_block(buf, 24 * rs, 32 * tside, 16 * ob, bf, gout + r, ldg, nr, g, t);
      fence_async_smem();  // generic writes before the slot's next TMA fill
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.updb[st]);
    if (!lag) {
      if (gram) cy_gram_chunk<CW>(buf, nr, cb, acc, g, t);
      release(st);
    } else if (c > 0) {
      const unsigned gp = gc - 1;
      const int sp = (int)(gp % kCyStages);
      mbar_wait(&S.updb[sp], (gp / kCyStages) & 1);
      cy_gram_chunk<CW>(&S.u.ring[sp][0][0], kBR, cb, acc, g, t);
      release(sp);
    }
  }
  if (lag && nchunk > 0) {
    const unsigned gp = base + nchunk - 1;
    const int sp = (int)(gp % kCyStages);
    mbar_wait(&S.updb[sp], (gp / kCyStages) & 1);
    cy_gram_chunk<CW>(&S.u.ring[sp][0][0], (int)(m - (int64_t)(nchunk - 1) * kBR), cb, acc, g, t);
    release(sp);
  }
  if (gram) cy_gram_store<CW>(J.H, acc, g, t);
}

__device__ __noinline__ void cy_stream_b(CySmem &S, const CyArgs &a, const CyB &J,
                                         unsigned rank) {
  const int warp = threadIdx.x >> 5;
  const int nchunk = (int)cdiv(a.m, kBR);
  const unsigned base = S.chunk;
  const uint32_t peer_empty0 = cluster_map(&S.empty[0], rank ^ 1u);
  switch (warp) {
    case 0: cy_b_consume<0>(S, a, J, rank, base, nchunk, peer_empty0); break;
    case 1: cy_b_consume<1>(S, a, J, rank, base, nchunk, peer_empty0); break;
    case 2: cy_b_consume<2>(S, a, J, rank, base, nchunk, peer_empty0); break;
    default: cy_b_consume<3>(S, a, J, rank, base, nchunk, peer_empty0); break;
  }
  __syncthreads();
  if (threadIdx.x == 0) S.chunk = base + nchunk;
  __syncthreads();
}

__device__ void cy_item_b(CySmem &S, const CyArgs &a, unsigned rank, int bi, int c,
                          unsigned long long *t_stream) {
  const int s = a.s_begin + bi;  // boundary between p-steps s-1 and s
  const int32_t *cy = cy_cycle(a, s, c);
  const int t1 = cy[0], t2 = cy[1];
  const int32_t *pa = cy_pair(a, s + a.S - 1, t1), *pb = cy_pair(a, s + a.S - 1, t2);
  const int64_t WW = (int64_t)kCyW * kCyW;
  CyB J;
  J.blk[0] = pa[0];
  J.blk[1] = pa[1];
  J.blk[2] = pb[0];
  J.blk[3] = pb[1];
  J.upd[0] = J.upd[1] = false;
  J.VA[0] = J.VA[1] = nullptr;
  if (bi > 0) {
    const int64_t i1 = (int64_t)(bi - 1) * a.T + t1, i2 = (int64_t)(bi - 1) * a.T + t2;
    J.upd[0] = __ldcg(&a.rot[i1]) > 0;
    J.upd[1] = __ldcg(&a.rot[i2]) > 0;
    J.VA[0] = a.Vp + i1 * WW;
    J.VA[1] = a.Vp + i2 * WW;
  }
  const int u = cy[2 + rank];
  J.ob[0] = cy[4 + 2 * rank];
  J.ob[1] = cy[5 + 2 * rank];
  J.gram = bi < a.nsteps;
  const int64_t idx = (int64_t)bi * a.T + u;
  J.H = a.H + idx * WW;
  // uniform over the cluster (each u owns one block of t1 and one of t2)
  if (J.gram || J.upd[0] || J.upd[1]) cy_stream_b(S, a, J, rank);
  if (a.trace) *t_stream = cy_clock();
  if (!J.gram) return;
  // inner Jacobi of this CTA's task
  const int32_t *pr = cy_pair(a, s, u);
  inner5_task<kCyW, kCyThreads>(reinterpret_cast<unsigned char *>(&S.u.inner), J.H, a.Vp + idx * WW,
                                pr[0], pr[1], a.n_plus, a.inner, a.inner_limit, a.tol_c,
                                a.counters, s, u, &a.rot[idx]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int ls = bi;
    const int cb = a.tpos[(int64_t)(s % a.S) * a.T + u] >> 1;
    if (atomicAdd(&a.bready[(int64_t)(ls + 1) * a.ncyc + cb], 1) == 1) {
      const long long it = cy_pack(kCyB, ls + 1, cb, 0);
      cy_push(a, 0, &it, 1);
    }
    if (a.nslab_v > 0) {
      const int j = ls >> 1;
      const int cv = ((ls & 1) ? a.upos[(int64_t)(s % a.S) * a.T + u]
                               : a.tpos[(int64_t)(s % a.S) * a.T + u]) >> 1;
      if (atomicAdd(&a.vready[(int64_t)j * a.ncyc + cv], 1) == cy_vtarget(a, j) - 1)
        cy_push_vslabs(a, j, cv);
    }
  }
}

// ---- V items: two p-steps of V updates, rows split over the cluster ------------------

struct CyV {
  int64_t r0, r1;
  int blk[4];
  bool upd[2], updB[2], second;
  int ij[2][2];  // slot blocks of u1, u2
};

// in-place post-multiplication of rows row0..row0+31 of the 32 slot columns
// col(k) = cb0 + k (k < 16), cb1 + k - 16 (k >= 16) by V' in shared memory.
// Output block b also goes straight to HBM when bit b of `fin` is set (its
// value is final after this transform): column gcol[b] + n of V, rows
// grow + row (nr valid rows).
__device__ __forceinline__ void cy_transform_s(double *buf, int row0, int cb0, int cb1,
                                               const double *vp, double *V, int64_t ld,
                                               const int64_t (&gcol)[4], unsigned fin,
                                               int64_t grow, int nr, int g, int t) {
#pragma unroll 1
  for (int rp = 0; rp < 2; rp++) {
    const int rb = row0 + 16 * rp + g;
    double acc[2][4][2];
#pragma unroll
    for (int rt = 0; rt < 2; rt++)
#pragma unroll
      for (int Y = 0; Y < 4; Y++) acc[rt][Y][0] = acc[rt][Y][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
      double b[4];
#pragma unroll
      for (int Y = 0; Y < 4; Y++) b[Y] = vp[(8 * Y + g) * kCyVpLd + 4 * kk + t];
      const int col = (kk < 4 ? cb0 + 4 * kk : cb1 + 4 * kk - 16) + t;
#pragma unroll
      for (int rt = 0; rt < 2; rt++) {
        const double av = buf[col * kLd + rb + 8 * rt];
#pragma unroll
        for (int Y = 0; Y < 4; Y++) dmma(acc[rt][Y][0], acc[rt][Y][1], av, b[Y]);
      }
    }
    // lanes with t >= 2 store their two columns in the opposite order:
    // conflict-free 64-bit shared stores (column stride == 8 banks mod 32)
    const int sw = (t >> 1) & 1;
#pragma unroll
    for (int rt = 0; rt < 2; rt++) {
      const int row = rb + 8 * rt;
#pragma unroll
      for (int Y = 0; Y < 4; Y++) {
        const int cbase = Y < 2 ? cb0 : cb1, blk = cbase >> 4;
        const bool to_global = ((fin >> blk) & 1) && row < nr;
#pragma unroll
        for (int jj = 0; jj < 2; jj++) {
          const int j = jj ^ sw;
          const double v = j ? acc[rt][Y][1] : acc[rt][Y][0];
          const int n = 8 * (Y & 1) + 2 * t + j;
          buf[(cbase + n) * kLd + row] = v;
          if (to_global) st_f64(V + (gcol[blk] + n) * ld + grow + row, v);
        }
      }
    }
  }
}

// compute warp cw owns slot half h = cw / 2 (transform t_h, then u_h) and
// rows 32 (cw % 2) .. +32 of every chunk
__device__ __forceinline__ void cy_issue_v(CySmem &S, const double *V, int64_t ldv, const CyV &J,
                                           unsigned base, int c) {
  const int lane = threadIdx.x & 31;
  const unsigned gc = base + c;
  const int st = (int)(gc % kCyVStages);
  if (gc >= (unsigned)kCyVStages) mbar_wait(&S.vempty[st], ((gc / kCyVStages) - 1) & 1);
  const int64_t r = J.r0 + (int64_t)c * kRch;
  const uint32_t bytes = (uint32_t)min64(kRch, J.r1 - r) * 8u;
  if (lane == 0) mbar_expect_tx(&S.vfull[st], bytes * kCyCols);
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int j = lane + 32 * h;
    const int64_t col = (int64_t)J.blk[j >> 4] * 16 + (j & 15);
    bulk_g2s(&S.u.v.ring[st][j][0], V + col * ldv + r, bytes, &S.vfull[st]);
  }
}

__device__ __noinline__ void cy_stream_v(CySmem &S, double *V, int64_t ldv, const CyV &J) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nchunk = (int)cdiv(J.r1 - J.r0, kRch);
  const unsigned base = S.vchunk;
  if (warp == 0) {
    fence_async_global();
    fence_async_smem();
    for (int c = 0; c < kCyVStages - 1 && c < nchunk; c++) cy_issue_v(S, V, ldv, J, base, c);
  }
  const int cw = warp, half = cw >> 1, rs = cw & 1;
  const bool myA = J.upd[half];
  const bool myB = J.second && J.updB[half];
  const int gb0 = 16 * J.ij[half][0], gb1 = 16 * J.ij[half][1];
  int64_t gcol[4];
#pragma unroll
  for (int b = 0; b < 4; b++) gcol[b] = (int64_t)J.blk[b] * 16;
  // blocks whose final value comes out of transform A (no B transform on them)
  unsigned finB = 0;
  if (J.second) {
    if (J.updB[0]) finB |= (1u << J.ij[0][0]) | (1u << J.ij[0][1]);
    if (J.updB[1]) finB |= (1u << J.ij[1][0]) | (1u << J.ij[1][1]);
  }
  const unsigned finA = 0xFu & ~finB;
  for (int c = 0; c < nchunk; c++) {
    if (warp == 0 && c + kCyVStages - 1 < nchunk) cy_issue_v(S, V, ldv, J, base, c + kCyVStages - 1);
    const unsigned gc = base + c;
    const int st = (int)(gc % kCyVStages);
    mbar_wait(&S.vfull[st], (gc / kCyVStages) & 1);
    double *buf = &S.u.v.ring[st][0][0];
    const int64_t r = J.r0 + (int64_t)c * kRch;
    const int nr = (int)min64(kRch, J.r1 - r);
    if (myA)
      cy_transform_s(buf, rs * 32, 32 * half, 32 * half + 16, &S.u.v.vp[half][0][0], V, ldv,
                     gcol, finA, r, nr, g, t);
    if (J.second) {
      compute_bar();
      if (myB)
        cy_transform_s(buf, rs * 32, gb0, gb1, &S.u.v.vp[2 + half][0][0], V, ldv, gcol, 0xFu,
                       r, nr, g, t);
    }
    fence_async_smem();  // generic writes before the slot's next TMA fill
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.vempty[st]);
  }
  __syncthreads();
  if (threadIdx.x == 0) S.vchunk = base + nchunk;
  __syncthreads();
}

__device__ void cy_item_v(CySmem &S, const CyArgs &a, unsigned rank, int j, int c, int k) {
  const int la = 2 * j;  // local index of step a
  const int sa = a.s_begin + la;
  const int32_t *cy = cy_cycle(a, sa + 1, c);  // boundary (a, a+1)
  const int t1 = cy[0], t2 = cy[1];
  const int32_t *pa = cy_pair(a, sa, t1), *pb = cy_pair(a, sa, t2);
  const int64_t WW = (int64_t)kCyW * kCyW;
  CyV J;
  const int64_t s0 = (int64_t)k * kCyVSlab, s1 = min64(s0 + kCyVSlab, a.nv);
  const int64_t half = cdiv(cdiv(s1 - s0, 2), kRch) * kRch;
  J.r0 = rank == 0 ? s0 : min64(s0 + half, s1);
  J.r1 = rank == 0 ? min64(s0 + half, s1) : s1;
  J.blk[0] = pa[0];
  J.blk[1] = pa[1];
  J.blk[2] = pb[0];
  J.blk[3] = pb[1];
  const int64_t i1 = (int64_t)la * a.T + t1, i2 = (int64_t)la * a.T + t2;
  J.upd[0] = __ldcg(&a.rot[i1]) > 0;
  J.upd[1] = __ldcg(&a.rot[i2]) > 0;
  J.second = la + 1 < a.nsteps;
  J.updB[0] = J.updB[1] = false;
  J.ij[0][0] = cy[4];
  J.ij[0][1] = cy[5];
  J.ij[1][0] = cy[6];
  J.ij[1][1] = cy[7];
  const double *src[4] = {a.Vp + i1 * WW, a.Vp + i2 * WW, nullptr, nullptr};
  if (J.second) {
    const int64_t u1 = (int64_t)(la + 1) * a.T + cy[2], u2 = (int64_t)(la + 1) * a.T + cy[3];
    J.updB[0] = __ldcg(&a.rot[u1]) > 0;
    J.updB[1] = __ldcg(&a.rot[u2]) > 0;
    src[2] = a.Vp + u1 * WW;
    src[3] = a.Vp + u2 * WW;
  }
  if (J.r1 > J.r0 && (J.upd[0] || J.upd[1] || J.updB[0] || J.updB[1])) {
    const bool use[4] = {J.upd[0], J.upd[1], J.updB[0], J.updB[1]};
    for (int e = threadIdx.x; e < 4 * kCyW * kCyW; e += blockDim.x) {
      const int i = e / (kCyW * kCyW), rr = e - i * kCyW * kCyW;
      if (use[i]) S.u.v.vp[i][rr / kCyW][rr % kCyW] = __ldcg(src[i] + rr);
    }
    __syncthreads();
    cy_stream_v(S, a.V, a.ldv, J);
  }
}

// thread 0 of rank 0, after both CTAs finished V item (j, c, k): the last V
// item of pair j releases the cycles of pair j+1 (whole CTA cooperates)
__device__ void cy_v_done(CySmem &S, const CyArgs &a, int j) {
  if (threadIdx.x == 0) {
    __threadfence();
    S.last = (atomicAdd(&a.vdone[j], 1) == a.ncyc * a.nslab_v - 1);
  }
  __syncthreads();
  if (S.last && j + 1 < a.npairs) {
    __threadfence();
    const int tg = cy_vtarget(a, j + 1);
    for (int cc = threadIdx.x; cc < a.ncyc; cc += blockDim.x)
      if (atomicAdd(&a.vready[(int64_t)(j + 1) * a.ncyc + cc], 1) == tg - 1)
        cy_push_vslabs(a, j + 1, cc);
  }
  __syncthreads();
}

// launched with 2-CTA clusters
__global__ void __launch_bounds__(kCyThreads, 2) k_cycle(CyArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  CySmem &S = *reinterpret_cast<CySmem *>(smraw);
  const unsigned rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kCyStages; i++) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], 8);  // 4 local + 4 peer compute warps
      mbar_init(&S.updb[i], 4);
    }
    for (int i = 0; i < kCyVStages; i++) {
      mbar_init(&S.vfull[i], 1);
      mbar_init(&S.vempty[i], 4);
    }
    fence_mbar_init();
    S.chunk = 0;
    S.vchunk = 0;
  }
  cluster_sync();
  for (;;) {
    if (rank == 0 && threadIdx.x == 0) {
      const long long it = cy_pop(a);
      S.item = it;
      asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(cluster_map(&S.item, 1)), "l"(it)
                   : "memory");
    }
    cluster_sync();
    const long long item = S.item;
    if (item < 0) break;
    const int type = (int)(item >> 60), x = (int)((item >> 40) & 0xfffff),
              y = (int)((item >> 16) & 0xffffff), k = (int)(item & 0xffff);
    const unsigned long long t0 = a.trace ? cy_clock() : 0;
    unsigned long long tm = t0;
    if (type == kCyB)
      cy_item_b(S, a, rank, x, y, &tm);
    else
      cy_item_v(S, a, rank, x, y, k);
    __syncthreads();
    cluster_sync();  // both halves done (and S.item free for the next pop)
    if (rank == 0) {
      if (type == kCyV) cy_v_done(S, a, x);
      if (threadIdx.x == 0) atomicAdd(&a.sched->done, 1ull);
    }
    if (a.trace && threadIdx.x == 0) {
      const unsigned long long t1 = cy_clock();
      const long long i = (long long)atomicAdd((unsigned long long *)a.trace, 1ull);
      if (i < a.trace_cap) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long *r = a.trace + 4 + 4 * i;
        r[0] = item;
        r[1] = smid | ((long long)rank << 16) | ((long long)((tm - t0) / 1000) << 32);
        r[2] = (long long)t0;
        r[3] = (long long)t1;
      }
    }
  }
  cluster_sync();  // no CTA leaves while its peer may still address its smem
}

__global__ void k_cycle_init(CyArgs a) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int i = tid; i < 2 * kCyQCap; i += nth)
    if (i >= a.ncyc) a.qseq[i] = -1;
  for (int i = tid; i < (a.nsteps + 1) * a.ncyc; i += nth) a.bready[i] = 0;
  for (int i = tid; i < a.npairs * a.ncyc; i += nth) a.vready[i] = i < a.ncyc ? 1 : 0;
  for (int i = tid; i < a.npairs; i += nth) a.vdone[i] = 0;
  if (tid == 0) {
    a.sched->head[0] = a.sched->head[1] = 0;
    a.sched->tail[0] = (unsigned long long)a.ncyc;
    a.sched->tail[1] = 0;
    a.sched->done = 0;
    if (a.trace) a.trace[0] = 0;
  }
  for (int c = tid; c < a.ncyc; c += nth) {
    a.qitem[c] = cy_pack(kCyB, 0, c, 0);
    a.qseq[c] = c;
  }
}

// ---- host side ------------------------------------------------------------------

static long long *g_cy_trace = nullptr;
static long long g_cy_trace_cap = 0;

void cycle_trace(void *buf, int64_t cap) {
  g_cy_trace = (long long *)buf;
  g_cy_trace_cap = buf ? cap : 0;
}

int64_t cycle_plan_ints(int b) {
  if (b < 4 || b % 4) return 0;
  const int64_t S = b - 1, T = b / 2, nc = T / 2;
  return S * nc * 8 + 2 * S * T;
}

int cycle_plan(const int32_t *outer, int b, int32_t *plan) {
  if (b < 4 || b % 4) return 1;
  const int S = b - 1, T = b / 2, nc = T / 2;
  int32_t *cyc = plan, *tpos = plan + (int64_t)S * nc * 8, *upos = tpos + (int64_t)S * T;
  std::vector<int> tprev(b), tcur(b), seen(T);
  auto pr = [&](int s, int t, int k) { return outer[((int64_t)s * T + t) * 2 + k]; };
  for (int s = 0; s < S; s++) {
    const int sp = (s + S - 1) % S;
    for (int t = 0; t < T; t++) {
      tprev[pr(sp, t, 0)] = t;
      tprev[pr(sp, t, 1)] = t;
      tcur[pr(s, t, 0)] = t;
      tcur[pr(s, t, 1)] = t;
      seen[t] = 0;
    }
    int c = 0;
    for (int t1 = 0; t1 < T; t1++) {
      if (seen[t1]) continue;
      const int p1 = pr(sp, t1, 0), q1 = pr(sp, t1, 1);
      const int u1 = tcur[p1], u2 = tcur[q1];
      if (u1 == u2) return 1;  // same pair in both steps: not a 4-cycle
      const int x = pr(s, u1, 0) == p1 ? pr(s, u1, 1) : pr(s, u1, 0);
      const int y = pr(s, u2, 0) == q1 ? pr(s, u2, 1) : pr(s, u2, 0);
      const int t2 = tprev[x];
      if (tprev[y] != t2 || t2 == t1 || seen[t2]) return 1;
      const int p2 = pr(sp, t2, 0), q2 = pr(sp, t2, 1);
      auto slot = [&](int col) {
        return col == p1 ? 0 : col == q1 ? 1 : col == p2 ? 2 : col == q2 ? 3 : -1;
      };
      int32_t *e = cyc + ((int64_t)s * nc + c) * 8;
      e[0] = t1;
      e[1] = t2;
      e[2] = u1;
      e[3] = u2;
      e[4] = slot(pr(s, u1, 0));
      e[5] = slot(pr(s, u1, 1));
      e[6] = slot(pr(s, u2, 0));
      e[7] = slot(pr(s, u2, 1));
      for (int i = 4; i < 8; i++)
        if (e[i] < 0) return 1;
      if (c >= nc) return 1;
      tpos[(int64_t)sp * T + t1] = 2 * c;
      tpos[(int64_t)sp * T + t2] = 2 * c + 1;
      upos[(int64_t)s * T + u1] = 2 * c;
      upos[(int64_t)s * T + u2] = 2 * c + 1;
      seen[t1] = seen[t2] = 1;
      c++;
    }
    if (c != nc) return 1;
  }
  return 0;
}

bool cycle_ok(int w, int64_t m, int64_t ldg, int64_t nv, int64_t ldv) {
  return w == kCyW && m % 2 == 0 && ldg % 2 == 0 && nv % 2 == 0 && ldv % 2 == 0;
}

int64_t cycle_workspace_bytes(int64_t n, int w) {
  if (w != kCyW) return 0;
  const int64_t T = n / w, b = n / (w / 2), nsteps = b - 1, nc = T / 2;
  const int64_t npairs = (nsteps + 1) / 2;
  auto rnd = [](int64_t x) { return (x + 255) / 256 * 256; };
  int64_t bytes = 0;
  bytes += 2 * rnd(nsteps * T * w * w * 8);  // H, Vp
  bytes += rnd(nsteps * T * 8);              // rot
  bytes += rnd((nsteps + 1) * nc * 4);       // bready
  bytes += rnd(npairs * nc * 4);             // vready
  bytes += rnd(npairs * 4);                  // vdone
  bytes += rnd(sizeof(CySched));
  bytes += 4 * rnd((int64_t)kCyQCap * 8);    // two queues
  return bytes + 4096;
}

int launch_cycle(double *G, int64_t ldg, int64_t m, double *V, int64_t ldv, int64_t nv,
                 const int32_t *outer, const int32_t *plan, int b, int s_begin, int nsteps,
                 const int32_t *inner, int64_t n_plus, int inner_limit, double tol_c,
                 unsigned long long *counters, void *ws, cudaStream_t st) {
  const int w = kCyW;
  CyArgs a{};
  a.G = G;
  a.ldg = ldg;
  a.m = m;
  a.V = V;
  a.ldv = ldv;
  a.nv = V ? nv : 0;
  a.outer = outer;
  a.S = b - 1;
  a.T = b / 2;
  a.ncyc = a.T / 2;
  a.cyc = plan;
  a.tpos = plan + (int64_t)a.S * a.ncyc * 8;
  a.upos = a.tpos + (int64_t)a.S * a.T;
  a.inner = inner;
  a.n_plus = n_plus;
  a.inner_limit = inner_limit;
  a.tol_c = tol_c;
  a.counters = counters;
  a.s_begin = s_begin;
  a.nsteps = nsteps;
  a.nslab_v = a.nv > 0 ? (int)cdiv(a.nv, kCyVSlab) : 0;
  a.npairs = a.nslab_v > 0 ? (nsteps + 1) / 2 : 0;
  a.total = (unsigned long long)(nsteps + 1) * a.ncyc +
            (unsigned long long)a.npairs * a.ncyc * a.nslab_v;
  char *p = (char *)ws;
  auto take = [&](int64_t bytes) {
    char *r = p;
    p += (bytes + 255) / 256 * 256;
    return (void *)r;
  };
  const int64_t T = a.T, nc = a.ncyc;
  a.H = (double *)take((int64_t)nsteps * T * w * w * 8);
  a.Vp = (double *)take((int64_t)nsteps * T * w * w * 8);
  a.rot = (int64_t *)take((int64_t)nsteps * T * 8);
  a.bready = (int *)take((int64_t)(nsteps + 1) * nc * 4);
  a.vready = (int *)take((int64_t)((nsteps + 1) / 2) * nc * 4);
  a.vdone = (int *)take((int64_t)((nsteps + 1) / 2) * 4);
  a.sched = (CySched *)take(sizeof(CySched));
  a.qitem = (long long *)take((int64_t)2 * kCyQCap * 8);
  a.qseq = (long long *)take((int64_t)2 * kCyQCap * 8);
  a.trace = g_cy_trace;
  a.trace_cap = g_cy_trace_cap;
  const size_t smem = sizeof(CySmem);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kCyThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int clusters = 0;
  if (!clusters) {
    cudaFuncSetAttribute(k_cycle, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cfg.gridDim = dim3(2 * sms);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_cycle, &cfg) != cudaSuccess || nc <= 0) nc = sms / 2;
    const char *e = getenv("JHSVD_CYCLE_CLUSTERS");  // override (tuning)
    if (e && atoi(e) > 0 && atoi(e) < nc) nc = atoi(e);
    clusters = nc;
  }
  cfg.gridDim = dim3(2 * clusters);
  k_cycle_init<<<64, 256, 0, st>>>(a);
  cudaLaunchKernelEx(&cfg, k_cycle, a);
  return 0;
}

}  // namespace jh
