// DMMA Gram-tile device code shared by the Gram kernel (jh_tiles.cu) and
// the Gram CTAs of the engine-1 update launch (jh_vpair.cu): staged 64-row
// chunks of a block pair (column stride kLd) are consumed by NW warps, each owning the lower 8x8
// tiles i == WARP (mod NW); every tile is one in-order DMMA chain over the
// rows (see jh_dmma.cuh for why that is bitwise the reference's fma chain).
#pragma once

#include "jh_dmma.cuh"

namespace jh {

constexpr int kRch = 64;          // rows per staged chunk
constexpr int kLd = kRch + 4;     // padded smem column stride (doubles)
constexpr int kStages = 3;


// Consumer side of the Gram for warp WARP of NW: it owns tiles i = WARP
// (mod NW) of the (W/8)(W/8+1)/2 lower tiles (enumerated row-major, X >= Y).
template <int W, int NW>
struct GramTiles {
  static constexpr int NT = W / 8;
  static constexpr int NTILE = NT * (NT + 1) / 2;
  static constexpr int MY = (NTILE + NW - 1) / NW;
};

template <int W, int NW, int WARP, int RCH = kRch, int LD = RCH + 4>
__device__ __forceinline__ void gram_chunk(const double *buf, int nr, double (&acc)[GramTiles<W, NW>::MY][2],
                                           int t) {
  constexpr int NT = W / 8;
  auto tiles = [&](const double (&f)[NT]) {
    int i = 0, mine = 0;
#pragma unroll
    for (int X = 0; X < NT; X++)
#pragma unroll
      for (int Y = 0; Y <= X; Y++, i++)
        if (i % NW == WARP) {
          dmma(acc[mine][0], acc[mine][1], f[X], f[Y]);
          mine++;
        }
  };
  auto step = [&](int kk, bool guard) {
    double f[NT];
    const bool ok = !guard || (4 * kk + t < nr);
#pragma unroll
    for (int X = 0; X < NT; X++) f[X] = ok ? buf[X * 8 * LD + 4 * kk] : 0.0;
    tiles(f);
  };
  if (nr == RCH) {
    // explicit two-stage register pipeline: fragments of k-step kk+1 are
    // loaded before the DMMAs of k-step kk are issued
    // (an odd k-step count -- RCH = 4 mod 16 for the dense tensor-tile
    // stages -- ends with one k-step in fa)
    constexpr int NKS = RCH / 4;
    double fa[NT], fb[NT];
#pragma unroll
    for (int X = 0; X < NT; X++) fa[X] = buf[X * 8 * LD];
#pragma unroll
    for (int kk = 0; kk + 1 < NKS; kk += 2) {
#pragma unroll
      for (int X = 0; X < NT; X++) fb[X] = buf[X * 8 * LD + 4 * (kk + 1)];
      tiles(fa);
      if (kk + 2 < NKS) {
#pragma unroll
        for (int X = 0; X < NT; X++) fa[X] = buf[X * 8 * LD + 4 * (kk + 2)];
      }
      tiles(fb);
    }
    if constexpr (NKS % 2) tiles(fa);
  } else {
    const int nks = (nr + 3) / 4;
    for (int kk = 0; kk < nks; kk++) step(kk, true);
  }
}

template <int W, int NW, int WARP>
__device__ __forceinline__ void gram_store(double *H, const double (&acc)[GramTiles<W, NW>::MY][2],
                                           int g, int t) {
  constexpr int NT = W / 8;
  int i = 0, mine = 0;
#pragma unroll
  for (int X = 0; X < NT; X++)
#pragma unroll
    for (int Y = 0; Y <= X; Y++, i++)
      if (i % NW == WARP) {
#pragma unroll
        for (int j = 0; j < 2; j++) {
          const int x = 8 * X + g, y = 8 * Y + 2 * t + j;
          H[y * W + x] = acc[mine][j];
          if (X != Y) H[x * W + y] = acc[mine][j];
        }
        mine++;
      }
}

}  // namespace jh
