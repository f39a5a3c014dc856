// grouped.cuh — persistent tile scheduler over the expert-sorted row space
// produced by realb_moe_align (layout words, include/realb.h).
//
// Tiles of one precision class are numbered t = mt * n_tiles + nt where mt
// runs over the concatenated 128-row m-tiles of the class's groups (experts)
// and nt over the BN-wide n-tiles of N. Consecutive CTAs therefore share an
// A m-block (L2 reuse of activations) and sweep the expert's weight rows.
#pragma once
#include "common.cuh"

namespace realb {

struct TileCoord {
  int group;    // global expert id
  int a_row;    // first row of the 128-row m-block in the grouped row space
  int n0;       // first output column
  int valid;    // rows of this m-block that carry real (token, expert) pairs
};

struct GroupedSched {
  const int32_t* glist;   // [G] expert ids of this precision class
  const int32_t* prefix;  // [G+1] exclusive prefix of m-tiles
  const int32_t* pprefix; // [G+1] exclusive prefix of m-tile pairs (2-CTA clusters)
  const int32_t* row_start;
  const int32_t* row_count;
  int G;
  int n_tiles;
  int BN;

  __device__ __forceinline__ static GroupedSched make(const int32_t* layout, int E, int prec,
                                                      int N, int BN) {
    GroupedSched s;
    s.glist = layout + LayoutView::off_glist(E, prec);
    s.prefix = layout + LayoutView::off_prefix(E, prec);
    s.pprefix = layout + LayoutView::off_pprefix(E, prec);
    s.row_start = layout + LayoutView::off_row_start(E);
    s.row_count = layout + LayoutView::off_row_count(E);
    s.G = layout[1 + prec];
    s.n_tiles = N / BN;
    s.BN = BN;
    return s;
  }
  __device__ __forceinline__ int total() const { return G > 0 ? prefix[G] * n_tiles : 0; }

  // 2-CTA pair units: u = pair * n_tiles + nt. Both CTAs of a cluster take the
  // same (expert, n-tile) and the two m-tiles of the pair (cluster rank 0 / 1);
  // an expert with an odd m-tile count gives rank 1 a dummy (no compute) slot.
  __device__ __forceinline__ int total_pairs() const { return G > 0 ? pprefix[G] * n_tiles : 0; }
  __device__ __forceinline__ TileCoord coord_pair(int u, int rank, bool& dummy) const {
    const int pp = u / n_tiles, nt = u - pp * n_tiles;
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pprefix[mid] <= pp) lo = mid; else hi = mid - 1;
    }
    TileCoord c;
    c.group = glist[lo];
    const int mt_lo = prefix[lo], mt_hi = prefix[lo + 1];
    int mt = mt_lo + 2 * (pp - pprefix[lo]) + rank;
    dummy = mt >= mt_hi;
    if (dummy) mt -= 1;
    const int local = mt - mt_lo;
    c.a_row = row_start[c.group] + local * 128;
    c.n0 = nt * BN;
    const int rem = row_count[c.group] - local * 128;
    c.valid = rem < 128 ? rem : 128;
    return c;
  }

  // Dynamic tile fetch: layout words [4 + 2p] (next tile) and [5 + 2p] (CTAs
  // done) of precision class p are zeroed by the align kernels; the last CTA
  // to finish re-zeroes them so the next launch on the same layout starts at 0.
  __device__ __forceinline__ static int* counters(const int32_t* layout, int prec) {
    return const_cast<int*>(layout) + 4 + 2 * prec;
  }
  __device__ __forceinline__ static void finish(const int32_t* layout, int prec) {
    int* c = counters(layout, prec);
    __threadfence();
    if (atomicAdd(c + 1, 1) == (int)gridDim.x - 1) {
      c[0] = 0;
      c[1] = 0;
      __threadfence();
    }
  }
  __device__ __forceinline__ TileCoord coord(int t) const {
    const int mt = t / n_tiles, nt = t - mt * n_tiles;
    // largest g with prefix[g] <= mt (groups with zero tiles are skipped naturally)
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= mt) lo = mid; else hi = mid - 1;
    }
    TileCoord c;
    c.group = glist[lo];
    const int local = mt - prefix[lo];
    c.a_row = row_start[c.group] + local * 128;
    c.n0 = nt * BN;
    const int rem = row_count[c.group] - local * 128;
    c.valid = rem < 128 ? rem : 128;
    return c;
  }
};

}  // namespace realb
