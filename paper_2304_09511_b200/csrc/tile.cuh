// Fixed-size entry tiles shared by the CSR and COO plain kernels.
//
// A tile is kTile consecutive stored entries plus a kExt-entry extension
// (the tail of a short row that starts in the tile), staged into shared
// memory by TMA bulk copies in a persistent, STAGES-deep pipeline.  Work per
// tile is independent of the row-length distribution (Zipf rows up to 50k
// entries), and every entry is read from HBM once.
#pragma once

#include "tma.cuh"

namespace spmv {

constexpr int kExt = 32;  // == kExactLen: a short row never reaches further
constexpr int kTileThreads = 256;
constexpr int kTileStages = 2;
constexpr uint32_t kNoRow = 0xffffffffu;

// Long segments per tile: at most TILE/(kExactLen+1) inner ones + 2 boundary.
template <int TILE>
constexpr int max_long_segs() { return TILE / (kExactLen + 1) + 4; }

// Tile size used by the plans (entries).  1024 keeps more CTAs resident per
// SM (smaller shared-memory ring); 2048 halves the per-tile overhead.
int tile_entries();
int ctas_per_sm_cap();  // 0 = occupancy limit

static_assert(kExt == kExactLen, "extension must cover a whole short row");

struct LongSeg {
  uint32_t row;
  uint32_t lo, hi;  // entry range inside this tile [lo, hi), tile-relative
  uint32_t flags;   // CSR: unused; COO: bit0 cont_before, bit1 cont_after
  uint32_t s, e;    // CSR: the row's global entry range
};

// Number of tiles whose [E0, E0 + kTile + kExt) window (clamped to nnz) can be
// bulk-copied without reading past the arrays: all of them when nnz % 4 == 0,
// otherwise those with E0 + kTile + kExt <= nnz.
inline int64_t bulk_tiles(int64_t nnz, int64_t ntiles, int64_t tile) {
  if (nnz % 4 == 0) return ntiles;
  const int64_t full = (nnz - tile - kExt) >= 0 ? (nnz - tile - kExt) / tile + 1 : 0;
  return full < ntiles ? full : ntiles;
}

// Left-to-right dot product of a staged row: acc = ((acc0 + p0) + p1) + ...
// with p_j = vals[j] * x[cols[j]] rounded first.  Eight gathers are issued
// before their adds (the add order is unchanged).  acc0 = -0.0 reproduces
// cumsum (the first product itself, kernels.py:81); acc0 = +0.0 reproduces
// np.add.at on a zeroed y (kernels.py:65).
template <typename T>
__device__ __forceinline__ T row_dot(const uint32_t* __restrict__ c, const T* __restrict__ v, int len,
                                     const T* __restrict__ xb, T acc) {
  int i = 0;
  for (; i + 8 <= len; i += 8) {
    T p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = mul_rn(v[i + j], __ldg(xb + c[i + j]));
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = add_rn(acc, p[j]);
  }
  for (; i < len; ++i) acc = add_rn(acc, mul_rn(v[i], __ldg(xb + c[i])));
  return acc;
}

// Warp-level vla-32 dot product of staged entries [lo, hi): lane l sums
// lo+l, lo+l+32, ... then the lanes.py:107-128 tree.  Equals
// spmv_csr_vla(32) when [lo, hi) is a whole row.
template <typename T>
__device__ __forceinline__ T warp_segment_dot(const uint32_t* __restrict__ c, const T* __restrict__ v, uint32_t lo,
                                              uint32_t hi, int lane, const T* __restrict__ xb) {
  T acc = T(0);
  for (uint32_t j = lo + lane; j < hi; j += 32) acc = add_rn(acc, mul_rn(v[j], __ldg(xb + c[j])));
  return tree_reduce_warp(acc, 32);
}

}  // namespace spmv
