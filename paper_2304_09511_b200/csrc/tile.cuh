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

static_assert(kExt == kExactLen, "extension must cover a whole short row");

// A consumer group of NT threads inside a tile CTA.  The single-group
// kernels use the whole CTA (barrier 0 == __syncthreads); the multi-group
// CSR kernel runs G groups of 128 threads, each on its own named barrier, so
// G tiles are computed at once while one more stage is loading.
template <int NT>
struct TileGroup {
  int tid;  // thread index inside the group
  int bar;  // named barrier id
  __device__ __forceinline__ void sync() const {
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NT) : "memory");
  }
};

struct LongSeg {
  uint32_t row;
  uint32_t lo, hi;  // entry range inside this tile [lo, hi), tile-relative
  uint32_t flags;   // CSR: unused; COO: bit0 cont_before, bit1 cont_after
  uint32_t s, e;    // CSR: the row's global entry range
};

// Number of tiles whose [E0, E0 + kTile + kExt) window (clamped to nnz) can be
// bulk-copied without reading past the arrays: all of them when nnz % 4 == 0,
// otherwise those with E0 + kTile + kExt <= nnz.
// Every tile is bulk-copyable: the issuing thread copies the last tiles'
// 1..3 entries past a 16-byte multiple itself (csr.cu / coo.cu issue()).
inline int64_t bulk_tiles(int64_t nnz, int64_t ntiles, int64_t tile) {
  (void)nnz;
  (void)tile;
  return ntiles;
}

// Left-to-right dot product of a staged row: acc = ((acc0 + p0) + p1) + ...
// with p_j = vals[j] * x[cols[j]] rounded first.  Eight gathers are issued
// before their adds (the add order is unchanged).  acc0 = -0.0 reproduces
// cumsum (the first product itself, kernels.py:81); acc0 = +0.0 reproduces
// np.add.at on a zeroed y (kernels.py:65).
#ifndef SPMV_ROW_BATCH
#define SPMV_ROW_BATCH 8
#endif
#ifndef SPMV_ROW_TAIL_SWITCH
#define SPMV_ROW_TAIL_SWITCH 1
#endif

// True when every active lane of the warp has the same tail count.
__device__ __forceinline__ bool tail_uniform(int r) {
  const unsigned am = __activemask();
  return __all_sync(am, r == __shfl_sync(am, r, __ffs(am) - 1));
}

template <typename T, int N>
__device__ __forceinline__ T row_tail(const uint32_t* __restrict__ c, const T* __restrict__ v,
                                      const T* __restrict__ xb, T acc) {
  T p[N];
#pragma unroll
  for (int j = 0; j < N; ++j) p[j] = mul_rn(v[j], ldx(xb + c[j]));
#pragma unroll
  for (int j = 0; j < N; ++j) acc = add_rn(acc, p[j]);
  return acc;
}

// Exact-count tail of r < N + 1 entries: compare chain over N .. 1.
template <typename T, int N>
__device__ __forceinline__ T row_tail_dispatch(int r, const uint32_t* __restrict__ c, const T* __restrict__ v,
                                               const T* __restrict__ xb, T acc) {
  if constexpr (N == 0) {
    return acc;
  } else {
    if (r == N) return row_tail<T, N>(c, v, xb, acc);
    return row_tail_dispatch<T, N - 1>(r, c, v, xb, acc);
  }
}

// BIG (the tile kernels): 16-wide batches plus an exact-count tail of up
// to 15, so a row of up to 16 entries (the banded matrix's 11) takes one
// gather round trip and the stencil's 27 take two (8-wide batches with a
// serial tail took four and six).
template <typename T, bool BIG = false>
__device__ __forceinline__ T row_dot(const uint32_t* __restrict__ c, const T* __restrict__ v, int len,
                                     const T* __restrict__ xb, T acc) {
#if SPMV_ROW_TAIL_SWITCH
  if constexpr (BIG) {
    int i = 0;
    for (; i + 16 <= len; i += 16) acc = row_tail<T, 16>(c + i, v + i, xb, acc);
    return row_tail_dispatch<T, 15>(len - i, c + i, v + i, xb, acc);
  }
#endif
  constexpr int B = SPMV_ROW_BATCH;
  int i = 0;
  for (; i + B <= len; i += B) {
    T p[B];
#pragma unroll
    for (int j = 0; j < B; ++j) p[j] = mul_rn(v[i + j], ldx(xb + c[i + j]));
#pragma unroll
    for (int j = 0; j < B; ++j) acc = add_rn(acc, p[j]);
  }
  if (B > 8)
    for (; i + 8 <= len; i += 8) {
      T p[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) p[j] = mul_rn(v[i + j], ldx(xb + c[i + j]));
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = add_rn(acc, p[j]);
    }
#if SPMV_ROW_TAIL_SWITCH
  // the last len - i < 8 entries: an exact-count batch (no predicates),
  // their gathers in flight together rather than one round trip each
  switch (len - i) {
    case 7: return row_tail<T, 7>(c + i, v + i, xb, acc);
    case 6: return row_tail<T, 6>(c + i, v + i, xb, acc);
    case 5: return row_tail<T, 5>(c + i, v + i, xb, acc);
    case 4: return row_tail<T, 4>(c + i, v + i, xb, acc);
    case 3: return row_tail<T, 3>(c + i, v + i, xb, acc);
    case 2: return row_tail<T, 2>(c + i, v + i, xb, acc);
    case 1: return add_rn(acc, mul_rn(v[i], ldx(xb + c[i])));
    default: return acc;
  }
#else
  for (; i < len; ++i) acc = add_rn(acc, mul_rn(v[i], ldx(xb + c[i])));
  return acc;
#endif
}

// vla rows from staged entries, one thread per row (rows of <= 32 entries).
// The reference's lane arithmetic does not depend on which hardware lane
// holds a logical lane, so one thread can play all W = next_pow2(L) of them
// in registers with the same adds in the same order — bit-exact, with the
// row-per-lane gather pattern of the plain tile kernels.
//   CSR (kernels.py:143-171): acc[l] = +0.0, then acc[l] += p_j for
//     j = l, l+L, ... (masked_fma, lanes.py:101-104); tree over W lanes,
//     vals[:w] + vals[w:2w] (lanes.py:107-128); inactive lanes stay 0.
//   COO (kernels.py:104-140): steps of L entries; each step's products
//     (0 on inactive lanes) tree-reduce to t_k; y = ((+0.0 + t_0) + t_1)...
template <typename T, int W>
__device__ __forceinline__ T tree_regs(T (&v)[W]) {
#pragma unroll
  for (int w = W / 2; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) v[i] = add_rn(v[i], v[i + w]);
  return v[0];
}

// lanes 0..N-1 of a partial last block (exact count: no predicates)
template <typename T, int W, int N>
__device__ __forceinline__ void vla_block_part(T (&acc)[W], const uint32_t* __restrict__ c,
                                               const T* __restrict__ v, const T* __restrict__ xb) {
  if constexpr (N > 0 && N < W) {
    T p[N];
#pragma unroll
    for (int l = 0; l < N; ++l) p[l] = mul_rn(v[l], ldx(xb + c[l]));
#pragma unroll
    for (int l = 0; l < N; ++l) acc[l] = add_rn(acc[l], p[l]);
  }
}

// tree of a partial last step: lanes 0..N-1 products, the others 0
template <typename T, int W, int N>
__device__ __forceinline__ T vla_step_part(const uint32_t* __restrict__ c, const T* __restrict__ v,
                                           const T* __restrict__ xb) {
  T p[W];
#pragma unroll
  for (int l = 0; l < W; ++l) p[l] = T(0);
  if constexpr (N > 0 && N < W) {
#pragma unroll
    for (int l = 0; l < N; ++l) p[l] = mul_rn(v[l], ldx(xb + c[l]));
  }
  return tree_regs<T, W>(p);
}

// MIXED: the warp's rows differ in length (the long-row plans' short-row
// kernels): the tail switch runs only when the counts agree, a switch over
// mixed counts would serialise its cases.
template <typename T, int W, bool MIXED = false>
__device__ __forceinline__ T row_vla_csr(const uint32_t* __restrict__ c, const T* __restrict__ v, int len,
                                         const T* __restrict__ xb, int L) {
  T acc[W];
#pragma unroll
  for (int l = 0; l < W; ++l) acc[l] = T(0);
  int base = 0;
  if (L == W) {  // power-of-two lane count: whole blocks without predicates
    if constexpr (W <= 8)  // two blocks' gathers in flight together
      for (; base + 2 * W <= len; base += 2 * W) {
        T p[2 * W];
#pragma unroll
        for (int l = 0; l < 2 * W; ++l) p[l] = mul_rn(v[base + l], ldx(xb + c[base + l]));
#pragma unroll
        for (int l = 0; l < W; ++l) acc[l] = add_rn(acc[l], p[l]);
#pragma unroll
        for (int l = 0; l < W; ++l) acc[l] = add_rn(acc[l], p[W + l]);
      }
    for (; base + W <= len; base += W) {
      T p[W];
#pragma unroll
      for (int l = 0; l < W; ++l) p[l] = mul_rn(v[base + l], ldx(xb + c[base + l]));
#pragma unroll
      for (int l = 0; l < W; ++l) acc[l] = add_rn(acc[l], p[l]);
    }
#if SPMV_ROW_TAIL_SWITCH
    // the partial last block: its lanes as one exact-count batch
    if (!MIXED || tail_uniform(len - base)) {
    switch (len - base) {
      case 1: vla_block_part<T, W, 1>(acc, c + base, v + base, xb); break;
      case 2: vla_block_part<T, W, 2>(acc, c + base, v + base, xb); break;
      case 3: vla_block_part<T, W, 3>(acc, c + base, v + base, xb); break;
      case 4: vla_block_part<T, W, 4>(acc, c + base, v + base, xb); break;
      case 5: vla_block_part<T, W, 5>(acc, c + base, v + base, xb); break;
      case 6: vla_block_part<T, W, 6>(acc, c + base, v + base, xb); break;
      case 7: vla_block_part<T, W, 7>(acc, c + base, v + base, xb); break;
      default: break;
    }
    return tree_regs<T, W>(acc);
    }
#endif
  }
  for (; base < len; base += L) {
    T p[W];
#pragma unroll
    for (int l = 0; l < W; ++l) p[l] = (l < L && base + l < len) ? mul_rn(v[base + l], ldx(xb + c[base + l])) : T(0);
#pragma unroll
    for (int l = 0; l < W; ++l)
      if (l < L && base + l < len) acc[l] = add_rn(acc[l], p[l]);
  }
  return tree_regs<T, W>(acc);
}

template <typename T, int W, bool MIXED = false>
__device__ __forceinline__ T row_vla_coo(const uint32_t* __restrict__ c, const T* __restrict__ v, int len,
                                         const T* __restrict__ xb, int L) {
  T y = T(0);
  int base = 0;
  if (L == W) {  // power-of-two lane count: whole steps without predicates
    if constexpr (W <= 8)  // two steps' gathers in flight together
      for (; base + 2 * W <= len; base += 2 * W) {
        T p[W], q[W];
#pragma unroll
        for (int l = 0; l < W; ++l) p[l] = mul_rn(v[base + l], ldx(xb + c[base + l]));
#pragma unroll
        for (int l = 0; l < W; ++l) q[l] = mul_rn(v[base + W + l], ldx(xb + c[base + W + l]));
        y = add_rn(y, tree_regs<T, W>(p));
        y = add_rn(y, tree_regs<T, W>(q));
      }
    for (; base + W <= len; base += W) {
      T p[W];
#pragma unroll
      for (int l = 0; l < W; ++l) p[l] = mul_rn(v[base + l], ldx(xb + c[base + l]));
      y = add_rn(y, tree_regs<T, W>(p));
    }
#if SPMV_ROW_TAIL_SWITCH
    // the partial last step: its lanes as one exact-count batch, the rest 0
    if (!MIXED || tail_uniform(len - base)) switch (len - base) {
      case 1: return add_rn(y, vla_step_part<T, W, 1>(c + base, v + base, xb));
      case 2: return add_rn(y, vla_step_part<T, W, 2>(c + base, v + base, xb));
      case 3: return add_rn(y, vla_step_part<T, W, 3>(c + base, v + base, xb));
      case 4: return add_rn(y, vla_step_part<T, W, 4>(c + base, v + base, xb));
      case 5: return add_rn(y, vla_step_part<T, W, 5>(c + base, v + base, xb));
      case 6: return add_rn(y, vla_step_part<T, W, 6>(c + base, v + base, xb));
      case 7: return add_rn(y, vla_step_part<T, W, 7>(c + base, v + base, xb));
      default: return y;
    }
#endif
  }
  for (; base < len; base += L) {
    T p[W];
#pragma unroll
    for (int l = 0; l < W; ++l) p[l] = (l < L && base + l < len) ? mul_rn(v[base + l], ldx(xb + c[base + l])) : T(0);
    y = add_rn(y, tree_regs<T, W>(p));
  }
  return y;
}

// W = 16 / 32 (and L > 32): too many registers for a lane array.  The
// row's rounded products are formed in place in the staged values (the row
// is this thread's alone), then the tree is evaluated as an adjacent
// pairwise sum over the logical lanes in bit-reversed order — the same
// pairs as vals[:w] + vals[w:2w] — with a log2(W)-deep stack.
template <int W>
__device__ __forceinline__ constexpr int bitrev(int k) {
  int r = 0;
  for (int b = 1; b < W; b <<= 1) {
    r = (r << 1) | (k & 1);
    k >>= 1;
  }
  return r;
}

template <typename T, int W, typename Leaf>
__device__ __forceinline__ T tree_stack(Leaf leaf) {
  constexpr int LOG = W == 16 ? 4 : 5;
  static_assert(W == 16 || W == 32, "wide trees");
  T st[LOG];
  T v = T(0);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    v = leaf(bitrev<W>(k));
#pragma unroll
    for (int b = 0; b < LOG; ++b) {
      if (!((k >> b) & 1)) {
        st[b] = v;
        break;
      }
      v = add_rn(st[b], v);
    }
  }
  return v;
}

template <typename T>
__device__ __forceinline__ void products_in_place(const uint32_t* __restrict__ c, T* __restrict__ v, int len,
                                                  const T* __restrict__ xb) {
  int i = 0;
  for (; i + 8 <= len; i += 8) {
    T x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = ldx(xb + c[i + j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[i + j] = mul_rn(v[i + j], x[j]);
  }
  for (; i < len; ++i) v[i] = mul_rn(v[i], ldx(xb + c[i]));
}

template <typename T, int W>
__device__ __forceinline__ T row_vla_csr_wide(const uint32_t* __restrict__ c, T* __restrict__ v, int len,
                                              const T* __restrict__ xb, int L) {
  products_in_place(c, v, len, xb);
  return tree_stack<T, W>([&](int l) {
    T a = T(0);
    if (l < L)
      for (int j = l; j < len; j += L) a = add_rn(a, v[j]);
    return a;
  });
}

// upper: next_pow2(L) > 32 — the tree levels above 32 lanes add +0.0 to
// every live lane once (which turns a -0.0 product into +0.0).
template <typename T, int W>
__device__ __forceinline__ T row_vla_coo_wide(const uint32_t* __restrict__ c, T* __restrict__ v, int len,
                                              const T* __restrict__ xb, int L, bool upper) {
  products_in_place(c, v, len, xb);
  T y = T(0);
  for (int base = 0; base < len; base += L) {
    const int cnt = min(L, len - base);
    y = add_rn(y, tree_stack<T, W>([&](int l) {
      const T p = l < cnt ? v[base + l] : T(0);
      return upper ? add_rn(p, T(0)) : p;
    }));
  }
  return y;
}

// Indices i whose segment starts[i+1] - starts[i] lies in (lo, hi] (CSR rows
// or COO runs of one length class; order irrelevant).  out == nullptr counts.
static __global__ void len_class_list_kernel(const uint32_t* __restrict__ starts, int64_t n, uint32_t lo,
                                             uint32_t hi, uint32_t* __restrict__ out,
                                             unsigned long long* __restrict__ cnt) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t len = starts[i + 1] - starts[i];
    if (len > lo && len <= hi) {
      const unsigned long long k = atomicAdd(cnt, 1ull);
      if (out) out[k] = uint32_t(i);
    }
  }
}

// Left-to-right sum of already-formed products (the "products" tile mode).
template <typename T>
__device__ __forceinline__ T row_sum(const T* __restrict__ p, int len, T acc) {
  for (int i = 0; i < len; ++i) acc = add_rn(acc, p[i]);
  return acc;
}

// Products mode: every thread forms the rounded products of entries
// tid, tid+256, ... in place (4 gathers in flight).  Used for tiles holding
// many short rows, where a row per lane would serialise ~1 L2 round trip
// per row; entry-per-lane issues the whole tile's gathers in parallel.
template <typename T, int NT = kTileThreads>
__device__ __forceinline__ void form_products(const uint32_t* __restrict__ cols, T* __restrict__ vals, int cnt,
                                              const T* __restrict__ xb, int gtid) {
  int k = gtid;
  for (; k + 3 * NT < cnt; k += 4 * NT) {
    const uint32_t c0 = cols[k], c1 = cols[k + NT], c2 = cols[k + 2 * NT], c3 = cols[k + 3 * NT];
    const T x0 = ldx(xb + c0), x1 = ldx(xb + c1), x2 = ldx(xb + c2), x3 = ldx(xb + c3);
    vals[k] = mul_rn(vals[k], x0);
    vals[k + NT] = mul_rn(vals[k + NT], x1);
    vals[k + 2 * NT] = mul_rn(vals[k + 2 * NT], x2);
    vals[k + 3 * NT] = mul_rn(vals[k + 3 * NT], x3);
  }
  for (; k < cnt; k += NT) vals[k] = mul_rn(vals[k], ldx(xb + cols[k]));
}

// Long segments of one tile, reduced by all warps of the CTA: every segment
// is cut into kUnit-entry units (lane-strided vla-32 reduction each); the
// partials of a segment are then added in unit order by one thread.  A
// segment of <= kUnit entries is a single unit, so a whole row of 33..kUnit
// entries inside one tile is bit-exact with spmv_csr_vla(32); longer ones
// are deterministic and within 1e-12.
constexpr int kUnit = 256;
template <int TILE>
constexpr int max_units() { return TILE / kUnit + max_long_segs<TILE>(); }

struct LongUnit {  // scratch slot; reduce_long_segments stores unit offsets here
  uint32_t a, b;
};

// seg_part[i] <- reduction of segment i (i < nl).  Ends with a group barrier.
template <typename T, int TILE, int NT = kTileThreads>
__device__ __forceinline__ void reduce_long_segments(const uint32_t* __restrict__ cols, const T* __restrict__ vals,
                                     const LongSeg* __restrict__ segs, int nl, LongUnit* units, T* unit_part,
                                     int* s_nunits, T* seg_part, const T* __restrict__ xb, bool products,
                                     bool warp_per_seg, const TileGroup<NT>& grp) {
  const int tid = grp.tid, lane = tid & 31, warp = tid >> 5;
  if (warp_per_seg) {
    for (int i = warp; i < nl; i += NT / 32) {
      T acc = T(0);
      for (uint32_t j = segs[i].lo + lane; j < segs[i].hi; j += 32)
        acc = add_rn(acc, products ? vals[j] : mul_rn(vals[j], ldx(xb + cols[j])));
      acc = tree_reduce_warp(acc, 32);
      if (lane == 0) seg_part[i] = acc;
    }
    grp.sync();
    return;
  }
  // unit offsets of the segments: warp 0 scans ceil(len / kUnit), up to
  // 4 segments per lane (nl <= max_long_segs < 128)
  int* first = reinterpret_cast<int*>(units);  // first[i] = first unit of segment i, first[nl] = total
  if (warp == 0) {
    int cnt[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane * 4 + q;
      cnt[q] = i < nl ? int((segs[i].hi - segs[i].lo + kUnit - 1) / kUnit) : 0;
      sum += cnt[q];
    }
    int incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - sum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane * 4 + q;
      if (i < nl) first[i] = run;
      run += cnt[q];
    }
    if (lane == 31) {
      first[nl] = incl;
      *s_nunits = incl;
    }
  }
  grp.sync();
  const int nu = *s_nunits;
  for (int u = warp; u < nu; u += NT / 32) {
    int lo_i = 0, hi_i = nl - 1;  // segment of unit u: last i with first[i] <= u
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i + 1) >> 1;
      if (first[mid] <= u) lo_i = mid; else hi_i = mid - 1;
    }
    const uint32_t ulo = segs[lo_i].lo + uint32_t(u - first[lo_i]) * kUnit;
    const uint32_t uhi = min(segs[lo_i].hi, ulo + uint32_t(kUnit));
    T acc = T(0);
    uint32_t j = ulo + lane;
    if (products) {
      for (; j < uhi; j += 32) acc = add_rn(acc, vals[j]);
    } else {
      // A unit is at most kUnit / 32 = 8 entries per lane: all of them are
      // gathered at once (predicated), then added in lane order, so a unit
      // costs one L2 round trip whatever its length.
      constexpr int PER_LANE = kUnit / 32;
      T p[PER_LANE];
#pragma unroll
      for (int k = 0; k < PER_LANE; ++k) {
        const uint32_t jk = j + 32u * uint32_t(k);
        p[k] = jk < uhi ? mul_rn(vals[jk], ldx(xb + cols[jk])) : T(0);
      }
#pragma unroll
      for (int k = 0; k < PER_LANE; ++k)
        if (j + 32u * uint32_t(k) < uhi) acc = add_rn(acc, p[k]);
    }
    acc = tree_reduce_warp(acc, 32);
    if (lane == 0) unit_part[u] = acc;
  }
  grp.sync();
  for (int i = tid; i < nl; i += NT) {
    T s = unit_part[first[i]];
    for (int u = first[i] + 1; u < first[i + 1]; ++u) s = add_rn(s, unit_part[u]);
    seg_part[i] = s;
  }
  grp.sync();
}

// Warp-level vla-32 dot product of staged entries [lo, hi): lane l sums
// lo+l, lo+l+32, ... then the lanes.py:107-128 tree.  Equals
// spmv_csr_vla(32) when [lo, hi) is a whole row.
template <typename T>
__device__ __forceinline__ T warp_segment_dot(const uint32_t* __restrict__ c, const T* __restrict__ v, uint32_t lo,
                                              uint32_t hi, int lane, const T* __restrict__ xb) {
  T acc = T(0);
  for (uint32_t j = lo + lane; j < hi; j += 32) acc = add_rn(acc, mul_rn(v[j], ldx(xb + c[j])));
  return tree_reduce_warp(acc, 32);
}

}  // namespace spmv
