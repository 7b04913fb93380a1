// CSR SpMV for sm_100a.
//
// Reference: spmv_csr_plain (kernels.py:69-82) sums each row strictly left
// to right after rounding every product; spmv_csr_vla (kernels.py:143-171)
// uses L strided lane accumulators and a pairwise tree (lanes.py:107-128).
//
// Plain path — csr_tile_kernel, persistent, TMA-fed (tile.cuh):
//   1. a producer thread bulk-copies the tile's column indices and values
//      (TILE + kExt entries) into a STAGES-deep shared-memory ring;
//   2. rows that start in the tile with <= exact_len entries (all stencil
//      rows) are computed by one thread each: rounded products of the
//      staged values and gathered x, summed left to right — the reference
//      order, so bit-exact; empty rows get +0.0.  Row-per-lane mapping puts
//      32 consecutive rows in a warp, so each gather instruction touches a
//      few consecutive x lines (entry-per-lane would touch ~10 and saturate
//      the L1 wavefront pipe);
//   3. longer rows: one warp per in-tile segment (vla-32 order, so a long
//      row inside one tile is bit-exact with spmv_csr_vla(32)); a row that
//      spans tiles leaves one partial per tile and the last tile to finish
//      (atomic ticket, no spinning) adds them in tile order — deterministic,
//      within 1e-12 of the reference.
// Every stored entry is read from HBM exactly once (+kExt/TILE = 1.6%
// overlap that hits L2), the row pointers once, x through L2, y written
// once: the minimum-byte model of SURVEY.md §8(d).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "hostpipe.cuh"
#include "panel.cuh"
#include "tile.cuh"
#include "wstream.cuh"

namespace spmv {

#ifdef SPMV_PHASE_TIMING
// [0] wait  [1] rows (thread 0, incl. barrier)  [2] long+end barrier  [3] issue
// [4] sum of row-thread loop cycles  [5] row-thread count  [6] tiles
__device__ unsigned long long g_phase[8];
#define PHASE_T(v) const unsigned long long v = clock64()
#define PHASE_ADD(i, v) (s_phase_acc[i] += (unsigned long long)(v))
#else
#define PHASE_T(v)
#define PHASE_ADD(i, v)
#endif

#ifdef SPMV_PHASE_TIMING
// per-CTA accumulators in shared memory (thread 0 writes), flushed once
#define PHASE_DECL __shared__ unsigned long long s_phase_acc[8];
#else
#define PHASE_DECL
#endif

template <typename T>
struct CsrParams {
  const uint32_t* irp;
  const uint32_t* aj;
  const T* av;
  const T* x;
  T* y;
  const uint32_t* row_lo;  // ntiles + 1: first row of each tile's row range
  T* head;
  T* tail;
  int64_t nrows, nnz, col_base, ntiles, n_bulk;
  int64_t tile_begin, tile_end;  // tiles [tile_begin, tile_end) of this launch
  int exact_len;
  int mode;
  int vla;  // lanes L of a vla tile launch (template VW = next_pow2(L) > 0)
  // rows >= y_split are stored y_gap entries further on (spmv_csr_gapped:
  // a slab's two boundary planes in one launch); y_split = INT64_MAX else
  int64_t y_split, y_gap;
  // row r of this matrix is y[ymap[r]] (the panel path's short-row CSR);
  // nullptr else
  const uint32_t* ymap;
};

template <typename T>
__device__ __forceinline__ int64_t yrow(const CsrParams<T>& P, int64_t r) {
  if (P.ymap) return int64_t(P.ymap[r]);
  return r >= P.y_split ? r + P.y_gap : r;
}

// Shared memory of a CSR tile CTA with G consumer groups and G + 1 stages:
// [0, 64) stage mbarriers, [64, 96) stage tickets, [96, 160) two counters
// per group, then one long-row scratch block per group, then the stage ring.
template <typename T, int TILE, int G = 1, bool LONG = true>
struct CsrSmem {
  static constexpr int stages = G + 1;
  static constexpr size_t cols_bytes = align_up(sizeof(uint32_t) * (TILE + kExt), 128);
  static constexpr size_t vals_bytes = align_up(sizeof(T) * (TILE + kExt), 128);
  static constexpr size_t stage_bytes = cols_bytes + vals_bytes;
  static constexpr size_t units_off = align_up(sizeof(LongSeg) * max_long_segs<TILE>(), 16);  // in a group block
  static constexpr size_t upart_off = units_off + align_up(sizeof(LongUnit) * max_units<TILE>(), 16);
  static constexpr size_t spart_off = upart_off + align_up(sizeof(T) * max_units<TILE>(), 16);
  // plans without long rows never queue a segment: no long-row scratch
  static constexpr size_t group_bytes = LONG ? align_up(spart_off + sizeof(T) * max_long_segs<TILE>(), 16) : 0;
  static constexpr size_t tickets_off = 64, counters_off = 96, groups_off = 160;
  static constexpr size_t header = align_up(groups_off + G * group_bytes, 128);
  static constexpr size_t total = header + stages * stage_bytes;
  static_assert(stages <= 8, "mbarrier / ticket / counter slots");
};

// Threads per CTA and resident CTAs per SM the CSR tile kernel is built for.
template <int G> constexpr int csr_group_threads() { return G == 1 ? kTileThreads : 128; }
template <int G> constexpr int csr_cta_threads() { return G * csr_group_threads<G>(); }
#ifndef SPMV_CSR_MINB
#define SPMV_CSR_MINB 4
#endif
template <int G> constexpr int csr_min_blocks() { return G == 1 ? SPMV_CSR_MINB : (G == 2 ? 3 : (G <= 4 ? 2 : 1)); }

// Rows of one tile.  Row-per-lane mode (few rows per tile, e.g. the
// stencil's ~77): each thread forms its row's products from the staged
// entries, so a warp's gathers hit consecutive x.  Products mode (more rows
// than threads, e.g. Zipf's short rows): all gathers of the tile are issued
// entry-per-lane first, then rows are summed from shared memory.  Long
// segments are only queued here.
template <typename T, int TILE, int NT, bool LONG, int VW = 0>
__device__ __forceinline__ void csr_tile_rows(const CsrParams<T>& P, int64_t t, const uint32_t* __restrict__ cols,
                                              T* __restrict__ vals, LongSeg* s_long, int* s_nlong,
                                              const TileGroup<NT>& grp
#ifdef SPMV_PHASE_TIMING
                                              , unsigned long long* s_phase_acc
#endif
) {
  const int tid = grp.tid;
  const int64_t E0 = t * TILE;
  const int64_t E1 = E0 + TILE;
  const T* xb = P.x - P.col_base;
  const int64_t R0 = t == 0 ? 0 : int64_t(P.row_lo[t]);
  const int64_t R1 = P.row_lo[t + 1];
  const int64_t rend = R1 < P.nrows ? R1 + 1 : P.nrows;
  int64_t r = R0 + tid;
  uint32_t s = 0, e = 0;
  if (r < rend) {
    s = __ldg(P.irp + r);
    e = __ldg(P.irp + r + 1);
  }
  const bool products = VW == 0 && (P.mode & 1) && (rend - R0) > NT;
  if (products) form_products<T, NT>(cols, vals, int(min(int64_t(TILE + kExt), P.nnz - E0)), xb, tid);
  if (tid == 0) *s_nlong = 0;
  grp.sync();
  PHASE_T(rt0);
#ifdef SPMV_PHASE_TIMING
  const bool had_row = r < rend;
#endif
  while (r < rend) {
    const uint32_t len = e - s;
    if (len == 0) {
      if (r < R1) P.y[yrow(P, r)] = T(0);
    } else if (len <= uint32_t(P.exact_len)) {
      if (int64_t(s) >= E0 && int64_t(s) < E1) {
        // vla: the CSR lane order, or (mode bit 3: a COO plan's row-pointer
        // view) the COO step order of kernels.py:174-210
        if constexpr (VW >= 16)
          P.y[yrow(P, r)] = (P.mode & 8) ? row_vla_coo_wide<T, VW>(cols + (s - E0), vals + (s - E0), int(len), xb,
                                                                   P.vla, P.vla > 32)
                                         : row_vla_csr_wide<T, VW>(cols + (s - E0), vals + (s - E0), int(len), xb,
                                                                   P.vla);
        else if constexpr (VW > 0)
          P.y[yrow(P, r)] = (P.mode & 8) ? row_vla_coo<T, VW>(cols + (s - E0), vals + (s - E0), int(len), xb, P.vla)
                                         : row_vla_csr<T, VW>(cols + (s - E0), vals + (s - E0), int(len), xb, P.vla);
        else
          // -0.0 seed: the sum starts from the first product, like cumsum;
          // +0.0 (mode bit 3) for a COO plan's row-pointer view: np.add.at
          // on a zeroed y (kernels.py:65)
          P.y[yrow(P, r)] = products ? row_sum(vals + (s - E0), int(len), (P.mode & 8) ? T(0) : T(-0.0))
                            : row_dot<T, true>(cols + (s - E0), vals + (s - E0), int(len), xb,
                                               (P.mode & 8) ? T(0) : T(-0.0));
      }
    } else {
      const int64_t lo = max(int64_t(s), E0), hi = min(int64_t(e), E1);
      if (LONG && lo < hi) {
        const int idx = atomicAdd(s_nlong, 1);
        LongSeg L;
        L.row = uint32_t(r);
        L.lo = uint32_t(lo - E0);
        L.hi = uint32_t(hi - E0);
        L.flags = products ? 1u : 0u;
        L.s = s;
        L.e = e;
        s_long[idx] = L;
      }
    }
    r += NT;
    if (r < rend) {
      s = __ldg(P.irp + r);
      e = __ldg(P.irp + r + 1);
    }
  }
#ifdef SPMV_PHASE_TIMING
  if (had_row && threadIdx.x == 0) {  // thread 0 only: no atomic contention
    PHASE_T(rt1);
    PHASE_ADD(4, rt1 - rt0);
    PHASE_ADD(5, 1);
  }
#endif
  grp.sync();
}

// Long segments of one tile.  A row inside the tile is written directly; a
// row spanning tiles leaves its partial in tail[t] (the tile holding its
// first entry) or head[t] (later tiles); csr_span_fixup_kernel adds them in
// tile order after the tile kernel (no fences or atomics in the hot kernel).
template <typename T, int TILE, int NT>
__device__ __forceinline__ void csr_tile_long(int64_t t, const uint32_t* __restrict__ cols, const T* __restrict__ vals,
                                           const LongSeg* __restrict__ s_long, int nl, unsigned char* scratch,
                                           int* s_nunits, const T* __restrict__ xb, T* __restrict__ y,
                                           T* __restrict__ head, T* __restrict__ tail, bool warp_per_seg,
                                           const TileGroup<NT>& grp) {
  using S = CsrSmem<T, TILE>;  // group-block offsets do not depend on G
  LongUnit* units = reinterpret_cast<LongUnit*>(scratch + S::units_off);
  T* unit_part = reinterpret_cast<T*>(scratch + S::upart_off);
  T* seg_part = reinterpret_cast<T*>(scratch + S::spart_off);
  const bool products = s_long[0].flags & 1u;
  reduce_long_segments<T, TILE, NT>(cols, vals, s_long, nl, units, unit_part, s_nunits, seg_part, xb, products,
                                    warp_per_seg, grp);
  const int64_t E0 = t * TILE, E1 = E0 + TILE;
  for (int i = grp.tid; i < nl; i += NT) {
    const LongSeg L = s_long[i];
    const T part = seg_part[i];
    if (int64_t(L.s) >= E0 && int64_t(L.e) <= E1)
      y[L.row] = part;
    else if (int64_t(L.s) >= E0)
      tail[t] = part;  // the row starts here and continues: csr_span_fixup_kernel adds the rest
    else
      head[t] = part;
  }
}

// G == 1: one 256-thread group, 2 stages (a tile computes while the next
// loads).  G > 1: G groups of 128 threads over G + 1 stages, tile i of the
// CTA going to group i % G and stage i % (G + 1): G tiles compute while one
// loads, so more rows are in flight per byte of shared memory (the stencil's
// limiter).  Multi-group CTAs take bulk tiles only; the host runs the tail
// tiles with G == 1.
template <typename T, bool BULK, int TILE, int G, bool LONG = true, int VW = 0>
__global__ void __launch_bounds__(csr_cta_threads<G>(), csr_min_blocks<G>())
csr_tile_kernel(const __grid_constant__ CsrParams<T> P) {
  static_assert(VW == 0 || !LONG, "vla tile launches serve plans without long rows");
  static_assert(G == 1 || BULK, "multi-group CTAs are TMA-fed");
  constexpr int NT = csr_group_threads<G>();
  extern __shared__ __align__(128) unsigned char smem[];
  PHASE_DECL
#ifdef SPMV_PHASE_TIMING
  if (threadIdx.x < 8) s_phase_acc[threadIdx.x] = 0;
  __syncthreads();
#endif
  using S = CsrSmem<T, TILE, G, LONG>;
  constexpr int STAGES = S::stages;
  const int g = int(threadIdx.x) / NT;
  const TileGroup<NT> grp{int(threadIdx.x) % NT, G == 1 ? 0 : 1 + g};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  volatile int* tickets = reinterpret_cast<volatile int*>(smem + S::tickets_off);  // CTA-local tile of each stage
  int* s_nlong = reinterpret_cast<int*>(smem + S::counters_off) + 2 * g;           // [0] segments, [1] units
  unsigned char* gscratch = smem + S::groups_off + size_t(g) * S::group_bytes;
  LongSeg* s_long = reinterpret_cast<LongSeg*>(gscratch);
  unsigned char* stages = smem + S::header;
  auto cols_of = [&](int s) { return reinterpret_cast<uint32_t*>(stages + s * S::stage_bytes); };
  auto vals_of = [&](int s) { return reinterpret_cast<T*>(stages + s * S::stage_bytes + S::cols_bytes); };

  // This CTA's tiles (grid-strided over [tile_begin, tile_end), so all SMs
  // sweep neighbouring rows together and share x lines in L2): bulk-copyable
  // ones first (TMA pipeline), then the tail tiles the bulk engine cannot
  // address (cooperative loads, G == 1 only).
  const int64_t n_bulk = BULK ? min(P.n_bulk, P.tile_end) : P.tile_begin;
  const int64_t first = P.tile_begin + blockIdx.x, stride = gridDim.x;
  const int64_t mine_bulk = first < n_bulk ? (n_bulk - 1 - first) / stride + 1 : 0;
  const int64_t tail0 = max(n_bulk, P.tile_begin) + blockIdx.x;
  const int64_t mine_tail = G == 1 && tail0 < P.tile_end ? (P.tile_end - 1 - tail0) / stride + 1 : 0;
  auto issue = [&](int64_t i) {
    const int64_t E0 = (first + i * stride) * TILE;
    const uint32_t cnt = uint32_t(min(int64_t(TILE + kExt), P.nnz - E0));
    const uint32_t cb = cnt & ~3u;  // bulk part: 16-byte multiples
    const int s = int(i % STAGES);
    if (G > 1) tickets[s] = int(i);
    // the last tiles' 1..3 odd entries: plain copies, published by the
    // arrive below (release) like the bulk bytes by complete_tx
    for (uint32_t k = cb; k < cnt; ++k) {
      cols_of(s)[k] = P.aj[E0 + k];
      vals_of(s)[k] = P.av[E0 + k];
    }
    mbar_arrive_expect_tx(&bars[s], cb * uint32_t(sizeof(uint32_t) + sizeof(T)));
    if (cb) {
      bulk_g2s(cols_of(s), P.aj + E0, cb * uint32_t(sizeof(uint32_t)), &bars[s], (P.mode & 4) != 0);
      bulk_g2s(vals_of(s), P.av + E0, cb * uint32_t(sizeof(T)), &bars[s], (P.mode & 4) != 0);
    }
  };
  if (BULK) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&bars[s], 1);
        tickets[s] = -1;
      }
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int64_t i = 0; i < STAGES && i < mine_bulk; ++i) issue(i);
  }
  for (int64_t i = g; i < mine_bulk + mine_tail; i += G) {
    int s = 0;
    int64_t t;
    PHASE_T(p0);
    if (i < mine_bulk) {
      s = int(i % STAGES);
      t = first + i * stride;
      // A parity wait only tells the current phase from the previous one.
      // With G > 1 the previous tile of this stage belongs to another group
      // and may still be in flight, so first wait until tile i is the one
      // issued into the stage (its predecessor's phase has then completed).
      if (G > 1)
        while (tickets[s] != int(i)) __nanosleep(32);
      mbar_wait(&bars[s], uint32_t((i / STAGES) & 1));
#ifdef SPMV_DEBUG_CHECKS
      {  // the staged tile is exactly the global entries (no ring race)
        const int64_t E0 = t * TILE;
        const int cnt = int(min(int64_t(TILE + kExt), P.nnz - E0));
        for (int k = grp.tid; k < cnt; k += NT) {
          SPMV_DCHECK(cols_of(s)[k] == P.aj[E0 + k], 0);
          SPMV_DCHECK(same_bits(vals_of(s)[k], P.av[E0 + k]), 0);
        }
      }
#endif
    } else {
      t = tail0 + (i - mine_bulk) * stride;
      const int64_t E0 = t * TILE;
      const int cnt = int(min(int64_t(TILE + kExt), P.nnz - E0));
      for (int k = grp.tid; k < cnt; k += NT) {
        cols_of(0)[k] = P.aj[E0 + k];
        vals_of(0)[k] = P.av[E0 + k];
      }
      grp.sync();
    }
    PHASE_T(p1);
#ifndef SPMV_STREAM_ONLY  // experiment: TMA stream alone (y is not written)
    csr_tile_rows<T, TILE, NT, LONG, VW>(P, t, cols_of(s), vals_of(s), s_long, s_nlong, grp
#ifdef SPMV_PHASE_TIMING
                               , s_phase_acc
#endif
    );
    PHASE_T(p2);
    const int nl = LONG ? *s_nlong : 0;
    if (LONG && nl > 0)
      csr_tile_long<T, TILE, NT>(t, cols_of(s), vals_of(s), s_long, nl, gscratch, s_nlong + 1, P.x - P.col_base,
                                 P.y, P.head, P.tail, (P.mode & 2) != 0, grp);
#endif
    grp.sync();  // stage s free
    PHASE_T(p3);
    if (BULK && grp.tid == 0 && i + STAGES < mine_bulk) {
      fence_proxy_async();
      issue(i + STAGES);
    }
#ifdef SPMV_PHASE_TIMING
    if (threadIdx.x == 0) {
      PHASE_T(p4);
      PHASE_ADD(0, p1 - p0);
      PHASE_ADD(1, p2 - p1);
      PHASE_ADD(2, p3 - p2);
      PHASE_ADD(3, p4 - p3);
      PHASE_ADD(6, 1);
    }
#endif
  }
#ifdef SPMV_PHASE_TIMING
  __syncthreads();
  if (threadIdx.x < 8) atomicAdd(&g_phase[threadIdx.x], s_phase_acc[threadIdx.x]);
#endif
}

// Rows spanning tiles: y = tail[t0] + head[t0+1] + ... + head[t1].
template <typename T>
__global__ void csr_span_fixup_kernel(const uint32_t* __restrict__ span_row, const uint32_t* __restrict__ span_t0,
                                      const uint32_t* __restrict__ span_t1, int64_t n_span, const T* __restrict__ head,
                                      const T* __restrict__ tail, T* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_span; i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t t0 = span_t0[i], t1 = span_t1[i];
    T sum = tail[t0];
    for (uint32_t u = t0 + 1; u <= t1; ++u) sum = add_rn(sum, head[u]);
    y[span_row[i]] = sum;
  }
}

__global__ void csr_span_list_kernel(const uint32_t* __restrict__ irp, int64_t nrows, int exact_len, int64_t tile,
                                     uint32_t* __restrict__ span_row, uint32_t* __restrict__ span_t0,
                                     uint32_t* __restrict__ span_t1, unsigned long long* __restrict__ n_span) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = irp[r], e = irp[r + 1];
    if (e - s <= uint32_t(exact_len)) continue;
    const uint64_t t0 = s / uint64_t(tile), t1 = (uint64_t(e) - 1) / uint64_t(tile);
    if (t0 == t1) continue;
    const unsigned long long k = atomicAdd(n_span, 1ull);
    if (span_row) {
      span_row[k] = uint32_t(r);
      span_t0[k] = uint32_t(t0);
      span_t1[k] = uint32_t(t1);
    }
  }
}

// maxcol[t] = largest column read by tile t (its entries + the kExt
// extension): the x prefix a tile-range launch needs (pipelined uploads).
__global__ void tile_maxcol_kernel(const uint32_t* __restrict__ aj, int64_t nnz, int64_t ntiles, int64_t tile,
                                   uint32_t* __restrict__ maxcol) {
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t e0 = t * tile, e1 = min(nnz, e0 + tile + kExt);
    uint32_t m = 0;
    for (int64_t j = e0 + threadIdx.x; j < e1; j += blockDim.x) m = max(m, aj[j]);
    for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    __shared__ uint32_t w[8];
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < int(blockDim.x >> 5); ++i) m = max(m, w[i]);
      maxcol[t] = max(m, w[0]);
    }
    __syncthreads();
  }
}

// row_lo[t] = row containing entry t*kTile (last r with irp[r] <= t*kTile);
// row_lo[ntiles] = nrows.
__global__ void csr_row_lo_kernel(const uint32_t* __restrict__ irp, int64_t nrows, int64_t ntiles, int64_t tile,
                                  uint32_t* __restrict__ row_lo) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t <= ntiles; t += int64_t(gridDim.x) * blockDim.x) {
    if (t == ntiles) {
      row_lo[t] = uint32_t(nrows);
      continue;
    }
    const uint64_t key = uint64_t(t) * uint64_t(tile);
    int64_t lo = 0, hi = nrows;  // find last r in [0, nrows) with irp[r] <= key
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (uint64_t(irp[mid]) <= key) lo = mid; else hi = mid - 1;
    }
    row_lo[t] = uint32_t(lo);
  }
}

__global__ void count_long_rows_kernel(const uint32_t* __restrict__ irp, int64_t nrows, int exact_len,
                                       unsigned long long* __restrict__ n_long) {
  unsigned long long c = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x)
    c += irp[r + 1] > irp[r] && (irp[r + 1] - irp[r]) > uint32_t(exact_len);
  for (int o = 16; o >= 1; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(n_long, c);
}

// ---- vla: sub-warp (L <= 32) or CTA (32 < L <= 1024) per row ------------
// Rows longer than kVlaLong entries go to csr_vla_long_kernel (L <= 32).
constexpr uint32_t kVlaLong = 256;

// One warp per long row.  The 32 lanes gather a 256-entry chunk of rounded
// products into shared memory at once (8 loads in flight per lane); then
// logical lane l < L folds its entries s+l, s+l+L, ... from shared memory in
// order — the same add sequence as csr_vla_warp_kernel, so bit-identical —
// and the tree over next_pow2(L) lanes follows (lanes.py:107-128).
template <typename T>
__global__ void __launch_bounds__(256)
csr_vla_long_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj, const T* __restrict__ av,
                    const T* __restrict__ x, int64_t col_base, T* __restrict__ y, int64_t nrows, int lanes,
                    int width) {
  __shared__ T s_p[8][kVlaLong];
  const T* xb = x - col_base;
  const int lane = threadIdx.x & 31;
  T* buf = s_p[threadIdx.x >> 5];
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t L = uint32_t(lanes);
  for (int64_t r0 = warp * 32; r0 < nrows; r0 += nwarps * 32) {
    // 32 rows per coalesced load; only the long ones are processed
    const int64_t rl = r0 + lane;
    const uint32_t sl = rl < nrows ? irp[rl] : 0u, el = rl < nrows ? irp[rl + 1] : 0u;
    unsigned long_rows = __ballot_sync(0xffffffffu, el - sl > kVlaLong);
    while (long_rows) {
    const int k = __ffs(long_rows) - 1;
    long_rows &= long_rows - 1;
    const int64_t r = r0 + k;
    const uint32_t s = __shfl_sync(0xffffffffu, sl, k), e = __shfl_sync(0xffffffffu, el, k);
    T acc = T(0);
    uint32_t n = s + uint32_t(lane);  // next entry of logical lane `lane`
    for (uint32_t c0 = s; c0 < e; c0 += kVlaLong) {
      const uint32_t c1 = min(e, c0 + kVlaLong);
      T p[kVlaLong / 32];
#pragma unroll
      for (int u = 0; u < int(kVlaLong / 32); ++u) {
        const uint32_t j = c0 + uint32_t(lane) + 32u * uint32_t(u);
        p[u] = j < c1 ? mul_rn(ld_stream(av + j), ldx(xb + ld_stream(aj + j))) : T(0);
      }
#pragma unroll
      for (int u = 0; u < int(kVlaLong / 32); ++u) buf[lane + 32 * u] = p[u];
      __syncwarp();
      if (uint32_t(lane) < L)
        for (; n < c1; n += L) acc = add_rn(acc, buf[n - c0]);
      __syncwarp();
    }
    acc = tree_reduce_warp(acc, width);
    if (lane == 0) y[r] = acc;
    }
  }
}

// Planned long-row vla path, two phases.  Phase 1 gathers the rounded
// products of every long row in 256-entry chunks spread over all warps
// (chunk_row: chunk -> long-row index, built by the plan).  Phase 2 folds
// each row per logical lane in order (one warp per row; chunks staged
// through shared memory, the next one prefetched), so a 50k-entry row costs a
// short sequential fold rather than ~200 gather round trips on one warp.
// Same products, same add order: bit-identical with csr_vla_warp_kernel.
template <typename T>
__global__ void __launch_bounds__(256)
csr_vla_products_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj, const T* __restrict__ av,
                        const T* __restrict__ x, int64_t col_base, const uint32_t* __restrict__ rows,
                        const uint32_t* __restrict__ chunk_pre, const uint32_t* __restrict__ chunk_row,
                        int64_t n_chunks, T* __restrict__ P) {
  const T* xb = x - col_base;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = warp; c < n_chunks; c += nwarps) {
    const uint32_t i = chunk_row[c];
    const uint32_t r = rows[i];
    const uint32_t s = irp[r], e = irp[r + 1];
    const uint32_t c0 = s + (uint32_t(c) - chunk_pre[i]) * kVlaLong, c1 = min(e, c0 + kVlaLong);
    T p[kVlaLong / 32];
#pragma unroll
    for (int u = 0; u < int(kVlaLong / 32); ++u) {
      const uint32_t j = c0 + uint32_t(lane) + 32u * uint32_t(u);
      p[u] = j < c1 ? mul_rn(ld_stream(av + j), ldx(xb + ld_stream(aj + j))) : T(0);
    }
#pragma unroll
    for (int u = 0; u < int(kVlaLong / 32); ++u) {
      const uint32_t j = c0 + uint32_t(lane) + 32u * uint32_t(u);
      if (j < c1) P[j] = p[u];
    }
  }
}

// Long rows' fold: one warp per row (longest rows first, see
// csr_vla_build).  The row's products stream through kVlaFoldDepth chunks
// held in registers, so a 50k-entry row's ~200 chunks do not each wait a
// DRAM round trip; each chunk is staged in shared memory and logical lane
// l < L adds its entries s+l, s+l+L, ... in order (csr_vla_warp_kernel's
// sequence, so bit-identical), then the tree over next_pow2(L) lanes.
constexpr int kVlaFoldDepth = 4;
template <typename T>
__global__ void __launch_bounds__(256)
csr_vla_fold_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ rows, int64_t n_long,
                    const T* __restrict__ P, T* __restrict__ y, int lanes, int width) {
  constexpr int PER = kVlaLong / 32;
  constexpr int D = kVlaFoldDepth;
  __shared__ T s_p[8][kVlaLong];
  const int lane = threadIdx.x & 31;
  T* buf = s_p[threadIdx.x >> 5];
  const uint32_t L = uint32_t(lanes);
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_long; i += nwarps) {
    const uint32_t r = rows[i];
    const uint32_t s = irp[r], e = irp[r + 1];
    const uint32_t nch = (e - s + kVlaLong - 1) / kVlaLong;
    T ring[D][PER];
    auto load = [&](T(&dst)[PER], uint32_t c) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const uint32_t j = s + c * kVlaLong + uint32_t(lane) + 32u * uint32_t(u);
        dst[u] = (c < nch && j < e) ? P[j] : T(0);
      }
    };
#pragma unroll
    for (int d = 0; d < D; ++d) load(ring[d], uint32_t(d));
    T acc = T(0);
    uint32_t n = s + uint32_t(lane);  // next entry of logical lane `lane`
    for (uint32_t cb = 0; cb < nch; cb += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const uint32_t c = cb + uint32_t(d);
        if (c >= nch) break;  // warp-uniform
        const uint32_t c0 = s + c * kVlaLong, c1 = min(e, c0 + kVlaLong);
#pragma unroll
        for (int u = 0; u < PER; ++u) buf[lane + 32 * u] = ring[d][u];
        __syncwarp();
        load(ring[d], c + D);  // refill: D chunks stay in flight
        if (uint32_t(lane) < L) {
          for (; n + 3 * L < c1; n += 4 * L) {  // loads ahead of the (ordered) adds
            const T q0 = buf[n - c0], q1 = buf[n + L - c0], q2 = buf[n + 2 * L - c0], q3 = buf[n + 3 * L - c0];
            acc = add_rn(add_rn(add_rn(add_rn(acc, q0), q1), q2), q3);
          }
          for (; n < c1; n += L) acc = add_rn(acc, buf[n - c0]);
        }
        __syncwarp();
      }
    }
    acc = tree_reduce_warp(acc, width);
    if (lane == 0) y[r] = acc;
  }
}

__global__ void vla_long_rows_kernel(const uint32_t* __restrict__ irp, int64_t nrows, uint32_t* __restrict__ rows,
                                     unsigned long long* __restrict__ n) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x)
    if (irp[r + 1] > irp[r] && irp[r + 1] - irp[r] > kVlaLong) rows[atomicAdd(n, 1ull)] = uint32_t(r);
}

__global__ void vla_chunk_count_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ rows,
                                       int64_t n_long, uint32_t* __restrict__ cnt) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_long; i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = rows[i];
    cnt[i] = (irp[r + 1] - irp[r] + kVlaLong - 1) / kVlaLong;
  }
}

__global__ void vla_chunk_row_kernel(const uint32_t* __restrict__ pre, const uint32_t* __restrict__ cnt,
                                     int64_t n_long, uint32_t* __restrict__ chunk_row) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_long; i += int64_t(gridDim.x) * blockDim.x)
    for (uint32_t k = 0; k < cnt[i]; ++k) chunk_row[pre[i] + k] = uint32_t(i);
}

template <typename T, bool SKIP_LONG>
__global__ void __launch_bounds__(256)
csr_vla_warp_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                    const T* __restrict__ av, const T* __restrict__ x, int64_t col_base,
                    T* __restrict__ y, int64_t nrows, int lanes, int width,
                    const uint32_t* __restrict__ list = nullptr) {  // list: rows to do (nrows of them)
  const T* xb = x - col_base;
  const int lane = threadIdx.x % width;
  const int rows_per_warp = 32 / width;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  // Uniform trip count per warp so the shuffles see every lane.
  for (int64_t base = warp * rows_per_warp; base < nrows; base += nwarps * rows_per_warp) {
    const int64_t ri = base + (threadIdx.x & 31) / width;
    const int64_t r = list && ri < nrows ? int64_t(list[ri]) : ri;
    uint32_t s = 0, e = 0;
    if (ri < nrows) {
      s = irp[r];
      e = irp[r + 1];
    }
    const bool mine = !SKIP_LONG || e <= s || e - s <= kVlaLong;  // longer rows: csr_vla_long_kernel
    T acc = T(0);
    if (lane < lanes && mine) {
      // The lane's entries j, j+L, j+2L, j+3L are loaded as one predicated
      // batch and added in that order (skipped slots add nothing), so a
      // short row costs one gather round trip instead of one per entry.
      const uint32_t L = uint32_t(lanes);
      for (uint32_t j = s + lane; j < e; j += 4 * L) {
        T p[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t jj = j + uint32_t(k) * L;
          p[k] = jj < e ? mul_rn(ld_stream(av + jj), ldx(xb + ld_stream(aj + jj))) : T(0);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (j + uint32_t(k) * L < e) acc = add_rn(acc, p[k]);
      }
    }
    acc = tree_reduce_warp(acc, width);
    if (lane == 0 && ri < nrows && mine) y[r] = (s == e) ? T(0) : acc;
  }
}

// Rows of <= 32 entries, one thread per row playing all W = next_pow2(L)
// logical lanes in registers (tile.cuh row_vla_csr; same adds, bit-exact).
// Longer rows are left to csr_vla_warp_kernel (list) and the two-phase path.
template <typename T, int W>
__global__ void __launch_bounds__(256)
csr_vla_short_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj, const T* __restrict__ av,
                     const T* __restrict__ x, int64_t col_base, T* __restrict__ y, int64_t nrows, int lanes) {
  const T* xb = x - col_base;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = __ldg(irp + r), e = __ldg(irp + r + 1);
    if (e - s > uint32_t(kExactLen)) continue;
    y[r] = e == s ? T(0) : row_vla_csr<T, W, true>(aj + s, av + s, int(e - s), xb, lanes);
  }
}

template <typename T>
__global__ void csr_vla_block_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                                     const T* __restrict__ av, const T* __restrict__ x, int64_t col_base,
                                     T* __restrict__ y, int64_t nrows, int lanes) {
  extern __shared__ unsigned char smem_raw[];
  T* red = reinterpret_cast<T*>(smem_raw);
  const T* xb = x - col_base;
  const int width = blockDim.x;  // next_pow2(lanes) > 32
  const int t = threadIdx.x;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const uint32_t s = irp[r], e = irp[r + 1];
    T acc = T(0);
    if (t < lanes)
      for (uint32_t j = s + t; j < e; j += uint32_t(lanes))
        acc = add_rn(acc, mul_rn(ld_stream(av + j), ldx(xb + ld_stream(aj + j))));
    red[t] = acc;
    __syncthreads();
    for (int w = width >> 1; w >= 32; w >>= 1) {
      if (t < w) red[t] = add_rn(red[t], red[t + w]);
      __syncthreads();
    }
    if (t < 32) {
      T v = red[t];
      v = tree_reduce_warp(v, 32);
      if (t == 0) y[r] = (s == e) ? T(0) : v;
    }
    __syncthreads();
  }
}

}  // namespace spmv

using namespace spmv;

struct spmv_csr_plan {
  int dtype = SPMV_F64;
  int64_t nrows = 0, ncols = 0, nnz = 0, ntiles = 0, tile = 2048;
  int exact_len = kExactLen;
  spmv_plan_config cfg = config_or_default(nullptr);  // as requested (auto fields unresolved)
  int64_t n_long = 0;     // rows over kExactLen (32): the tile kernels' long rows
  int64_t n_long_ws = 0;  // rows over exact_len: the warp-stream kernel's split rows
  // per-stream launch scratch: tile-span partials (head/tail), warp-stream
  // partials and range counter (StreamSlots: concurrent streams never share)
  mutable StreamSlots scratch;
  size_t off_head = 0, off_tail = 0, off_ws_head = 0, off_ws_tail = 0, off_ws_ctr = 0;
  mutable StreamSlots vla_scratch;  // two-phase vla product buffer (nnz values), per stream
  std::mutex build_mu;              // lazily built parts (vla lists, host staging, maxcol)
  HostPipe host;                    // host-buffer products (hostpipe.cuh)
  bool tma_hint = false;
  DevBuf row_lo, cnt;
  DevBuf span_row, span_t0, span_t1;
  int64_t n_span = 0;
  DevBuf maxcol;
  // host-buffer pipeline (spmv_csr_host): created on first use
  std::vector<uint32_t> h_row_lo;
  std::vector<int64_t> h_maxcol_prefix;
  int groups = 1;                    // consumer groups per tile CTA (csr_tile_kernel G)
  bool long_scratch = true;          // kernels with long-row scratch (false: plan has no long rows)
  // planned vla path: rows over kVlaLong entries, their 256-entry chunks and
  // a product buffer (built on the first spmv_csr_vla_planned call)
  bool vla_built = false;
  int64_t vla_n = 0, vla_chunks = 0;
  DevBuf vla_rows, vla_pre, vla_chunk_row;
  int64_t vla_n_mid = 0;  // rows of 33..kVlaLong entries (list for csr_vla_warp_kernel)
  DevBuf vla_mid;
  int grid_bulk = 0, grid_direct = 0;  // G-group TMA kernel / single-group kernel
  // warp-stream path (wstream.cuh) for plans with long rows: whole-matrix
  // launches only; tile ranges (halo split, host pipeline) keep the tiles
  bool ws = false;
  bool has_empty = false;
  // panel path (panel.cuh) for long rows with random columns: whole-matrix
  // launches; the short rows run as their own CSR (sub plan, y via srow)
  bool panel = false;
  int64_t pn_long = 0, pn_entries = 0, pn_seg = 0, pn_ctas = 0, pn_items = 0, pn_short = 0, pn_short_nnz = 0;
  DevBuf pn_lrow, pn_ptr, pn_col, pn_val, pn_flag, pn_rseg, pn_cta_item, pn_item_panel, pn_item_end, pn_task_begin,
      pn_task_seg0;
  DevBuf pn_srow, pn_scol, pn_sval;  // short rows by length class (ShortEll)
  ShortEll pn_ell;
  const void* pn_aj = nullptr;  // the arrays the panel copy was made from: other arrays take the ws path
  const void* pn_av = nullptr;
  size_t off_part = 0;
  int64_t ws_nwarps = 0, ws_nranges = 0, ws_n_span = 0;
  int64_t ws_ranges_per_warp = 8;
  DevBuf ws_bounds, ws_row0, ws_span_row, ws_span_w0, ws_span_w1;
};

// (tile, groups, long-row scratch) triples with compiled kernels.  The
// short-only variants (LF = 0) serve plans without long rows.
#define SPMV_CSR_CONFIGS(X)                                                                                  \
  X(1024, 1, 1) X(2048, 1, 1) X(4096, 1, 1) X(1024, 3, 1) X(2048, 3, 1) X(2048, 3, 0) X(2304, 1, 1)        \
  X(2304, 3, 0) X(1664, 1, 1) X(1664, 4, 0)
static bool csr_config_known(int64_t tile, int groups, bool long_rows) {
#define X(TL, GR, LF) \
  if (tile == TL && groups == GR && long_rows == bool(LF)) return true;
  SPMV_CSR_CONFIGS(X)
#undef X
  return false;
}

template <typename K>
static int csr_ctas_per_sm(K kernel, int threads, size_t smem, int cap, int* per_sm) {
  SPMV_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  SPMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kernel, threads, smem));
  *per_sm = cap_ctas(*per_sm, cap);
  return SPMV_OK;
}

template <typename T, int TILE, int G, bool LONG>
static int csr_launch_config(spmv_csr_plan* p) {
  int per_sm = 0, per_sm1 = 0, rc;
  using S1 = CsrSmem<T, TILE, 1>;
  const int cta_cap = p->cfg.ctas_per_sm;
  if ((rc = csr_ctas_per_sm(csr_tile_kernel<T, true, TILE, G, LONG>, csr_cta_threads<G>(),
                            CsrSmem<T, TILE, G, LONG>::total, cta_cap, &per_sm)))
    return rc;
  if ((rc = csr_ctas_per_sm(csr_tile_kernel<T, true, TILE, 1>, kTileThreads, S1::total, cta_cap, &per_sm1))) return rc;
  if ((rc = csr_ctas_per_sm(csr_tile_kernel<T, false, TILE, 1>, kTileThreads, S1::total, cta_cap, &per_sm1))) return rc;
  const int64_t cap = int64_t(sm_count()) * per_sm, cap1 = int64_t(sm_count()) * per_sm1;
  p->grid_bulk = int(p->ntiles < cap ? p->ntiles : cap);
  p->grid_direct = int(p->ntiles < cap1 ? p->ntiles : cap1);
  return SPMV_OK;
}

template <typename T, int TILE, int G, bool LONG, int VW = 0>
static int csr_run_tiled(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av, const T* x,
                   int64_t col_base, T* y, cudaStream_t st, int64_t tb, int64_t te, bool fixup, int vla = 0,
                   int64_t y_split = INT64_MAX, int64_t y_gap = 0, const uint32_t* ymap = nullptr) {
  if (p->nrows == 0) return SPMV_OK;
  if (p->nnz == 0) {
    if (ymap) {
      const int64_t g = std::min<int64_t>((p->nrows + 255) / 256, int64_t(sm_count()) * 8);
      scatter_zero_kernel<T><<<unsigned(g), 256, 0, st>>>(ymap, p->nrows, y);
      SPMV_LAUNCH_CHECK();
      return SPMV_OK;
    }
    SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(T) * p->nrows, st));
    return SPMV_OK;
  }
  unsigned char* scr = nullptr;
  int rc = p->scratch.get(st, reinterpret_cast<void**>(&scr));
  if (rc) return rc;
  CsrParams<T> P;
  P.irp = irp;
  P.aj = aj;
  P.av = av;
  P.x = x;
  P.y = y;
  P.row_lo = p->row_lo.as<uint32_t>();
  P.head = reinterpret_cast<T*>(scr + p->off_head);
  P.tail = reinterpret_cast<T*>(scr + p->off_tail);
  P.nrows = p->nrows;
  P.nnz = p->nnz;
  P.col_base = col_base;
  P.ntiles = p->ntiles;
  P.tile_begin = tb;
  P.tile_end = te;
  P.exact_len = kExactLen;  // tile kernels: the tile extension and long-row scratch are sized for 32
  P.vla = vla;
  P.y_split = y_split;
  P.y_gap = y_gap;
  P.ymap = ymap;
  P.mode = (p->cfg.flags & 3) | (p->tma_hint ? 4 : 0) | ((p->cfg.flags & 4) ? 8 : 0);
  const bool aligned = (reinterpret_cast<uintptr_t>(aj) % 16 == 0) && (reinterpret_cast<uintptr_t>(av) % 16 == 0);
  P.n_bulk = aligned ? bulk_tiles(p->nnz, p->ntiles, TILE) : 0;
  const size_t smem1 = CsrSmem<T, TILE, 1>::total;
  if constexpr (VW > 0) {
    // vla instantiations are not touched by the plan's occupancy queries
    static bool attrs = [] {
      cudaFuncSetAttribute(csr_tile_kernel<T, false, TILE, 1, false, VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(CsrSmem<T, TILE, 1>::total));
      cudaFuncSetAttribute(csr_tile_kernel<T, true, TILE, 1, false, VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(CsrSmem<T, TILE, 1>::total));
      cudaFuncSetAttribute(csr_tile_kernel<T, true, TILE, G, LONG, VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(CsrSmem<T, TILE, G, LONG>::total));
      return true;
    }();
    (void)attrs;
  }
  if (!aligned) {
    const int64_t grid = std::min<int64_t>(p->grid_direct, te - tb);
    if (grid > 0) csr_tile_kernel<T, false, TILE, 1, VW == 0, VW><<<unsigned(grid), kTileThreads, smem1, st>>>(P);
  } else if (G == 1) {
    const int64_t grid = std::min<int64_t>(p->grid_bulk, te - tb);
    if (grid > 0) csr_tile_kernel<T, true, TILE, 1, LONG, VW><<<unsigned(grid), kTileThreads, smem1, st>>>(P);
  } else {
    // bulk tiles on the multi-group kernel, the (rare) tail tiles past
    // n_bulk on the single-group one
    const int64_t bulk_end = std::min<int64_t>(te, P.n_bulk);
    const int64_t grid = std::min<int64_t>(p->grid_bulk, bulk_end - tb);
    if (grid > 0)
      csr_tile_kernel<T, true, TILE, G, LONG, VW>
          <<<unsigned(grid), csr_cta_threads<G>(), CsrSmem<T, TILE, G, LONG>::total, st>>>(P);
    if (te > bulk_end) {
      CsrParams<T> Q = P;
      Q.tile_begin = std::max<int64_t>(tb, bulk_end);
      const int64_t g1 = std::min<int64_t>(p->grid_direct, te - Q.tile_begin);
      csr_tile_kernel<T, true, TILE, 1, VW == 0, VW><<<unsigned(g1), kTileThreads, smem1, st>>>(Q);
    }
  }
  SPMV_LAUNCH_CHECK();
  if (fixup && p->n_span > 0) {
    const int64_t g = std::min<int64_t>((p->n_span + 255) / 256, int64_t(sm_count()) * 8);
    csr_span_fixup_kernel<T><<<unsigned(g), 256, 0, st>>>(p->span_row.as<uint32_t>(), p->span_t0.as<uint32_t>(),
                                                          p->span_t1.as<uint32_t>(), p->n_span, P.head, P.tail, y);
    SPMV_LAUNCH_CHECK();
  }
  return SPMV_OK;
}

template <typename T>
static int csr_run_ws(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av, const T* x,
                      int64_t col_base, T* y, cudaStream_t st, const uint32_t* ymap = nullptr) {
  unsigned char* scr = nullptr;
  int rc = p->scratch.get(st, reinterpret_cast<void**>(&scr));
  if (rc) return rc;
  // empty rows: a memset of y (with a row map the caller zeroes them)
  if (p->has_empty && !ymap) SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(T) * p->nrows, st));
  WsParams<T> P;
  P.irp = irp;
  P.aj = aj;
  P.av = av;
  P.x = x;
  P.y = y;
  P.bounds = p->ws_bounds.as<uint32_t>();
  P.row0 = p->ws_row0.as<uint32_t>();
  P.head = reinterpret_cast<double*>(scr + p->off_ws_head);
  P.tail = reinterpret_cast<double*>(scr + p->off_ws_tail);
  P.exact_len = uint32_t(p->exact_len);
  P.nrows = p->nrows;
  P.col_base = col_base;
  P.nwarps = p->ws_nwarps;
  P.nranges = p->ws_nranges;
  P.ctr = reinterpret_cast<uint32_t*>(scr + p->off_ws_ctr);
  P.ymap = ymap;
  const int64_t grid = (p->ws_nwarps + kWsWarps - 1) / kWsWarps;
  csr_wstream_kernel<T><<<unsigned(grid), kWsWarps * 32, 0, st>>>(P);
  SPMV_LAUNCH_CHECK();
  if (p->ws_n_span > 0) {
    const int64_t g = std::min<int64_t>((p->ws_n_span + 7) / 8, int64_t(sm_count()) * 8);  // a warp per row
    ws_span_fixup_kernel<T><<<unsigned(g), 256, 0, st>>>(p->ws_span_row.as<uint32_t>(), p->ws_span_w0.as<uint32_t>(),
                                                         p->ws_span_w1.as<uint32_t>(), p->ws_n_span, P.head, P.tail, y);
    SPMV_LAUNCH_CHECK();
  }
  return SPMV_OK;
}

template <typename T>
static int csr_run_panel(const spmv_csr_plan* p, const T* x, int64_t col_base, int64_t x_len, T* y, cudaStream_t st);

template <typename T>
static int csr_run(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av, const T* x,
                   int64_t col_base, T* y, cudaStream_t st, int64_t tb = 0, int64_t te = -1, bool fixup = true,
                   int64_t y_split = INT64_MAX, int64_t y_gap = 0, const uint32_t* ymap = nullptr,
                   int64_t x_len = -1) {
  if (te < 0) te = p->ntiles;
  const bool whole = tb == 0 && te == p->ntiles && fixup && y_gap == 0;
  if (p->panel && whole && !ymap && aj == p->pn_aj && av == p->pn_av)
    return csr_run_panel<T>(p, x, col_base, x_len < 0 ? p->ncols - col_base : x_len, y, st);
  if (p->ws && whole) return csr_run_ws<T>(p, irp, aj, av, x, col_base, y, st, ymap);
#define X(TL, GR, LF)                                                          \
  if (p->tile == TL && p->groups == GR && p->long_scratch == bool(LF))          \
    return csr_run_tiled<T, TL, GR, bool(LF)>(p, irp, aj, av, x, col_base, y, st, tb, te, fixup, 0, y_split, y_gap, \
                                              ymap);
  SPMV_CSR_CONFIGS(X)
#undef X
  return fail(SPMV_INVALID_ARG, "no CSR kernel for tile %lld x %d groups", (long long)p->tile, p->groups);
}

// Panel path (panel.cuh): the short rows through the sub plan's tile kernel
// (y via the short-row map), the long rows' panel kernel, their partial sums.
template <typename T>
static int csr_run_panel(const spmv_csr_plan* p, const T* x, int64_t col_base, int64_t x_len, T* y,
                         cudaStream_t st) {
  unsigned char* scr = nullptr;
  int rc = p->scratch.get(st, reinterpret_cast<void**>(&scr));
  if (rc) return rc;
  if (p->pn_short > 0) {
    const int64_t gs = std::min<int64_t>((p->pn_short + 255) / 256, int64_t(sm_count()) * 16);
    short_ell_kernel<T><<<unsigned(gs), 256, 0, st>>>(p->pn_ell, p->pn_scol.as<uint32_t>(), p->pn_sval.as<T>(),
                                                      p->pn_srow.as<uint32_t>(), p->pn_short, x, col_base, y,
                                                      (p->cfg.flags & 4) != 0);
    SPMV_LAUNCH_CHECK();
  }
  if (p->pn_long == 0) return SPMV_OK;
  PanelParams<T> P;
  P.pcol = p->pn_col.as<uint16_t>();
  P.pval = p->pn_val.as<T>();
  P.pflag = p->pn_flag.as<uint8_t>();
  P.x = x;
  P.col_base = col_base;
  P.x_len = x_len;
  P.ncols = p->ncols;
  P.cta_item = p->pn_cta_item.as<uint32_t>();
  P.item_panel = p->pn_item_panel.as<uint32_t>();
  P.item_end = p->pn_item_end.as<uint32_t>();
  P.task_begin = p->pn_task_begin.as<uint32_t>();
  P.task_seg0 = p->pn_task_seg0.as<uint32_t>();
  P.part = reinterpret_cast<double*>(scr + p->off_part);
  csr_panel_kernel<T><<<unsigned(p->pn_ctas), kPanelWarps * 32, panel_smem_bytes<T>(), st>>>(P);
  SPMV_LAUNCH_CHECK();
  const int64_t g = std::min<int64_t>((p->pn_long * 8 + 255) / 256, int64_t(sm_count()) * 16);
  csr_panel_finish_kernel<T><<<unsigned(g), 256, 0, st>>>(p->pn_lrow.as<uint32_t>(), p->pn_ptr.as<uint32_t>(),
                                                          p->pn_rseg.as<uint32_t>(), p->pn_long, P.part, y);
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

// vla through the tile kernels (row-per-lane vla, tile.cuh row_vla_csr):
// plans without long rows whose tile configuration has vla instantiations
// (any lane count: rows of <= 32 entries never reach lanes past 32).
#define SPMV_CSR_VLA_CONFIGS(X) X(2304, 3, 0) X(1664, 4, 0) X(2048, 3, 0)
template <typename T>
static int csr_run_vla_tiles(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av,
                             const T* x, int64_t col_base, T* y, int lanes, cudaStream_t st, bool* done) {
  *done = false;
  if (p->n_long > 0 || p->long_scratch || lanes < 1) return SPMV_OK;
  // rows have <= 32 entries: lanes past 32 only add zero lanes (see tile.cuh)
  const int w = lanes <= 1 ? 1 : lanes <= 2 ? 2 : lanes <= 4 ? 4 : lanes <= 8 ? 8 : lanes <= 16 ? 16 : 32;
#define X(TL, GR, LF)                                                                                           \
  if (p->tile == TL && p->groups == GR && !p->long_scratch) {                                                    \
    *done = true;                                                                                               \
    switch (w) {                                                                                                \
      case 1: return csr_run_tiled<T, TL, GR, false, 1>(p, irp, aj, av, x, col_base, y, st, 0, p->ntiles, true, lanes); \
      case 2: return csr_run_tiled<T, TL, GR, false, 2>(p, irp, aj, av, x, col_base, y, st, 0, p->ntiles, true, lanes); \
      case 4: return csr_run_tiled<T, TL, GR, false, 4>(p, irp, aj, av, x, col_base, y, st, 0, p->ntiles, true, lanes); \
      case 8: return csr_run_tiled<T, TL, GR, false, 8>(p, irp, aj, av, x, col_base, y, st, 0, p->ntiles, true, lanes); \
      case 16: return csr_run_tiled<T, TL, GR, false, 16>(p, irp, aj, av, x, col_base, y, st, 0, p->ntiles, true, lanes); \
      default: return csr_run_tiled<T, TL, GR, false, 32>(p, irp, aj, av, x, col_base, y, st, 0, p->ntiles, true, lanes); \
    }                                                                                                           \
  }
  SPMV_CSR_VLA_CONFIGS(X)
#undef X
  return SPMV_OK;
}

// Host x -> host y product (spmv_csr_host): the generic pipeline of
// hostpipe.cuh with tile ranges as the unit of work.  Per-tile row ranges
// and largest columns come to the host once (under the build lock).
static int csr_host_prepare(spmv_csr_plan* p, const uint32_t* aj, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(p->build_mu);  // maxcol is shared with spmv_csr_plan_tile_info
  if (!p->h_row_lo.empty()) return SPMV_OK;
  int rc;
  if (!p->maxcol.ptr) {
    if ((rc = p->maxcol.alloc(4 * p->ntiles))) return rc;
    const int64_t g = std::min<int64_t>(p->ntiles, int64_t(sm_count()) * 8);
    tile_maxcol_kernel<<<unsigned(g), 256, 0, st>>>(aj, p->nnz, p->ntiles, p->tile, p->maxcol.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
  }
  std::vector<uint32_t> row_lo(p->ntiles + 1), mc(p->ntiles);
  SPMV_CUDA_TRY(cudaMemcpyAsync(row_lo.data(), p->row_lo.ptr, 4 * (p->ntiles + 1), cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(mc.data(), p->maxcol.ptr, 4 * p->ntiles, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<int64_t> prefix(p->ntiles);
  int64_t m = 0;
  for (int64_t t = 0; t < p->ntiles; ++t) prefix[t] = m = std::max<int64_t>(m, mc[t]);
  p->h_maxcol_prefix = std::move(prefix);
  p->h_row_lo = std::move(row_lo);
  return SPMV_OK;
}

template <typename T>
static int csr_host_run(spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av, const T* xh, T* yh,
                        int chunks, cudaStream_t st) {
  int rc = csr_host_prepare(p, aj, st);
  if (rc) return rc;
  const std::vector<int64_t> xb = host_x_chunks(p->ncols, chunks);
  const int nx = int(xb.size()) - 1;
  int64_t tb = 0;
  // after x chunk j has landed, run every tile whose columns are all below
  // xb[j + 1] (h_maxcol_prefix is non-decreasing): rows before the next
  // tile's first row are then final
  // plans whose whole-matrix kernel is not the tile kernel (panel,
  // warp-stream): the product runs once all of x is on the device
  const bool whole = p->panel || p->ws;
  auto compute = [&](int j, char* xd, char* yd, cudaStream_t s) -> int64_t {
    if (whole) {
      if (j < nx - 1) return 0;
      const int r = csr_run<T>(p, irp, aj, av, reinterpret_cast<const T*>(xd), 0, reinterpret_cast<T*>(yd), s, 0,
                               -1, true, INT64_MAX, 0, nullptr, p->ncols);
      return r ? -r : p->nrows;
    }
    const int64_t te = j == nx - 1 ? p->ntiles
                                   : int64_t(std::lower_bound(p->h_maxcol_prefix.begin(), p->h_maxcol_prefix.end(),
                                                              xb[j + 1]) - p->h_maxcol_prefix.begin());
    if (te > tb) {
      const int r = csr_run<T>(p, irp, aj, av, reinterpret_cast<const T*>(xd), 0, reinterpret_cast<T*>(yd), s, tb, te,
                               te == p->ntiles);
      if (r) return -r;
      tb = te;
    }
    return tb < p->ntiles ? int64_t(p->h_row_lo[tb]) : p->nrows;
  };
  return run_host_pipeline(p->host, xh, yh, sizeof(T), p->ncols, p->nrows, xb, compute, !whole && p->n_span > 0,
                           st);
}

static int count_async(unsigned long long* dev, unsigned long long* host, cudaStream_t st) {
  SPMV_CUDA_TRY(cudaMemcpyAsync(host, dev, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  return SPMV_OK;
}

// Warp-stream plan (wstream.cuh): chosen for matrices with long rows
// (spmv_plan_config.warp_stream overrides).  One range per resident warp.
static int csr_ws_build(spmv_csr_plan* p, const uint32_t* irp, cudaStream_t st) {
  const int mode = p->cfg.warp_stream;
  p->ws = (mode < 0 ? p->n_long_ws > 0 : mode > 0) || p->panel;  // the panel path falls back to it
  if (!p->ws) return SPMV_OK;
  int rc, per_sm = 0;
  unsigned long long* ctr = p->cnt.as<unsigned long long>();
  unsigned long long h = 0;
  const int64_t g_rows = std::min<int64_t>((p->nrows + 255) / 256, int64_t(sm_count()) * 16);
  SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
  count_empty_rows_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, p->nrows, ctr);
  SPMV_LAUNCH_CHECK();
  if ((rc = count_async(ctr, &h, st))) return rc;
  p->has_empty = h > 0;
  if (p->dtype == SPMV_F64)
    SPMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_wstream_kernel<double>, kWsWarps * 32, 0));
  else
    SPMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_wstream_kernel<float>, kWsWarps * 32, 0));
  per_sm = cap_ctas(per_sm, p->cfg.ctas_per_sm);
  // at least one chunk per warp: targets strictly increase, so no empty
  // range sits inside a split row
  // ranges: kWsRangesPerWarp per resident warp (dynamic hand-out evens out
  // uneven row work), at least one chunk each
  p->ws_nwarps = std::max<int64_t>(1, std::min<int64_t>(int64_t(sm_count()) * per_sm * kWsWarps, p->nnz / kWsChunk));
  p->ws_nranges =
      std::max<int64_t>(p->ws_nwarps, std::min<int64_t>(p->ws_nwarps * p->ws_ranges_per_warp, p->nnz / kWsChunk));
  const int64_t nr = p->ws_nranges;
  if ((rc = p->ws_bounds.alloc(4 * (nr + 1))) || (rc = p->ws_row0.alloc(4 * nr))) return rc;
  const int64_t gw = std::min<int64_t>((nr + 256) / 256, int64_t(sm_count()) * 16);
  ws_bounds_kernel<<<unsigned(gw), 256, 0, st>>>(irp, p->nrows, p->nnz, nr, p->exact_len,
                                                 p->ws_bounds.as<uint32_t>(), p->ws_row0.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
  ws_span_list_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, p->nrows, p->exact_len, p->ws_bounds.as<uint32_t>(),
                                                        nr, nullptr, nullptr, nullptr, ctr);
  SPMV_LAUNCH_CHECK();
  if ((rc = count_async(ctr, &h, st))) return rc;
  p->ws_n_span = int64_t(h);
  if (p->ws_n_span > 0) {
    if ((rc = p->ws_span_row.alloc(4 * p->ws_n_span)) || (rc = p->ws_span_w0.alloc(4 * p->ws_n_span)) ||
        (rc = p->ws_span_w1.alloc(4 * p->ws_n_span)))
      return rc;
    SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
    ws_span_list_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, p->nrows, p->exact_len, p->ws_bounds.as<uint32_t>(),
                                                          nr, p->ws_span_row.as<uint32_t>(),
                                                          p->ws_span_w0.as<uint32_t>(), p->ws_span_w1.as<uint32_t>(),
                                                          ctr);
    SPMV_LAUNCH_CHECK();
  }
  return SPMV_OK;
}

__global__ void long_entries_kernel(const uint32_t* __restrict__ irp, int64_t nrows, uint32_t thr,
                                    unsigned long long* __restrict__ n) {
  unsigned long long c = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t l = irp[r + 1] - irp[r];
    c += l > thr ? l : 0u;
  }
  for (int o = 16; o >= 1; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(n, c);
}

// panel_ptr[q] = first panel-major entry of panel q (skey sorted).
__global__ void panel_bounds_kernel(const uint32_t* __restrict__ skey, int64_t nl, int64_t npanels,
                                    uint32_t* __restrict__ pan_ptr) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= nl; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q1 = i < nl ? int64_t(skey[i]) : npanels;
    const int64_t q0 = i == 0 ? -1 : int64_t(skey[i - 1]);
    for (int64_t q = q0 + 1; q <= q1; ++q) pan_ptr[q] = uint32_t(i);
  }
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, int64_t n,
                                  int64_t limit, uint32_t* __restrict__ dst) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = idx[i] < limit ? src[idx[i]] : 0u;
}

__global__ void iota_u32_kernel(uint32_t* __restrict__ a, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    a[i] = uint32_t(i);
}

template <typename Fn>
static int cub_call(Fn fn, ScratchBuf& tmp, cudaStream_t st) {
  size_t bytes = 0;
  SPMV_CUDA_TRY(fn(static_cast<void*>(nullptr), bytes));
  if (bytes > tmp.bytes) {
    int rc = tmp.alloc(bytes, st);
    if (rc) return rc;
  }
  SPMV_CUDA_TRY(fn(tmp.ptr, bytes));
  return SPMV_OK;
}

// The panel path's structures (panel.cuh): long rows copied panel-major
// with segment flags and slots, the CTA / warp work cuts, and the short
// rows as their own CSR with a sub plan.  Device work with cub sorts and
// scans; a few small host round trips for the cuts.
template <typename T>
static int csr_panel_build(spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av, cudaStream_t st) {
  int rc;
  const int64_t n = p->nrows;
  const int sms = sm_count();
  const int64_t g = std::min<int64_t>((n + 255) / 256, int64_t(sms) * 16);
  ScratchBuf is_long, pos, tmp;
  if ((rc = is_long.alloc(4 * n, st)) || (rc = pos.alloc(4 * (n + 1), st))) return rc;
  split_rows_flags_kernel<<<unsigned(g), 256, 0, st>>>(irp, n, uint32_t(kExactLen), is_long.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  if ((rc = cub_call([&](void* t, size_t& b) {
         return cub::DeviceScan::ExclusiveSum(t, b, is_long.as<uint32_t>(), pos.as<uint32_t>(), n, st);
       }, tmp, st)))
    return rc;
  const int64_t nlong = p->n_long, ns = n - nlong;
  p->pn_long = nlong;
  p->pn_short = ns;
  if ((rc = p->pn_lrow.alloc(4 * std::max<int64_t>(nlong, 1))) || (rc = p->pn_srow.alloc(4 * std::max<int64_t>(ns, 1))))
    return rc;
  split_rows_scatter_kernel<<<unsigned(g), 256, 0, st>>>(is_long.as<uint32_t>(), pos.as<uint32_t>(), n,
                                                         p->pn_lrow.as<uint32_t>(), p->pn_srow.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  // row lengths -> lptr (long rows)
  ScratchBuf len, lptr;
  if ((rc = len.alloc(4 * (std::max(nlong, ns) + 1), st)) || (rc = lptr.alloc(4 * (nlong + 1), st))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(len.ptr, 0, 4 * (nlong + 1), st));
  if (nlong > 0) {
    const int64_t gg = std::min<int64_t>((nlong + 255) / 256, int64_t(sms) * 16);
    listed_lengths_kernel<<<unsigned(gg), 256, 0, st>>>(irp, p->pn_lrow.as<uint32_t>(), nlong, len.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
  }
  if ((rc = cub_call([&](void* t, size_t& bb) {
         return cub::DeviceScan::ExclusiveSum(t, bb, len.as<uint32_t>(), lptr.as<uint32_t>(), nlong + 1, st);
       }, tmp, st)))
    return rc;
  uint32_t hnl = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&hnl, lptr.as<uint32_t>() + nlong, 4, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t nl = hnl;
  p->pn_entries = nl;
  p->pn_short_nnz = p->nnz - nl;
  // the short rows (<= 32 entries) grouped by exact length, each class
  // stored column-major (entry j of every row of the class contiguous):
  // one thread per row, coalesced loads, the row summed left to right
  if (ns > 0) {
    ScratchBuf skey2, srow2;
    if ((rc = skey2.alloc(4 * ns, st)) || (rc = srow2.alloc(4 * ns, st))) return rc;
    const int64_t gs = std::min<int64_t>((ns + 255) / 256, int64_t(sms) * 16);
    listed_lengths_kernel<<<unsigned(gs), 256, 0, st>>>(irp, p->pn_srow.as<uint32_t>(), ns, len.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    if ((rc = cub_call([&](void* t, size_t& bb) {
           return cub::DeviceRadixSort::SortPairs(t, bb, len.as<uint32_t>(), skey2.as<uint32_t>(),
                                                  p->pn_srow.as<uint32_t>(), srow2.as<uint32_t>(), ns, 0, 6, st);
         }, tmp, st)))
      return rc;
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->pn_srow.ptr, srow2.ptr, 4 * ns, cudaMemcpyDeviceToDevice, st));
    ScratchBuf dcls;
    if ((rc = dcls.alloc(4 * (kShortClasses + 1), st))) return rc;
    panel_bounds_kernel<<<unsigned(gs), 256, 0, st>>>(skey2.as<uint32_t>(), ns, kShortClasses, dcls.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->pn_ell.cls, dcls.ptr, 4 * (kShortClasses + 1), cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    uint64_t acc = 0;
    for (int L = 0; L < kShortClasses; ++L) {
      p->pn_ell.ebase[L] = uint32_t(acc);
      acc += uint64_t(L) * (p->pn_ell.cls[L + 1] - p->pn_ell.cls[L]);
    }
    if ((rc = p->pn_scol.alloc(4 * std::max<uint64_t>(acc, 1))) || (rc = p->pn_sval.alloc(sizeof(T) * std::max<uint64_t>(acc, 1))))
      return rc;
    short_ell_fill_kernel<T><<<unsigned(gs), 256, 0, st>>>(p->pn_ell, irp, aj, av, p->pn_srow.as<uint32_t>(), ns,
                                                            p->pn_scol.as<uint32_t>(), p->pn_sval.as<T>());
    SPMV_LAUNCH_CHECK();
  }
  if (nlong == 0) return SPMV_OK;
  // long entries: (panel, long-entry index), stable sort by panel
  const int64_t npanels = (p->ncols + kPanelCols - 1) / kPanelCols;
  int end_bit = 1;
  while (end_bit < 32 && (int64_t(1) << end_bit) < npanels) ++end_bit;
  ScratchBuf key, skey, val, perm, erow, eidx;
  if ((rc = key.alloc(4 * nl, st)) || (rc = skey.alloc(4 * nl, st)) || (rc = val.alloc(4 * nl, st)) ||
      (rc = perm.alloc(4 * nl, st)) || (rc = erow.alloc(4 * nl, st)) || (rc = eidx.alloc(4 * nl, st)))
    return rc;
  const int64_t gl = std::min<int64_t>((nlong * 32 + 255) / 256, int64_t(sms) * 16);
  panel_expand_kernel<<<unsigned(gl), 256, 0, st>>>(irp, aj, p->pn_lrow.as<uint32_t>(), lptr.as<uint32_t>(), nlong,
                                                    key.as<uint32_t>(), val.as<uint32_t>(), erow.as<uint32_t>(),
                                                    eidx.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  if ((rc = cub_call([&](void* t, size_t& b) {
         return cub::DeviceRadixSort::SortPairs(t, b, key.as<uint32_t>(), skey.as<uint32_t>(), val.as<uint32_t>(),
                                                perm.as<uint32_t>(), nl, 0, end_bit, st);
       }, tmp, st)))
    return rc;
  // panel-major copy (padded: the kernel loads whole 8-entry groups)
  const int64_t pad = 32 * kPanelK + 8;
  if ((rc = p->pn_col.alloc(2 * (nl + pad))) || (rc = p->pn_val.alloc(sizeof(T) * (nl + pad)))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(p->pn_col.ptr, 0, 2 * (nl + pad), st));
  SPMV_CUDA_TRY(cudaMemsetAsync(p->pn_val.ptr, 0, sizeof(T) * (nl + pad), st));
  ScratchBuf flag, seg_of;
  if ((rc = flag.alloc(4 * nl, st)) || (rc = seg_of.alloc(4 * (nl + 1), st))) return rc;
  const int64_t ge = std::min<int64_t>((nl + 255) / 256, int64_t(sms) * 32);
  panel_gather_kernel<T><<<unsigned(ge), 256, 0, st>>>(skey.as<uint32_t>(), perm.as<uint32_t>(), erow.as<uint32_t>(),
                                                       eidx.as<uint32_t>(), aj, av, nl, p->pn_col.as<uint16_t>(),
                                                       p->pn_val.as<T>(), flag.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  if ((rc = cub_call([&](void* t, size_t& b) {
         return cub::DeviceScan::ExclusiveSum(t, b, flag.as<uint32_t>(), seg_of.as<uint32_t>(), nl, st);
       }, tmp, st)))
    return rc;
  if ((rc = p->pn_flag.alloc((nl + pad) / 8 + 8))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(p->pn_flag.ptr, 0, (nl + pad) / 8 + 8, st));
  panel_flag_bytes_kernel<<<unsigned(std::min<int64_t>((nl / 8 + 256) / 256, int64_t(sms) * 16)), 256, 0, st>>>(
      flag.as<uint32_t>(), nl, p->pn_flag.as<uint8_t>());
  SPMV_LAUNCH_CHECK();
  uint32_t hs[2];
  SPMV_CUDA_TRY(cudaMemcpyAsync(&hs[0], seg_of.as<uint32_t>() + nl - 1, 4, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(&hs[1], flag.as<uint32_t>() + nl - 1, 4, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t nseg = int64_t(hs[0]) + hs[1];
  p->pn_seg = nseg;
  // per segment its long row; per long row its segment count -> partial ptr
  ScratchBuf seg_row, row_cnt, order, iota;
  if ((rc = seg_row.alloc(4 * nseg, st)) || (rc = row_cnt.alloc(4 * (nlong + 1), st)) ||
      (rc = order.alloc(4 * nseg, st)) || (rc = iota.alloc(4 * nseg, st)) || (rc = p->pn_ptr.alloc(4 * (nlong + 1))) ||
      (rc = p->pn_rseg.alloc(4 * nseg)))
    return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(row_cnt.ptr, 0, 4 * (nlong + 1), st));
  panel_segments_kernel<<<unsigned(ge), 256, 0, st>>>(flag.as<uint32_t>(), seg_of.as<uint32_t>(), perm.as<uint32_t>(),
                                                      erow.as<uint32_t>(), nl, seg_row.as<uint32_t>(),
                                                      row_cnt.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  if ((rc = cub_call([&](void* t, size_t& b) {
         return cub::DeviceScan::ExclusiveSum(t, b, row_cnt.as<uint32_t>(), p->pn_ptr.as<uint32_t>(), nlong + 1, st);
       }, tmp, st)))
    return rc;
  const int64_t gsg = std::min<int64_t>((nseg + 255) / 256, int64_t(sms) * 16);
  iota_u32_kernel<<<unsigned(gsg), 256, 0, st>>>(iota.as<uint32_t>(), nseg);
  SPMV_LAUNCH_CHECK();
  int row_bits = 1;
  while (row_bits < 32 && (int64_t(1) << row_bits) < nlong) ++row_bits;
  ScratchBuf srow_key;
  if ((rc = srow_key.alloc(4 * nseg, st))) return rc;
  if ((rc = cub_call([&](void* t, size_t& b) {
         return cub::DeviceRadixSort::SortPairs(t, b, seg_row.as<uint32_t>(), srow_key.as<uint32_t>(),
                                                iota.as<uint32_t>(), order.as<uint32_t>(), nseg, 0, row_bits, st);
       }, tmp, st)))
    return rc;
  // row-major segment list (rseg): the sorted order itself
  SPMV_CUDA_TRY(cudaMemcpyAsync(p->pn_rseg.ptr, order.ptr, 4 * nseg, cudaMemcpyDeviceToDevice, st));
  // CTA cuts: equal entry counts, moved to segment starts
  std::vector<uint32_t> pan_ptr(npanels + 1);
  {
    ScratchBuf dp;
    if ((rc = dp.alloc(4 * (npanels + 1), st))) return rc;
    panel_bounds_kernel<<<unsigned(ge), 256, 0, st>>>(skey.as<uint32_t>(), nl, npanels, dp.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaMemcpyAsync(pan_ptr.data(), dp.ptr, 4 * (npanels + 1), cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  }
  auto snap = [&](std::vector<uint32_t>& pos, const std::vector<uint32_t>& lim) -> int {
    const int64_t m = int64_t(pos.size());
    ScratchBuf dpos, dlim;
    int r2;
    if ((r2 = dpos.alloc(4 * m, st)) || (r2 = dlim.alloc(4 * m, st))) return r2;
    SPMV_CUDA_TRY(cudaMemcpyAsync(dpos.ptr, pos.data(), 4 * m, cudaMemcpyHostToDevice, st));
    SPMV_CUDA_TRY(cudaMemcpyAsync(dlim.ptr, lim.data(), 4 * m, cudaMemcpyHostToDevice, st));
    panel_snap_kernel<<<unsigned(std::min<int64_t>((m + 255) / 256, 1024)), 256, 0, st>>>(
        flag.as<uint32_t>(), dpos.as<uint32_t>(), m, dlim.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaMemcpyAsync(pos.data(), dpos.ptr, 4 * m, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    return SPMV_OK;
  };
  const int64_t C = std::max<int64_t>(1, std::min<int64_t>(sms, (nl + 4095) / 4096));
  std::vector<uint32_t> cut(C + 1), cut_lim(C + 1, uint32_t(nl));
  for (int64_t c = 0; c <= C; ++c) cut[c] = uint32_t(nl * c / C);
  if ((rc = snap(cut, cut_lim))) return rc;
  cut[0] = 0;
  cut[C] = uint32_t(nl);
  std::vector<uint32_t> cta_item(C + 1), item_panel, item_end, tb, tlim;
  for (int64_t c = 0; c < C; ++c) {
    cta_item[c] = uint32_t(item_panel.size());
    for (int64_t q = 0; q < npanels; ++q) {
      const uint32_t lo = std::max(cut[c], pan_ptr[q]), hi = std::min(cut[c + 1], pan_ptr[q + 1]);
      if (lo >= hi) continue;
      item_panel.push_back(uint32_t(q));
      item_end.push_back(hi);
      for (int w = 0; w < kPanelWarps; ++w) {
        tb.push_back(uint32_t(lo + (uint64_t(hi - lo) * w) / kPanelWarps));
        tlim.push_back(hi);
      }
    }
  }
  cta_item[C] = uint32_t(item_panel.size());
  if ((rc = snap(tb, tlim))) return rc;
  p->pn_ctas = C;
  p->pn_items = int64_t(item_panel.size());
  const int64_t nt = int64_t(tb.size());
  if ((rc = p->pn_cta_item.alloc(4 * (C + 1))) || (rc = p->pn_item_panel.alloc(4 * std::max<int64_t>(1, p->pn_items))) ||
      (rc = p->pn_item_end.alloc(4 * std::max<int64_t>(1, p->pn_items))) ||
      (rc = p->pn_task_begin.alloc(4 * std::max<int64_t>(1, nt))) ||
      (rc = p->pn_task_seg0.alloc(4 * std::max<int64_t>(1, nt))))
    return rc;
  SPMV_CUDA_TRY(cudaMemcpyAsync(p->pn_cta_item.ptr, cta_item.data(), 4 * (C + 1), cudaMemcpyHostToDevice, st));
  if (p->pn_items) {
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->pn_item_panel.ptr, item_panel.data(), 4 * p->pn_items, cudaMemcpyHostToDevice,
                                  st));
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->pn_item_end.ptr, item_end.data(), 4 * p->pn_items, cudaMemcpyHostToDevice, st));
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->pn_task_begin.ptr, tb.data(), 4 * nt, cudaMemcpyHostToDevice, st));
    gather_u32_kernel<<<unsigned(std::min<int64_t>((nt + 255) / 256, 1024)), 256, 0, st>>>(
        seg_of.as<uint32_t>(), p->pn_task_begin.as<uint32_t>(), nt, nl, p->pn_task_seg0.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
  }
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));  // temporaries are released on return
  return SPMV_OK;
}

// Plan analysis (once per matrix): long-row census, tile size, per-tile row
// ranges and the list of long rows spanning tiles.
static int csr_plan_build(spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const void* av,
                          cudaStream_t st) {
  const int64_t nrows = p->nrows;
  unsigned long long* ctr = p->cnt.as<unsigned long long>();
  unsigned long long h = 0;
  int rc;
  const int64_t g_rows = std::min<int64_t>((nrows + 255) / 256, int64_t(sm_count()) * 16);
  SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
  count_long_rows_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, nrows, kExactLen, ctr);
  SPMV_LAUNCH_CHECK();
  if ((rc = count_async(ctr, &h, st))) return rc;
  p->n_long = int64_t(h);
  p->n_long_ws = p->n_long;
  if (p->exact_len < kExactLen) {  // the warp-stream kernel's threshold
    SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
    count_long_rows_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, nrows, p->exact_len, ctr);
    SPMV_LAUNCH_CHECK();
    if ((rc = count_async(ctr, &h, st))) return rc;
    p->n_long_ws = int64_t(h);
  }
  // Long rows: 1024-entry tiles, 3 groups (2 CTAs/SM: six tiles in flight
  // hide the long-row gathers).  Otherwise G consumer groups share a G + 1
  // stage ring of kernels without long-row scratch, sized per row length
  // below (measured on the 27-point stencil and the 11-diagonal banded
  // matrix).
  if (p->n_long > 0) {
    p->tile = 1024;
    p->groups = 3;  // Zipf: 269 -> 276 GFLOP/s over one group (long-row phases overlap other groups' rows)
  } else if (p->nnz < 16 * p->nrows) {
    p->tile = 1664;  // short rows: 62 per group fill two warps; banded 801 -> 825
    p->groups = 4;
  } else {
    // stencil-like rows: the largest tile whose 4-stage ring still fits two
    // CTAs per SM (256^3: 1039 -> 1068); small matrices keep 2048-entry
    // tiles for more tiles per group (64^3: 436 vs 415)
    p->tile = p->nnz >= (int64_t(64) << 20) ? 2304 : 2048;
    p->groups = 3;
  }
  const int t = p->cfg.tile;
  if (t == 1024 || t == 1664 || t == 2048 || t == 2304 || t == 4096) {
    p->tile = t;
    p->groups = 1;
  }
  if (p->cfg.groups > 0) p->groups = p->cfg.groups;
  p->long_scratch = p->n_long > 0;
  if (!csr_config_known(p->tile, p->groups, p->long_scratch)) {
    p->long_scratch = true;  // the kernels with long-row scratch serve any matrix
    if (!csr_config_known(p->tile, p->groups, true)) {
      p->groups = 1;
      if (!csr_config_known(p->tile, 1, true)) p->tile = p->n_long > 0 ? 1024 : 2048;
    }
  }
  p->ntiles = (p->nnz + p->tile - 1) / p->tile;
  p->tma_hint = p->cfg.tma_hint < 0 ? p->n_long > 0 : p->cfg.tma_hint > 0;
  p->ws_ranges_per_warp = p->cfg.ranges_per_warp >= 1 && p->cfg.ranges_per_warp <= 64 ? p->cfg.ranges_per_warp : 8;
  const size_t vs = value_size(p->dtype);
  if ((rc = p->row_lo.alloc(4 * (p->ntiles + 1)))) return rc;
  const int64_t g_tiles = std::min<int64_t>((p->ntiles + 256) / 256, int64_t(sm_count()) * 16);
  csr_row_lo_kernel<<<unsigned(g_tiles), 256, 0, st>>>(irp, nrows, p->ntiles, p->tile, p->row_lo.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  if (p->n_long > 0) {
    // two passes: count, then fill (order is irrelevant: rows are independent)
    SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
    csr_span_list_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, nrows, kExactLen, p->tile, nullptr, nullptr,
                                                             nullptr, ctr);
    SPMV_LAUNCH_CHECK();
    if ((rc = count_async(ctr, &h, st))) return rc;
    p->n_span = int64_t(h);
    if (p->n_span > 0) {
      if ((rc = p->span_row.alloc(4 * p->n_span)) || (rc = p->span_t0.alloc(4 * p->n_span)) ||
          (rc = p->span_t1.alloc(4 * p->n_span)))
        return rc;
      SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
      csr_span_list_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, nrows, kExactLen, p->tile,
                                                               p->span_row.as<uint32_t>(), p->span_t0.as<uint32_t>(),
                                                               p->span_t1.as<uint32_t>(), ctr);
      SPMV_LAUNCH_CHECK();
    }
  }
  // panel path: rows over 32 entries holding at least half the entries of
  // a matrix whose x does not fit L1 (spmv_plan_config.panels overrides);
  // needs the column indices and values (copied panel-major)
  if (p->n_long > 0 && aj && av && p->cfg.panels != 0) {
    SPMV_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8, st));
    long_entries_kernel<<<unsigned(g_rows), 256, 0, st>>>(irp, nrows, uint32_t(kExactLen), ctr);
    SPMV_LAUNCH_CHECK();
    if ((rc = count_async(ctr, &h, st))) return rc;
    p->panel = p->cfg.panels > 0 || (2 * int64_t(h) >= p->nnz && p->ncols >= 65536);
  }
  if ((rc = csr_ws_build(p, irp, st))) return rc;
  if (p->panel) {
    rc = p->dtype == SPMV_F64 ? csr_panel_build<double>(p, irp, aj, static_cast<const double*>(av), st)
                              : csr_panel_build<float>(p, irp, aj, static_cast<const float*>(av), st);
    if (rc) return rc;
    p->pn_aj = aj;
    p->pn_av = av;
    if (p->dtype == SPMV_F64)
      SPMV_CUDA_TRY(cudaFuncSetAttribute(csr_panel_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         panel_smem_bytes<double>()));
    else
      SPMV_CUDA_TRY(cudaFuncSetAttribute(csr_panel_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         panel_smem_bytes<float>()));
  }
  SlotLayout lay;  // per-stream launch scratch
  p->off_head = lay.add(vs * p->ntiles);
  p->off_tail = lay.add(vs * p->ntiles);
  p->off_ws_head = lay.add(8 * p->ws_nranges);
  p->off_ws_tail = lay.add(8 * p->ws_nranges);
  p->off_ws_ctr = lay.add(8);
  p->off_part = lay.add(8 * p->pn_seg);
  p->scratch.bytes = lay.total;
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
#define X(TL, GR, LF)                                                                      \
  if (p->tile == TL && p->groups == GR && p->long_scratch == bool(LF))                        \
    return p->dtype == SPMV_F64 ? csr_launch_config<double, TL, GR, bool(LF)>(p)             \
                                : csr_launch_config<float, TL, GR, bool(LF)>(p);
  SPMV_CSR_CONFIGS(X)
#undef X
  return fail(SPMV_INVALID_ARG, "no CSR kernel for tile %lld x %d groups", (long long)p->tile, p->groups);
}

template <typename T>
static int csr_vla_split_launch(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av,
                                const T* x, int64_t col_base, T* y, int lanes, cudaStream_t st) {
  const int64_t cap = int64_t(sm_count()) * 16;
  const int64_t gs = std::min<int64_t>((p->nrows + 255) / 256, cap);
  switch (lanes <= 1 ? 1 : lanes <= 2 ? 2 : lanes <= 4 ? 4 : 8) {
    case 1: csr_vla_short_kernel<T, 1><<<unsigned(gs), 256, 0, st>>>(irp, aj, av, x, col_base, y, p->nrows, lanes); break;
    case 2: csr_vla_short_kernel<T, 2><<<unsigned(gs), 256, 0, st>>>(irp, aj, av, x, col_base, y, p->nrows, lanes); break;
    case 4: csr_vla_short_kernel<T, 4><<<unsigned(gs), 256, 0, st>>>(irp, aj, av, x, col_base, y, p->nrows, lanes); break;
    default: csr_vla_short_kernel<T, 8><<<unsigned(gs), 256, 0, st>>>(irp, aj, av, x, col_base, y, p->nrows, lanes);
  }
  SPMV_LAUNCH_CHECK();
  if (p->vla_n_mid > 0) {
    int width = 1;
    while (width < lanes) width <<= 1;
    const int64_t gm = std::min<int64_t>((p->vla_n_mid * width + 255) / 256, cap);
    csr_vla_warp_kernel<T, true><<<unsigned(gm), 256, 0, st>>>(irp, aj, av, x, col_base, y, p->vla_n_mid, lanes, width,
                                                               p->vla_mid.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
  }
  return SPMV_OK;
}

namespace spmv {
int debug_counts_csr(unsigned long long* out4) { return debug_read_tu(out4); }
}  // namespace spmv

extern "C" {

int spmv_csr_plan_create(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* row_pointers,
                         int exact_len, void* stream, spmv_csr_plan** out) {
  spmv_plan_config cfg = config_or_default(nullptr);
  cfg.exact_len = exact_len;
  return spmv_csr_plan_create_ex(dtype, nrows, ncols, nnz, row_pointers, nullptr, nullptr, &cfg, stream, out);
}

int spmv_csr_plan_config(const spmv_csr_plan* p, spmv_plan_config* out) {
  if (!p || !out) return fail(SPMV_INVALID_ARG, "NULL argument");
  *out = p->cfg;
  out->tile = int32_t(p->tile);
  out->groups = p->groups;
  out->exact_len = p->exact_len;
  out->warp_stream = p->ws ? 1 : 0;
  out->ranges_per_warp = int32_t(p->ws_ranges_per_warp);
  out->tma_hint = p->tma_hint ? 1 : 0;
  out->panels = p->panel ? 1 : 0;
  return SPMV_OK;
}

int spmv_csr_plan_create_ex(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* row_pointers,
                            const uint32_t* col_indices, const void* values, const spmv_plan_config* cfg,
                            void* stream, spmv_csr_plan** out) {
  if (!out) return fail(SPMV_INVALID_ARG, "spmv_csr_plan_create: out is NULL");
  if (cfg && cfg->version != SPMV_PLAN_CONFIG_VERSION)
    return fail(SPMV_INVALID_ARG, "spmv_plan_config version %d, expected %d", cfg->version, SPMV_PLAN_CONFIG_VERSION);
  int exact_len = cfg ? cfg->exact_len : 0;
  *out = nullptr;
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows < 0 || ncols < 0 || nnz < 0 || nnz > int64_t(UINT32_MAX) || nrows >= int64_t(UINT32_MAX))
    return fail(SPMV_INVALID_ARG, "bad CSR sizes nrows=%lld ncols=%lld nnz=%lld", (long long)nrows,
                (long long)ncols, (long long)nnz);
  if (!row_pointers) return fail(SPMV_INVALID_ARG, "row_pointers is NULL");
  if (exact_len <= 0 || exact_len > kExactLen) exact_len = kExactLen;  // tile extension covers 32
  cudaStream_t st = as_stream(stream);
  auto* p = new spmv_csr_plan();
  p->dtype = dtype;
  p->nrows = nrows;
  p->ncols = ncols;
  p->nnz = nnz;
  p->exact_len = exact_len;
  p->cfg = config_or_default(cfg);
  int rc = p->cnt.alloc(8);  // scratch counter
  if (!rc && nrows > 0 && nnz > 0) rc = csr_plan_build(p, row_pointers, col_indices, values, st);
  if (rc) {
    delete p;
    return rc;
  }
  *out = p;
  return SPMV_OK;
}

// Debug builds only (-DSPMV_PHASE_TIMING): read and reset the phase counters.
int spmv_debug_csr_phases(unsigned long long* out8) {
#ifdef SPMV_PHASE_TIMING
  SPMV_CUDA_TRY(cudaDeviceSynchronize());
  SPMV_CUDA_TRY(cudaMemcpyFromSymbol(out8, g_phase, sizeof(unsigned long long) * 8));
  unsigned long long z[8] = {0};
  SPMV_CUDA_TRY(cudaMemcpyToSymbol(g_phase, z, sizeof(z)));
  return SPMV_OK;
#else
  (void)out8;
  return fail(SPMV_UNSUPPORTED, "library built without SPMV_PHASE_TIMING");
#endif
}

int spmv_csr_plan_destroy(spmv_csr_plan* plan) {
  delete plan;
  return SPMV_OK;
}

int spmv_csr_plan_info(const spmv_csr_plan* p, int64_t* n_long_rows, int64_t* n_items, int64_t* launches) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (n_long_rows) *n_long_rows = p->n_long_ws;
  if (n_items) *n_items = p->tile;
  if (launches && p->panel) {
    *launches = (p->pn_short > 0 ? 1 : 0) + (p->pn_long > 0 ? 2 : 0);
  } else if (launches && p->ws)
    *launches = 1 + (p->ws_n_span > 0 ? 1 : 0);
  else if (launches)
    *launches = (p->nrows > 0 ? 1 : 0) + (p->n_span > 0 ? 1 : 0) +
                (p->groups > 1 && p->nnz > 0 && bulk_tiles(p->nnz, p->ntiles, p->tile) < p->ntiles ? 1 : 0);
  return SPMV_OK;
}

int spmv_csr_plan_groups(const spmv_csr_plan* p, int* groups) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (groups) *groups = p->groups;
  return SPMV_OK;
}

int spmv_csr_plan_path(const spmv_csr_plan* p, int* warp_stream, int64_t* nwarps) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (warp_stream) *warp_stream = p->panel ? 2 : p->ws ? 1 : 0;
  if (nwarps) *nwarps = p->panel ? p->pn_ctas * kPanelWarps : p->ws_nwarps;
  return SPMV_OK;
}

int spmv_csr_plan_tiles(const spmv_csr_plan* p, int64_t* ntiles, int64_t* tile) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (ntiles) *ntiles = p->ntiles;
  if (tile) *tile = p->tile;
  return SPMV_OK;
}

int spmv_csr_plan_tile_info(spmv_csr_plan* p, const uint32_t* aj, uint32_t* row_lo_host, uint32_t* maxcol_host,
                            void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (p->ntiles == 0) return SPMV_OK;
  cudaStream_t st = as_stream(stream);
  std::lock_guard<std::mutex> lock(p->build_mu);
  if (!p->maxcol.ptr) {
    int rc = p->maxcol.alloc(4 * p->ntiles);
    if (rc) return rc;
    const int64_t g = std::min<int64_t>(p->ntiles, int64_t(sm_count()) * 8);
    tile_maxcol_kernel<<<unsigned(g), 256, 0, st>>>(aj, p->nnz, p->ntiles, p->tile, p->maxcol.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
  }
  if (row_lo_host)
    SPMV_CUDA_TRY(cudaMemcpyAsync(row_lo_host, p->row_lo.ptr, 4 * (p->ntiles + 1), cudaMemcpyDeviceToHost, st));
  if (maxcol_host)
    SPMV_CUDA_TRY(cudaMemcpyAsync(maxcol_host, p->maxcol.ptr, 4 * p->ntiles, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  return SPMV_OK;
}

int spmv_csr_range(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const void* av, const void* x,
                   int64_t col_base, int64_t x_len, void* y, int64_t tile_begin, int64_t tile_end, int fixup,
                   void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (tile_begin < 0 || tile_end > p->ntiles || tile_begin > tile_end) return fail(SPMV_INVALID_ARG, "bad tile range");
  if (p->nrows == 0 || p->nnz == 0) return fail(SPMV_INVALID_ARG, "tile ranges need a non-empty matrix");
  if (x_len < 0 || col_base < 0) return fail(SPMV_DIMENSION_MISMATCH, "bad x window");
  cudaStream_t st = as_stream(stream);
  if (p->dtype == SPMV_F64)
    return csr_run<double>(p, irp, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base,
                           static_cast<double*>(y), st, tile_begin, tile_end, fixup != 0);
  return csr_run<float>(p, irp, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
                        static_cast<float*>(y), st, tile_begin, tile_end, fixup != 0);
}

int spmv_csr_gapped(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const void* av, const void* x,
                    int64_t col_base, int64_t x_len, void* y, int64_t y_split, int64_t y_gap, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (p->nrows == 0 || p->nnz == 0) return fail(SPMV_INVALID_ARG, "gapped products need a non-empty matrix");
  if (y_split < 0 || y_split > p->nrows || y_gap < 0) return fail(SPMV_INVALID_ARG, "bad y split / gap");
  // long rows would need the span fix-up to honour the gap; a warp-stream
  // choice without long rows (SPMV_CSR_WS=1) falls back to the tile kernel
  if (p->n_long > 0)
    return fail(SPMV_UNSUPPORTED, "gapped products serve plans without rows over %d entries", p->exact_len);
  if (x_len < 0 || col_base < 0) return fail(SPMV_DIMENSION_MISMATCH, "bad x window");
  cudaStream_t st = as_stream(stream);
  if (p->dtype == SPMV_F64)
    return csr_run<double>(p, irp, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base,
                           static_cast<double*>(y), st, 0, p->ntiles, true, y_split, y_gap);
  return csr_run<float>(p, irp, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
                        static_cast<float*>(y), st, 0, p->ntiles, true, y_split, y_gap);
}

int spmv_csr_host(spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const void* av, const void* x_host,
                  void* y_host, int chunks, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (!x_host || !y_host) return fail(SPMV_INVALID_ARG, "NULL host buffer");
  if (p->nrows == 0 || p->nnz == 0) return fail(SPMV_INVALID_ARG, "host pipeline needs a non-empty matrix");
  if (chunks <= 0) chunks = 16;
  if (chunks > 1024) chunks = 1024;
  if (chunks > p->ntiles) chunks = int(p->ntiles);
  cudaStream_t st = as_stream(stream);
  if (p->dtype == SPMV_F64)
    return csr_host_run<double>(p, irp, aj, static_cast<const double*>(av), static_cast<const double*>(x_host),
                                static_cast<double*>(y_host), chunks, st);
  return csr_host_run<float>(p, irp, aj, static_cast<const float*>(av), static_cast<const float*>(x_host),
                             static_cast<float*>(y_host), chunks, st);
}

int spmv_csr(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const void* av, const void* x,
             int64_t col_base, int64_t x_len, void* y, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (p->nrows && (!irp || !y)) return fail(SPMV_INVALID_ARG, "NULL pointer");
  if (p->nnz && (!aj || !av || !x)) return fail(SPMV_INVALID_ARG, "NULL pointer");
  if (x_len < 0 || col_base < 0) return fail(SPMV_DIMENSION_MISMATCH, "bad x window");
  cudaStream_t st = as_stream(stream);
  if (p->dtype == SPMV_F64)
    return csr_run<double>(p, irp, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base,
                           static_cast<double*>(y), st, 0, -1, true, INT64_MAX, 0, nullptr, x_len);
  return csr_run<float>(p, irp, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
                        static_cast<float*>(y), st, 0, -1, true, INT64_MAX, 0, nullptr, x_len);
}

// The planned vla path's row list: rows over kVlaLong entries, their chunk
// offsets (host prefix sum, once per plan) and chunk -> row map.
static int csr_vla_build(spmv_csr_plan* p, const uint32_t* irp, cudaStream_t st) {
  int rc;
  const int64_t g = std::min<int64_t>((p->nrows + 255) / 256, int64_t(sm_count()) * 16);
  DevBuf ctr;
  if ((rc = ctr.alloc(16))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 16, st));
  count_long_rows_kernel<<<unsigned(g), 256, 0, st>>>(irp, p->nrows, int(kVlaLong), ctr.as<unsigned long long>());
  SPMV_LAUNCH_CHECK();
  unsigned long long n = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&n, ctr.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  p->vla_n = int64_t(n);
  if (p->vla_n > 0) {
    if ((rc = p->vla_rows.alloc(4 * p->vla_n))) return rc;
    vla_long_rows_kernel<<<unsigned(g), 256, 0, st>>>(irp, p->nrows, p->vla_rows.as<uint32_t>(),
                                                       ctr.as<unsigned long long>() + 1);
    SPMV_LAUNCH_CHECK();
    // longest rows first: the fold runs one warp per row, so the longest
    // rows' sequential folds must start in the first wave (the list order
    // from the atomics is arbitrary; results do not depend on it)
    std::vector<uint32_t> rows(p->vla_n), h_irp(p->nrows + 1);
    SPMV_CUDA_TRY(cudaMemcpyAsync(rows.data(), p->vla_rows.ptr, 4 * p->vla_n, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaMemcpyAsync(h_irp.data(), irp, 4 * (p->nrows + 1), cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    std::sort(rows.begin(), rows.end(), [&](uint32_t a, uint32_t b) {
      const uint32_t la = h_irp[a + 1] - h_irp[a], lb = h_irp[b + 1] - h_irp[b];
      return la != lb ? la > lb : a < b;
    });
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->vla_rows.ptr, rows.data(), 4 * p->vla_n, cudaMemcpyHostToDevice, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (p->vla_n > 0) {
    DevBuf cnt;
    if ((rc = cnt.alloc(4 * p->vla_n)) || (rc = p->vla_pre.alloc(4 * (p->vla_n + 1)))) return rc;
    const int64_t gi = std::min<int64_t>((p->vla_n + 255) / 256, int64_t(sm_count()) * 16);
    vla_chunk_count_kernel<<<unsigned(gi), 256, 0, st>>>(irp, p->vla_rows.as<uint32_t>(), p->vla_n,
                                                          cnt.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    std::vector<uint32_t> h(p->vla_n), pre(p->vla_n + 1);
    SPMV_CUDA_TRY(cudaMemcpyAsync(h.data(), cnt.ptr, 4 * p->vla_n, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    pre[0] = 0;
    for (int64_t i = 0; i < p->vla_n; ++i) pre[i + 1] = pre[i] + h[i];
    p->vla_chunks = pre[p->vla_n];
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->vla_pre.ptr, pre.data(), 4 * (p->vla_n + 1), cudaMemcpyHostToDevice, st));
    if ((rc = p->vla_chunk_row.alloc(4 * p->vla_chunks))) return rc;
    p->vla_scratch.bytes = value_size(p->dtype) * p->nnz;  // product buffer, one per stream
    vla_chunk_row_kernel<<<unsigned(gi), 256, 0, st>>>(p->vla_pre.as<uint32_t>(), cnt.as<uint32_t>(), p->vla_n,
                                                        p->vla_chunk_row.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));  // cnt and the host vector go out of scope
  }
  {
    SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 8, st));
    len_class_list_kernel<<<unsigned(g), 256, 0, st>>>(irp, p->nrows, uint32_t(kExactLen), kVlaLong, nullptr,
                                                       ctr.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    unsigned long long m = 0;
    SPMV_CUDA_TRY(cudaMemcpyAsync(&m, ctr.ptr, 8, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    p->vla_n_mid = int64_t(m);
    if (p->vla_n_mid > 0) {
      if ((rc = p->vla_mid.alloc(4 * p->vla_n_mid))) return rc;
      SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 8, st));
      len_class_list_kernel<<<unsigned(g), 256, 0, st>>>(irp, p->nrows, uint32_t(kExactLen), kVlaLong,
                                                         p->vla_mid.as<uint32_t>(), ctr.as<unsigned long long>());
      SPMV_LAUNCH_CHECK();
      SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  p->vla_built = true;
  return SPMV_OK;
}

// long_mode: 0 no row over kVlaLong; 1 such rows, csr_vla_long_kernel
// takes them; 2 such rows, the caller runs the two-phase path for them.
static int csr_vla_launch(int dtype, int64_t nrows, int64_t nnz, const uint32_t* irp, const uint32_t* aj,
                          const void* av, const void* x, int64_t col_base, int64_t x_len, void* y, int lanes,
                          int long_mode, cudaStream_t st) {
  const bool long_rows = long_mode != 0;
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (lanes < 1) return fail(SPMV_INVALID_ARG, "lane count must be >= 1");
  if (lanes > 1024) return fail(SPMV_UNSUPPORTED, "vla CSR supports at most 1024 lanes, got %d", lanes);
  if (nrows < 0 || nnz < 0 || x_len < 0) return fail(SPMV_INVALID_ARG, "bad sizes");
  if (nrows == 0) return SPMV_OK;
  int width = 1;
  while (width < lanes) width <<= 1;
  const int64_t cap = int64_t(sm_count()) * 16;
  if (width <= 32) {
    const int tb = 256;
    int64_t grid = (nrows * width + tb - 1) / tb;
    if (grid > cap) grid = cap;
    int64_t grid_long = (nrows + tb - 1) / tb;  // a warp tests 32 rows at a time
    if (grid_long > cap) grid_long = cap;
    if (dtype == SPMV_F64) {
      if (long_rows)
        csr_vla_warp_kernel<double, true><<<unsigned(grid), tb, 0, st>>>(
            irp, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base,
            static_cast<double*>(y), nrows, lanes, width);
      else
        csr_vla_warp_kernel<double, false><<<unsigned(grid), tb, 0, st>>>(
            irp, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base,
            static_cast<double*>(y), nrows, lanes, width);
      if (long_mode == 1)
        csr_vla_long_kernel<double><<<unsigned(grid_long), tb, 0, st>>>(irp, aj, static_cast<const double*>(av),
                                                                       static_cast<const double*>(x), col_base,
                                                                       static_cast<double*>(y), nrows, lanes, width);
    } else {
      if (long_rows)
        csr_vla_warp_kernel<float, true><<<unsigned(grid), tb, 0, st>>>(
            irp, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
            static_cast<float*>(y), nrows, lanes, width);
      else
        csr_vla_warp_kernel<float, false><<<unsigned(grid), tb, 0, st>>>(
            irp, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
            static_cast<float*>(y), nrows, lanes, width);
      if (long_mode == 1)
        csr_vla_long_kernel<float><<<unsigned(grid_long), tb, 0, st>>>(irp, aj, static_cast<const float*>(av),
                                                                      static_cast<const float*>(x), col_base,
                                                                      static_cast<float*>(y), nrows, lanes, width);
    }
  } else {
    int64_t grid = nrows < cap ? nrows : cap;
    const size_t sm = value_size(dtype) * width;
    if (dtype == SPMV_F64)
      csr_vla_block_kernel<double><<<unsigned(grid), width, sm, st>>>(irp, aj, static_cast<const double*>(av),
                                                                       static_cast<const double*>(x), col_base,
                                                                       static_cast<double*>(y), nrows, lanes);
    else
      csr_vla_block_kernel<float><<<unsigned(grid), width, sm, st>>>(irp, aj, static_cast<const float*>(av),
                                                                      static_cast<const float*>(x), col_base,
                                                                      static_cast<float*>(y), nrows, lanes);
  }
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

int spmv_csr_vla(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* irp, const uint32_t* aj,
                 const void* av, const void* x, int64_t col_base, int64_t x_len, void* y, int lanes,
                 void* stream) {
  (void)ncols;
  return csr_vla_launch(dtype, nrows, nnz, irp, aj, av, x, col_base, x_len, y, lanes, 1, as_stream(stream));
}

// vla through the tile kernels only (plans without long rows); *done = 0
// when the plan has no such kernel.  COO plans call it for their
// row-pointer view (the view's plan carries the COO-order flag).
int spmvi_csr_vla_tiles(spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const void* av, const void* x,
                       int64_t col_base, void* y, int lanes, void* stream, int* done) {
  if (!p || !done) return fail(SPMV_INVALID_ARG, "NULL argument");
  *done = 0;
  if (p->nrows == 0 || p->nnz == 0) return SPMV_OK;
  bool d = false;
  cudaStream_t st = as_stream(stream);
  const int rc = p->dtype == SPMV_F64
                     ? csr_run_vla_tiles<double>(p, irp, aj, static_cast<const double*>(av),
                                                 static_cast<const double*>(x), col_base, static_cast<double*>(y), lanes,
                                                 st, &d)
                     : csr_run_vla_tiles<float>(p, irp, aj, static_cast<const float*>(av), static_cast<const float*>(x),
                                                col_base, static_cast<float*>(y), lanes, st, &d);
  *done = d ? 1 : 0;
  return rc;
}

int spmv_csr_vla_planned(spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const void* av,
                         const void* x, int64_t col_base, int64_t x_len, void* y, int lanes, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  cudaStream_t st = as_stream(stream);
  if (p->nrows > 0 && p->nnz > 0 && x_len >= 0 && col_base >= 0) {
    bool done = false;
    const int rc = p->dtype == SPMV_F64
                       ? csr_run_vla_tiles<double>(p, irp, aj, static_cast<const double*>(av),
                                                   static_cast<const double*>(x), col_base, static_cast<double*>(y),
                                                   lanes, st, &done)
                       : csr_run_vla_tiles<float>(p, irp, aj, static_cast<const float*>(av),
                                                  static_cast<const float*>(x), col_base, static_cast<float*>(y), lanes,
                                                  st, &done);
    if (done || rc) return rc;
  }
  // rows over kVlaLong entries are only possible when the plan saw long rows
  const bool long_rows = p->n_long > 0 || p->exact_len >= int(kVlaLong);
  if (!long_rows || lanes > 32 || lanes < 1)
    return csr_vla_launch(p->dtype, p->nrows, p->nnz, irp, aj, av, x, col_base, x_len, y, lanes, long_rows ? 1 : 0,
                          st);
  int rc;
  {
    std::lock_guard<std::mutex> lock(p->build_mu);
    if (!p->vla_built && (rc = csr_vla_build(p, irp, st))) return rc;
  }
  if (lanes <= 8) {
    // rows <= 32: one thread per row (all logical lanes in registers);
    // rows of 33..kVlaLong: sub-warp groups over the plan's list; longer:
    // the two-phase path below
    if ((rc = p->dtype == SPMV_F64
                  ? csr_vla_split_launch<double>(p, irp, aj, static_cast<const double*>(av),
                                                 static_cast<const double*>(x), col_base, static_cast<double*>(y),
                                                 lanes, st)
                  : csr_vla_split_launch<float>(p, irp, aj, static_cast<const float*>(av),
                                                static_cast<const float*>(x), col_base, static_cast<float*>(y), lanes,
                                                st)))
      return rc;
  } else if ((rc = csr_vla_launch(p->dtype, p->nrows, p->nnz, irp, aj, av, x, col_base, x_len, y, lanes, 2, st))) {
    return rc;
  }
  if (p->vla_n == 0) return SPMV_OK;
  int width = 1;
  while (width < lanes) width <<= 1;
  const int64_t cap = int64_t(sm_count()) * 16;
  const int64_t g1 = std::min<int64_t>((p->vla_chunks * 32 + 255) / 256, cap);
  const int64_t g2 = std::min<int64_t>((p->vla_n * 32 + 255) / 256, cap);
  const uint32_t* rows = p->vla_rows.as<uint32_t>();
  void* prod = nullptr;
  if ((rc = p->vla_scratch.get(st, &prod))) return rc;
  if (p->dtype == SPMV_F64) {
    double* P = static_cast<double*>(prod);
    csr_vla_products_kernel<double><<<unsigned(g1), 256, 0, st>>>(
        irp, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base, rows,
        p->vla_pre.as<uint32_t>(), p->vla_chunk_row.as<uint32_t>(), p->vla_chunks, P);
    csr_vla_fold_kernel<double><<<unsigned(g2), 256, 0, st>>>(irp, rows, p->vla_n, P, static_cast<double*>(y),
                                                               lanes, width);
  } else {
    float* P = static_cast<float*>(prod);
    csr_vla_products_kernel<float><<<unsigned(g1), 256, 0, st>>>(
        irp, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base, rows,
        p->vla_pre.as<uint32_t>(), p->vla_chunk_row.as<uint32_t>(), p->vla_chunks, P);
    csr_vla_fold_kernel<float><<<unsigned(g2), 256, 0, st>>>(irp, rows, p->vla_n, P, static_cast<float*>(y), lanes,
                                                              width);
  }
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

}  // extern "C"
