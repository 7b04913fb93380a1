// COO SpMV for sm_100a.
//
// Reference: spmv_coo_plain (kernels.py:56-66) is np.add.at(y, rows,
// values * x[cols]) on a zeroed y — per row, a strictly sequential sum in
// storage order that starts from +0.0.  spmv_coo_vla (kernels.py:104-140)
// walks each row in L-entry steps, tree-reduces every step and adds it once
// into y[row].
//
// Plain path — coo_tile_kernel, persistent, TMA-fed (tile.cuh): fixed
// 2048-entry tiles, so work per CTA does not depend on row lengths.  The
// row indices (plus 32 on each side), column indices and values of a tile
// are bulk-copied into a shared-memory ring; segments are found with a block
// scan; no atomics touch y.
//   * a row of <= 32 entries is owned by the tile holding its first entry;
//     one thread sums it left to right from +0.0 out of shared memory (the
//     32-entry extension covers rows crossing the tile end) => bit-exact
//     with np.add.at.  Both neighbouring tiles decide "short" from the same
//     32-entry windows, so they agree on the owner.
//   * longer rows: one warp per in-tile segment (vla-32 order); segments of
//     rows crossing tile boundaries leave carries that coo_fixup_kernel adds
//     in tile order (deterministic, within 1e-12).
//   * each tile zero-fills the empty rows before its row starts, so y needs
//     no separate memset pass.
// Rows must be non-decreasing; the plan makes a stable row-sorted copy when
// they are not (np.add.at order inside a row = storage order, kept).
#include <cub/cub.cuh>

#include "hostpipe.cuh"

#include <algorithm>
#include <type_traits>
#include <vector>

#include "tile.cuh"
#include "wstream.cuh"

namespace spmv {

template <typename T>
struct CooParams {
  const uint32_t* ai;
  const uint32_t* aj;
  const T* av;
  const T* x;
  T* y;
  uint32_t* head_row;
  uint32_t* tail_row;
  uint32_t* pass;
  T* head_val;
  T* tail_val;
  int64_t nrows, nnz, col_base, ntiles, n_bulk;
  int64_t tile_begin;  // first tile of the launch's tail range (tail-only launches)
  int mode;
  int vla;  // lanes L of a vla tile launch (template VW = next_pow2(L) > 0)
};

// Shared memory of a COO tile CTA with G consumer groups over G + 1 stages
// (see csr.cu): [0, 64) stage mbarriers, [64, 96) stage tickets, [96, 224)
// four counters per group, then one scan/long-row block per group, then the
// stage ring.
template <typename T, int TILE, int G = 1>
struct CooSmem {
  static constexpr int stages = G + 1;
  static constexpr size_t rows_bytes = align_up(sizeof(uint32_t) * (TILE + 2 * kExt), 128);
  static constexpr size_t cols_bytes = align_up(sizeof(uint32_t) * (TILE + kExt), 128);
  static constexpr size_t vals_bytes = align_up(sizeof(T) * (TILE + kExt), 128);
  static constexpr size_t stage_bytes = rows_bytes + cols_bytes + vals_bytes;
  // group block: starts | long segments | scan counts | long-row scratch
  static constexpr size_t starts_bytes = align_up(sizeof(uint16_t) * (TILE + 1), 128);
  // Multi-group kernels run only on plans without long runs (no segment is
  // ever queued), so their group blocks carry no long-row scratch.
  static constexpr bool long_rows = G == 1;
  static constexpr size_t long_bytes = long_rows ? align_up(sizeof(LongSeg) * max_long_segs<TILE>(), 128) : 0;
  // warp counts, their offsets, and the boundary-row extents [128], [129]
  static constexpr size_t counts_bytes = align_up(sizeof(int) * (2 * 64 + 2), 128);
  static constexpr size_t units_bytes = long_rows ? align_up(sizeof(LongUnit) * max_units<TILE>(), 128) : 0;
  static constexpr size_t upart_bytes = long_rows ? align_up(sizeof(T) * max_units<TILE>(), 128) : 0;
  static constexpr size_t spart_bytes = long_rows ? align_up(sizeof(T) * max_long_segs<TILE>(), 128) : 0;
  static constexpr size_t group_bytes =
      starts_bytes + long_bytes + counts_bytes + units_bytes + upart_bytes + spart_bytes;
  static constexpr size_t tickets_off = 64, counters_off = 96, groups_off = 256;
  static constexpr size_t header = groups_off + G * group_bytes;
  static constexpr size_t total = header + stages * stage_bytes;
  static_assert(TILE / 32 <= 64, "segment scan covers at most 64 warp counts");
  static_assert(stages <= 8, "mbarrier / ticket / counter slots");
};

template <int G> constexpr int coo_group_threads() { return G == 1 ? kTileThreads : 128; }
template <int G> constexpr int coo_min_blocks() { return G == 1 ? 3 : 1; }

// rows: tile-relative view, valid for k in [-kExt, TILE + kExt).
template <typename T, int TILE, int NT, bool LONG, int VW = 0>
__device__ void coo_process_tile(const CooParams<T>& P, int64_t t, const uint32_t* __restrict__ rows,
                                 const uint32_t* __restrict__ cols, T* __restrict__ vals, uint16_t* s_start,
                                 LongSeg* s_long, int* s_nseg, int* s_nlong, int* s_wcnt,
                                 const TileGroup<NT>& grp) {
  constexpr int R = TILE / NT;
  constexpr int W = NT / 32;
  static_assert(TILE % NT == 0, "rounds");
  const int tid = grp.tid, lane = tid & 31, warp = tid >> 5;
  const int64_t E0 = t * TILE;
  const int cnt_in = int(min(int64_t(TILE), P.nnz - E0));
  const int cnt_ext = int(min(int64_t(TILE + kExt), P.nnz - E0));
  const T* xb = P.x - P.col_base;

  // 2. segment heads, striped (round i, warp w covers entries
  //    [256 i + 32 w, +32)): ballots + a 64-entry warp scan give every head
  //    its position in entry order without shared-memory bank conflicts.
  unsigned bal[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int k = i * NT + tid;
    const bool h = k < cnt_in && (k == 0 || rows[k] != rows[k - 1]);
    bal[i] = __ballot_sync(0xffffffffu, h);
    if (lane == 0) s_wcnt[i * W + warp] = __popc(bal[i]);
  }
  grp.sync();
  if (warp == 0) {
    const int v0 = (2 * lane < R * W) ? s_wcnt[2 * lane] : 0;
    const int v1 = (2 * lane + 1 < R * W) ? s_wcnt[2 * lane + 1] : 0;
    int incl = v0 + v1;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const int excl = incl - v0 - v1;
    s_wcnt[64 + 2 * lane] = excl;
    s_wcnt[64 + 2 * lane + 1] = excl + v0;
    // How far the tile's first / last row extends into the 32-entry windows
    // before / after it: one ballot each instead of a serial scan.
    const unsigned bb = __ballot_sync(0xffffffffu, rows[-1 - lane] == rows[0]);
    const unsigned ba = __ballot_sync(0xffffffffu, rows[cnt_in + lane] == rows[cnt_in - 1]);
    if (lane == 0) {
      s_wcnt[128] = bb == 0xffffffffu ? kExt : __ffs(~bb) - 1;
      s_wcnt[129] = ba == 0xffffffffu ? kExt : __ffs(~ba) - 1;
    }
    if (lane == 31) {
      *s_nseg = incl;
      *s_nlong = 0;
      s_start[incl] = uint16_t(cnt_in);
      P.head_row[t] = kNoRow;
      P.tail_row[t] = kNoRow;
      P.pass[t] = 0;
    }
  }
  grp.sync();
  {
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < R; ++i)
      if ((bal[i] >> lane) & 1u)
        s_start[s_wcnt[64 + i * W + warp] + __popc(bal[i] & lt)] = uint16_t(i * NT + tid);
  }
  grp.sync();
  const int nseg = *s_nseg;
  // Many short rows (more segments than threads): issue the whole tile's
  // gathers entry-per-lane first (see tile.cuh form_products).
  const bool products = VW == 0 && (P.mode & 1) && nseg > NT;
  if (products) {
    form_products<T, NT>(cols, vals, cnt_ext, xb, tid);
    grp.sync();
  }

  // 3. one thread per segment: short owned rows summed left to right from
  //    +0.0 (np.add.at order); long ones queued; empty rows zero-filled.
  for (int s = tid; s < nseg; s += NT) {
    const int k0 = s_start[s], k1 = s_start[s + 1];
    const uint32_t r = rows[k0];
    const bool cont_before = (k0 == 0) && rows[-1] == r;
    const int before = cont_before ? s_wcnt[128] : 0;
    const int after = k1 == cnt_in ? s_wcnt[129] : 0;
    const int n = before + (k1 - k0) + after;
    const bool is_long = before == kExt || after == kExt || n > kExactLen;
    // Empty rows: zero-filled here by the tile owning the next row start
    // (no y pass) unless the plan saw empty rows and pre-zeroed y (mode bit
    // 3), which keeps long gaps off a single thread.
    if (!(P.mode & 8)) {
      if (!cont_before) {
        const int64_t prev = k0 > 0 ? int64_t(rows[k0 - 1]) : (E0 > 0 ? int64_t(rows[-1]) : int64_t(-1));
        for (int64_t q = prev + 1; q < int64_t(r); ++q) P.y[q] = T(0);
      }
      if (k1 == cnt_in && E0 + cnt_in == P.nnz)
        for (int64_t q = int64_t(r) + 1; q < P.nrows; ++q) P.y[q] = T(0);
    }
    if (LONG && is_long) {
      const int idx = atomicAdd(s_nlong, 1);
      LongSeg L;
      L.row = r;
      L.lo = uint32_t(k0);
      L.hi = uint32_t(k1);
      L.flags = (cont_before ? 1u : 0u) | ((after > 0) ? 2u : 0u) | (products ? 4u : 0u);
      L.s = L.e = 0;
      s_long[idx] = L;
    } else if (!cont_before) {
      if constexpr (VW >= 16)
        P.y[r] = row_vla_coo_wide<T, VW>(cols + k0, vals + k0, k1 + after - k0, xb, P.vla, P.vla > 32);
      else if constexpr (VW > 0)
        P.y[r] = row_vla_coo<T, VW>(cols + k0, vals + k0, k1 + after - k0, xb, P.vla);
      else
        // +0.0 seed: np.add.at accumulates into a zeroed y
        P.y[r] = products ? row_sum(vals + k0, k1 + after - k0, T(0))
                          : row_dot<T, true>(cols + k0, vals + k0, k1 + after - k0, xb, T(0));
    }
  }
  grp.sync();
}

// 4. long segments (out of line): units over all warps (vla-32 order inside
//    a unit); cross-tile parts go to the carry slots for coo_fixup_kernel.
template <typename T, int TILE, int NT>
__device__ __forceinline__ void coo_tile_long(int64_t t, const uint32_t* __restrict__ cols, const T* __restrict__ vals,
                                           const LongSeg* __restrict__ s_long, int nl, unsigned char* scratch,
                                           int* s_nunits, const T* __restrict__ xb, T* __restrict__ y,
                                           uint32_t* head_row, T* head_val, uint32_t* pass, uint32_t* tail_row,
                                           T* tail_val, bool warp_per_seg, const TileGroup<NT>& grp) {
  using S = CooSmem<T, TILE>;
  LongUnit* units = reinterpret_cast<LongUnit*>(scratch);
  T* unit_part = reinterpret_cast<T*>(scratch + S::units_bytes);
  T* seg_part = reinterpret_cast<T*>(scratch + S::units_bytes + S::upart_bytes);
  const bool products = s_long[0].flags & 4u;
  reduce_long_segments<T, TILE, NT>(cols, vals, s_long, nl, units, unit_part, s_nunits, seg_part, xb, products,
                                    warp_per_seg, grp);
  for (int i = grp.tid; i < nl; i += NT) {
    const LongSeg L = s_long[i];
    const T part = seg_part[i];
    const bool cb = L.flags & 1u, ca = L.flags & 2u;
    if (!cb && !ca) {
      y[L.row] = part;
    } else if (cb) {
      head_row[t] = L.row;
      head_val[t] = part;
      pass[t] = ca ? 1u : 0u;
    } else {
      tail_row[t] = L.row;
      tail_val[t] = part;
    }
  }
}

// G == 1: one 256-thread group over a double buffer.  G > 1: G groups of
// 128 threads over G + 1 stages (tile i of the CTA -> group i % G, stage
// i % (G + 1)), bulk tiles only; the host runs tail tiles with G == 1.
template <typename T, bool BULK, int TILE, int G, int VW = 0>
__global__ void __launch_bounds__(G * coo_group_threads<G>(), coo_min_blocks<G>())
coo_tile_kernel(const __grid_constant__ CooParams<T> P) {
  static_assert(G == 1 || BULK, "multi-group CTAs are TMA-fed");
  constexpr int NT = coo_group_threads<G>();
  extern __shared__ __align__(128) unsigned char smem[];
  using S = CooSmem<T, TILE, G>;
  constexpr int STAGES = S::stages;
  const int g = int(threadIdx.x) / NT;
  const TileGroup<NT> grp{int(threadIdx.x) % NT, G == 1 ? 0 : 1 + g};
  const int tid = grp.tid;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  volatile int* tickets = reinterpret_cast<volatile int*>(smem + S::tickets_off);
  int* s_nseg = reinterpret_cast<int*>(smem + S::counters_off) + 4 * g;
  int* s_nlong = s_nseg + 1;  // s_nlong[1]: long-row unit count
  unsigned char* gblock = smem + S::groups_off + size_t(g) * S::group_bytes;
  uint16_t* s_start = reinterpret_cast<uint16_t*>(gblock);
  LongSeg* s_long = reinterpret_cast<LongSeg*>(gblock + S::starts_bytes);
  int* s_wcnt = reinterpret_cast<int*>(gblock + S::starts_bytes + S::long_bytes);
  unsigned char* scratch = reinterpret_cast<unsigned char*>(s_wcnt) + S::counts_bytes;
  unsigned char* stages = smem + S::header;
  auto rows_of = [&](int s) { return reinterpret_cast<uint32_t*>(stages + s * S::stage_bytes); };
  auto cols_of = [&](int s) { return reinterpret_cast<uint32_t*>(stages + s * S::stage_bytes + S::rows_bytes); };
  auto vals_of = [&](int s) {
    return reinterpret_cast<T*>(stages + s * S::stage_bytes + S::rows_bytes + S::cols_bytes);
  };

  const int64_t n_bulk = BULK ? P.n_bulk : 0;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t mine_bulk = first < n_bulk ? (n_bulk - 1 - first) / stride + 1 : 0;
  const int64_t tail0 = max(n_bulk, P.tile_begin) + first;
  const int64_t mine_tail = G == 1 && tail0 < P.ntiles ? (P.ntiles - 1 - tail0) / stride + 1 : 0;
  auto issue = [&](int64_t i) {
    const int64_t t = first + i * stride;
    const int64_t E0 = t * TILE;
    const uint32_t cnt = uint32_t(min(int64_t(TILE + kExt), P.nnz - E0));
    const uint32_t cb = cnt & ~3u;  // bulk part: 16-byte multiples
    const uint32_t pre = t > 0 ? uint32_t(kExt) : 0u;
    const int s = int(i % STAGES);
    if (G > 1) tickets[s] = int(i);
    // the last tiles' 1..3 odd entries: plain copies, published by the
    // arrive below (release) like the bulk bytes by complete_tx
    for (uint32_t k = cb; k < cnt; ++k) {
      rows_of(s)[kExt + k] = P.ai[E0 + k];
      cols_of(s)[k] = P.aj[E0 + k];
      vals_of(s)[k] = P.av[E0 + k];
    }
    mbar_arrive_expect_tx(&bars[s], (cb + pre) * 4u + cb * (4u + uint32_t(sizeof(T))));
    if (cb + pre) bulk_g2s(rows_of(s) + (kExt - pre), P.ai + E0 - pre, (cb + pre) * 4u, &bars[s], (P.mode & 4) != 0);
    if (cb) {
      bulk_g2s(cols_of(s), P.aj + E0, cb * 4u, &bars[s], (P.mode & 4) != 0);
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
    if (i < mine_bulk) {
      s = int(i % STAGES);
      t = first + i * stride;
      // parity waits only tell the current phase from the previous one: with
      // G > 1 wait until tile i is the one issued into the stage (csr.cu)
      if (G > 1)
        while (tickets[s] != int(i)) __nanosleep(32);
      mbar_wait(&bars[s], uint32_t((i / STAGES) & 1));
#ifdef SPMV_DEBUG_CHECKS
      {  // the staged rows / columns / values are exactly the global ones
        const int64_t E0 = t * TILE;
        const int cnt = int(min(int64_t(TILE + kExt), P.nnz - E0));
        const int pre = t > 0 ? kExt : 0;
        for (int k = tid - pre; k < cnt; k += NT) {
          SPMV_DCHECK(rows_of(s)[kExt + k] == P.ai[E0 + k], 0);
          if (k >= 0) {
            SPMV_DCHECK(cols_of(s)[k] == P.aj[E0 + k], 0);
            SPMV_DCHECK(same_bits(vals_of(s)[k], P.av[E0 + k]), 0);
          }
        }
      }
#endif
    } else {
      t = tail0 + (i - mine_bulk) * stride;
      const int64_t E0 = t * TILE;
      const int cnt = int(min(int64_t(TILE + kExt), P.nnz - E0));
      for (int k = tid - kExt; k < cnt; k += NT) {
        const int64_t gk = E0 + k;
        if (gk >= 0) rows_of(0)[kExt + k] = P.ai[gk];
        if (k >= 0) {
          cols_of(0)[k] = P.aj[gk];
          vals_of(0)[k] = P.av[gk];
        }
      }
    }
    // Row slots the copy did not fill: the window before tile 0, past nnz.
    {
      const int64_t E0 = t * TILE;
      const int cnt_ext = int(min(int64_t(TILE + kExt), P.nnz - E0));
      uint32_t* rb = rows_of(s);
      if (t == 0)
        for (int k = tid; k < kExt; k += NT) rb[k] = kNoRow;
      for (int k = cnt_ext + tid; k < TILE + kExt; k += NT) rb[kExt + k] = kNoRow;
    }
    grp.sync();
    coo_process_tile<T, TILE, NT, S::long_rows, VW>(P, t, rows_of(s) + kExt, cols_of(s), vals_of(s), s_start, s_long,
                                                s_nseg, s_nlong, s_wcnt, grp);
    const int nl = S::long_rows ? *s_nlong : 0;
    if (S::long_rows && nl > 0)
      coo_tile_long<T, TILE, NT>(t, cols_of(s), vals_of(s), s_long, nl, scratch, s_nlong + 1, P.x - P.col_base, P.y,
                                 P.head_row, P.head_val, P.pass, P.tail_row, P.tail_val, (P.mode & 2) != 0, grp);
    grp.sync();  // stage s free
    if (BULK && tid == 0 && i + STAGES < mine_bulk) {
      fence_proxy_async();
      issue(i + STAGES);
    }
  }
}

// Cross-tile long rows: walk from the tile where the row starts (its tail
// slot) through the following tiles' head slots, adding in tile order.
template <typename T>
__global__ void coo_fixup_kernel(const CooParams<T> P) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < P.ntiles;
       t += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = P.tail_row[t];
    if (r == kNoRow) continue;
    T acc = P.tail_val[t];
    for (int64_t u = t + 1; u < P.ntiles && P.head_row[u] == r; ++u) {
      acc = add_rn(acc, P.head_val[u]);
      if (!P.pass[u]) break;
    }
    P.y[r] = acc;
  }
}

// ---- plan-time helpers ---------------------------------------------------
__global__ void rows_descending_kernel(const uint32_t* __restrict__ ai, int64_t nnz, int* __restrict__ flag) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x + 1; k < nnz; k += int64_t(gridDim.x) * blockDim.x)
    if (ai[k] < ai[k - 1]) {
      *flag = 1;
      return;
    }
}

__global__ void iota_kernel(uint32_t* __restrict__ v, int64_t n) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
    v[k] = uint32_t(k);
}

template <typename T>
__global__ void gather_triples_kernel(const uint32_t* __restrict__ perm, int64_t n, const uint32_t* __restrict__ aj,
                                      const T* __restrict__ av, uint32_t* __restrict__ aj_out,
                                      T* __restrict__ av_out) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t p = perm[k];
    aj_out[k] = aj[p];
    av_out[k] = av[p];
  }
}

__global__ void run_heads_kernel(const uint32_t* __restrict__ ai, int64_t nnz, uint32_t* __restrict__ head) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz; k += int64_t(gridDim.x) * blockDim.x)
    head[k] = (k == 0 || ai[k] != ai[k - 1]) ? 1u : 0u;
}

__global__ void run_scatter_kernel(const uint32_t* __restrict__ ai, int64_t nnz, const uint32_t* __restrict__ head,
                                   const uint32_t* __restrict__ pos, uint32_t* __restrict__ run_start,
                                   uint32_t* __restrict__ run_row) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz; k += int64_t(gridDim.x) * blockDim.x)
    if (head[k]) {
      run_start[pos[k]] = uint32_t(k);
      run_row[pos[k]] = ai[k];
    }
}

// ---- vla: L-entry steps per run, tree per step ----------------------------
// Runs longer than kVlaLong entries go to coo_vla_long_kernel (L <= 32).
constexpr uint32_t kVlaLong = 256;

// Planned long-run path, two phases.  Phase 1: a warp per 256-entry chunk
// of a long run computes the tree sum of every step whose first entry lies
// in the chunk (gathers for 8 sub-passes in flight) and stores step st of
// the run starting at a in S[a + st] (st < run length, so runs never
// collide and a run's step sums are contiguous).  Phase 2: a warp per long
// run folds its step sums in step order (kernels.py:129-137), 256 at a
// time through shared memory with the next chunk prefetched.
template <typename T>
__global__ void __launch_bounds__(256)
coo_vla_steps_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ runs,
                     const uint32_t* __restrict__ chunk_pre, const uint32_t* __restrict__ chunk_run, int64_t n_chunks,
                     const uint32_t* __restrict__ aj, const T* __restrict__ av, const T* __restrict__ x,
                     int64_t col_base, int lanes, int width, T* __restrict__ S) {
  constexpr int U = 8;
  const T* xb = x - col_base;
  const int lane = threadIdx.x & 31;
  const int W = width, G = 32 / width, sub = lane / W, l = lane % W;
  const uint32_t L = uint32_t(lanes);
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = warp; c < n_chunks; c += nwarps) {
    const uint32_t i = chunk_run[c], ri = runs[i];
    const uint32_t a = run_start[ri], b = run_start[ri + 1];
    const uint32_t e0 = a + (uint32_t(c) - chunk_pre[i]) * kVlaLong, e1 = min(b, e0 + kVlaLong);
    const uint32_t st_lo = (e0 - a + L - 1) / L, st_hi = (e1 - a + L - 1) / L;
    for (uint32_t st0 = st_lo; st0 < st_hi; st0 += uint32_t(U * G)) {
      T p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t st = st0 + uint32_t(u * G + sub);
        const uint32_t j = a + st * L + uint32_t(l);
        p[u] = (uint32_t(l) < L && st < st_hi && j < b) ? mul_rn(ld_stream(av + j), ldx(xb + ld_stream(aj + j)))
                                                       : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const T q = tree_reduce_warp(p[u], W);
        const uint32_t st = st0 + uint32_t(u * G + sub);
        if (l == 0 && st < st_hi) S[a + st] = q;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
coo_vla_fold_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ run_row,
                    const uint32_t* __restrict__ runs, int64_t n_long, const T* __restrict__ S, int lanes,
                    T* __restrict__ y, unsigned long long* __restrict__ steps_out) {
  constexpr int PER = kVlaLong / 32;
  __shared__ T s_q[8][kVlaLong];
  const int lane = threadIdx.x & 31;
  T* buf = s_q[threadIdx.x >> 5];
  const uint32_t L = uint32_t(lanes);
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long my_steps = 0;
  for (int64_t i = warp; i < n_long; i += nwarps) {
    const uint32_t ri = runs[i];
    const uint32_t a = run_start[ri], b = run_start[ri + 1];
    const uint32_t nsteps = (b - a + L - 1) / L;
    T cur[PER], nxt[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const uint32_t st = uint32_t(lane) + 32u * uint32_t(u);
      cur[u] = st < nsteps ? S[a + st] : T(0);
    }
    T yv = T(0);
    for (uint32_t c0 = 0; c0 < nsteps; c0 += kVlaLong) {
      const uint32_t c1 = min(nsteps, c0 + kVlaLong);
      if (c1 < nsteps) {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const uint32_t st = c1 + uint32_t(lane) + 32u * uint32_t(u);
          nxt[u] = st < nsteps ? S[a + st] : T(0);
        }
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) buf[lane + 32 * u] = cur[u];
      __syncwarp();
      if (lane == 0) {
        uint32_t k = 0;
        for (; k + 3 < c1 - c0; k += 4) {
          const T q0 = buf[k], q1 = buf[k + 1], q2 = buf[k + 2], q3 = buf[k + 3];
          yv = add_rn(add_rn(add_rn(add_rn(yv, q0), q1), q2), q3);
        }
        for (; k < c1 - c0; ++k) yv = add_rn(yv, buf[k]);
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < PER; ++u) cur[u] = nxt[u];
    }
    if (lane == 0) {
      y[run_row[ri]] = yv;
      my_steps += nsteps;
    }
  }
  if (steps_out && lane == 0 && my_steps) atomicAdd(steps_out, my_steps);
}

__global__ void vla_long_runs_kernel(const uint32_t* __restrict__ run_start, int64_t n_runs,
                                     uint32_t* __restrict__ runs, unsigned long long* __restrict__ n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_runs; i += int64_t(gridDim.x) * blockDim.x)
    if (run_start[i + 1] - run_start[i] > kVlaLong) {
      if (runs) runs[atomicAdd(n, 1ull)] = uint32_t(i);
      else atomicAdd(n, 1ull);
    }
}

__global__ void vla_run_chunks_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ runs,
                                      int64_t n_long, uint32_t* __restrict__ cnt) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_long; i += int64_t(gridDim.x) * blockDim.x)
    cnt[i] = (run_start[runs[i] + 1] - run_start[runs[i]] + kVlaLong - 1) / kVlaLong;
}

__global__ void vla_run_chunk_map_kernel(const uint32_t* __restrict__ pre, const uint32_t* __restrict__ cnt,
                                         int64_t n_long, uint32_t* __restrict__ chunk_run) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_long; i += int64_t(gridDim.x) * blockDim.x)
    for (uint32_t k = 0; k < cnt[i]; ++k) chunk_run[pre[i] + k] = uint32_t(i);
}

template <typename T, bool SKIP_LONG>
__global__ void __launch_bounds__(256)
coo_vla_warp_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ run_row, int64_t n_runs,
                    const uint32_t* __restrict__ aj, const T* __restrict__ av, const T* __restrict__ x,
                    int64_t col_base, T* __restrict__ y, int lanes, int width,
                    unsigned long long* __restrict__ steps_out,
                    const uint32_t* __restrict__ list = nullptr) {  // list: runs to do (n_runs of them)
  const T* xb = x - col_base;
  const int lane = threadIdx.x % width;
  const int rows_per_warp = 32 / width;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long my_steps = 0;
  for (int64_t bidx = warp * rows_per_warp; bidx < n_runs; bidx += nwarps * rows_per_warp) {
    const int64_t li = bidx + (threadIdx.x & 31) / width;
    const int64_t ri = list && li < n_runs ? int64_t(list[li]) : li;
    uint32_t a = 0, b = 0, row = 0;
    if (li < n_runs) {
      a = run_start[ri];
      b = run_start[ri + 1];
      row = run_row[ri];
    }
    const bool mine = !SKIP_LONG || b - a <= kVlaLong;  // longer runs: coo_vla_long_kernel
    const uint32_t nsteps = mine ? (b - a + uint32_t(lanes) - 1) / uint32_t(lanes) : 0u;
    unsigned max_steps = __reduce_max_sync(0xffffffffu, nsteps);
    T yv = T(0);
    // Four steps' products are loaded before their trees run (in step
    // order), so a short run costs one gather round trip.
    for (uint32_t st0 = 0; st0 < max_steps; st0 += 4) {
      T p[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t st = st0 + uint32_t(k);
        const uint32_t j = a + st * uint32_t(lanes) + uint32_t(lane);
        p[k] = (st < nsteps && lane < lanes && j < b) ? mul_rn(ld_stream(av + j), ldx(xb + ld_stream(aj + j)))
                                                      : T(0);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t st = st0 + uint32_t(k);
        if (st < max_steps) {  // warp-uniform: every lane joins the shuffles
          const T q = tree_reduce_warp(p[k], width);
          if (st < nsteps) yv = add_rn(yv, q);
        }
      }
    }
    if (lane == 0 && li < n_runs && mine) {
      y[row] = yv;
      my_steps += nsteps;
    }
  }
  if (steps_out) {
    for (int o = 16; o >= 1; o >>= 1) my_steps += __shfl_down_sync(0xffffffffu, my_steps, o);
    if ((threadIdx.x & 31) == 0 && my_steps) atomicAdd(steps_out, my_steps);
  }
}

// Runs of <= 32 entries, one thread per run playing all W = next_pow2(L)
// logical lanes in registers (tile.cuh row_vla_coo; same adds, bit-exact).
template <typename T, int W>
__global__ void __launch_bounds__(256)
coo_vla_short_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ run_row, int64_t n_runs,
                     const uint32_t* __restrict__ aj, const T* __restrict__ av, const T* __restrict__ x,
                     int64_t col_base, T* __restrict__ y, int lanes) {
  const T* xb = x - col_base;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_runs; i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t a = __ldg(run_start + i), b = __ldg(run_start + i + 1);
    if (b - a > uint32_t(kExactLen)) continue;
    y[__ldg(run_row + i)] = row_vla_coo<T, W, true>(aj + a, av + a, int(b - a), xb, lanes);
  }
}

template <typename T>
__global__ void coo_vla_block_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ run_row,
                                     int64_t n_runs, const uint32_t* __restrict__ aj, const T* __restrict__ av,
                                     const T* __restrict__ x, int64_t col_base, T* __restrict__ y, int lanes,
                                     unsigned long long* __restrict__ steps_out) {
  extern __shared__ unsigned char smem_raw[];
  T* red = reinterpret_cast<T*>(smem_raw);
  const T* xb = x - col_base;
  const int width = blockDim.x;
  const int t = threadIdx.x;
  unsigned long long my_steps = 0;
  for (int64_t ri = blockIdx.x; ri < n_runs; ri += gridDim.x) {
    const uint32_t a = run_start[ri], b = run_start[ri + 1];
    T yv = T(0);
    uint32_t nsteps = 0;
    for (uint32_t c0 = a; c0 < b; c0 += uint32_t(lanes), ++nsteps) {
      T p = T(0);
      if (t < lanes && c0 + t < b) p = mul_rn(ld_stream(av + c0 + t), ldx(xb + ld_stream(aj + c0 + t)));
      red[t] = p;
      __syncthreads();
      for (int w = width >> 1; w >= 32; w >>= 1) {
        if (t < w) red[t] = add_rn(red[t], red[t + w]);
        __syncthreads();
      }
      if (t < 32) {
        T v = tree_reduce_warp(red[t], 32);
        if (t == 0) yv = add_rn(yv, v);
      }
      __syncthreads();
    }
    if (t == 0) {
      y[run_row[ri]] = yv;
      my_steps += nsteps;
    }
  }
  if (steps_out && t == 0 && my_steps) atomicAdd(steps_out, my_steps);
}

}  // namespace spmv

using namespace spmv;

struct spmv_coo_plan {
  int dtype = SPMV_F64;
  int64_t nrows = 0, ncols = 0, nnz = 0;
  bool row_sorted = true;
  DevBuf sorted_ai, sorted_aj, sorted_av;  // only when the input rows were unsorted
  DevBuf run_start, run_row;
  int64_t n_runs = 0, n_long = 0, ntiles = 0, tile = 2048;
  spmv_plan_config cfg = config_or_default(nullptr);
  bool tma_hint = true;
  int64_t ws_ranges_per_warp = 8;
  // per-stream launch scratch (StreamSlots): tile boundary partials, warp-
  // stream partials and range counter, the vla step counter
  mutable StreamSlots scratch;
  size_t off_head_row = 0, off_tail_row = 0, off_pass = 0, off_head_val = 0, off_tail_val = 0;
  size_t off_ws_head = 0, off_ws_tail = 0, off_ws_ctr = 0, off_steps = 0;
  mutable StreamSlots vla_scratch;  // two-phase vla step sums (nnz values), per stream
  // column-panel path (csr.cu / panel.cuh) through a CSR view of the
  // row-sorted triples: whole-matrix products with the create-time arrays
  spmv_csr_plan* csr_view = nullptr;
  bool view_panel = false;  // the view runs the column-panel path (else the CSR tile kernel)
  DevBuf view_irp;
  const void* view_ai = nullptr;
  const void* view_aj = nullptr;
  const void* view_av = nullptr;
  HostPipe host;  // host-buffer products (hostpipe.cuh)
  ~spmv_coo_plan() { spmv_csr_plan_destroy(csr_view); }
  std::mutex build_mu;              // the lazily built vla lists
  int groups = 1;                // consumer groups per tile CTA (coo_tile_kernel G)
  int grid = 0, grid_direct = 0;  // G-group TMA kernel / single-group kernel
  // vla long runs (over kVlaLong entries): list, 256-entry chunk map and the
  // step-sum buffer, built on the first vla call that needs them
  bool vla_built = false;
  int64_t vla_n = 0, vla_chunks = 0;
  DevBuf vla_runs, vla_pre, vla_chunk_run;
  int64_t vla_n_mid = 0;  // runs of 33..kVlaLong entries (list for coo_vla_warp_kernel)
  DevBuf vla_mid;
  // warp-stream path (wstream.cuh) for plans with long runs
  bool ws = false;
  int64_t ws_nwarps = 0, ws_nranges = 0, ws_n_span = 0;
  DevBuf ws_bounds, ws_row0, ws_span_run, ws_span_w0, ws_span_w1;
};

static int coo_vla_build(spmv_coo_plan* p, cudaStream_t st) {
  int rc;
  const uint32_t* rs = p->run_start.as<uint32_t>();
  const int64_t g = std::min<int64_t>((p->n_runs + 255) / 256, int64_t(sm_count()) * 16);
  DevBuf ctr;
  if ((rc = ctr.alloc(16))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 16, st));
  vla_long_runs_kernel<<<unsigned(g), 256, 0, st>>>(rs, p->n_runs, nullptr, ctr.as<unsigned long long>());
  SPMV_LAUNCH_CHECK();
  unsigned long long n = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&n, ctr.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  p->vla_n = int64_t(n);
  if (p->vla_n > 0) {
    DevBuf cnt;
    if ((rc = p->vla_runs.alloc(4 * p->vla_n)) || (rc = cnt.alloc(4 * p->vla_n)) ||
        (rc = p->vla_pre.alloc(4 * (p->vla_n + 1))))
      return rc;
    vla_long_runs_kernel<<<unsigned(g), 256, 0, st>>>(rs, p->n_runs, p->vla_runs.as<uint32_t>(),
                                                       ctr.as<unsigned long long>() + 1);
    SPMV_LAUNCH_CHECK();
    {
      // longest runs first: the fold's single-lane step sum of a 50k-entry
      // run is the critical path; the atomics' list order is arbitrary
      std::vector<uint32_t> runs(p->vla_n), h_rs(p->n_runs + 1);
      SPMV_CUDA_TRY(cudaMemcpyAsync(runs.data(), p->vla_runs.ptr, 4 * p->vla_n, cudaMemcpyDeviceToHost, st));
      SPMV_CUDA_TRY(cudaMemcpyAsync(h_rs.data(), rs, 4 * (p->n_runs + 1), cudaMemcpyDeviceToHost, st));
      SPMV_CUDA_TRY(cudaStreamSynchronize(st));
      std::sort(runs.begin(), runs.end(), [&](uint32_t a, uint32_t b) {
        const uint32_t la = h_rs[a + 1] - h_rs[a], lb = h_rs[b + 1] - h_rs[b];
        return la != lb ? la > lb : a < b;
      });
      SPMV_CUDA_TRY(cudaMemcpyAsync(p->vla_runs.ptr, runs.data(), 4 * p->vla_n, cudaMemcpyHostToDevice, st));
      SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    }
    const int64_t gi = std::min<int64_t>((p->vla_n + 255) / 256, int64_t(sm_count()) * 16);
    vla_run_chunks_kernel<<<unsigned(gi), 256, 0, st>>>(rs, p->vla_runs.as<uint32_t>(), p->vla_n, cnt.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    std::vector<uint32_t> h(p->vla_n), pre(p->vla_n + 1);
    SPMV_CUDA_TRY(cudaMemcpyAsync(h.data(), cnt.ptr, 4 * p->vla_n, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    pre[0] = 0;
    for (int64_t i = 0; i < p->vla_n; ++i) pre[i + 1] = pre[i] + h[i];
    p->vla_chunks = pre[p->vla_n];
    SPMV_CUDA_TRY(cudaMemcpyAsync(p->vla_pre.ptr, pre.data(), 4 * (p->vla_n + 1), cudaMemcpyHostToDevice, st));
    if ((rc = p->vla_chunk_run.alloc(4 * p->vla_chunks))) return rc;
    p->vla_scratch.bytes = value_size(p->dtype) * p->nnz;
    vla_run_chunk_map_kernel<<<unsigned(gi), 256, 0, st>>>(p->vla_pre.as<uint32_t>(), cnt.as<uint32_t>(), p->vla_n,
                                                            p->vla_chunk_run.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  }
  {
    SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 8, st));
    len_class_list_kernel<<<unsigned(g), 256, 0, st>>>(rs, p->n_runs, uint32_t(kExactLen), kVlaLong, nullptr,
                                                       ctr.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    unsigned long long m = 0;
    SPMV_CUDA_TRY(cudaMemcpyAsync(&m, ctr.ptr, 8, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    p->vla_n_mid = int64_t(m);
    if (p->vla_n_mid > 0) {
      if ((rc = p->vla_mid.alloc(4 * p->vla_n_mid))) return rc;
      SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 8, st));
      len_class_list_kernel<<<unsigned(g), 256, 0, st>>>(rs, p->n_runs, uint32_t(kExactLen), kVlaLong,
                                                         p->vla_mid.as<uint32_t>(), ctr.as<unsigned long long>());
      SPMV_LAUNCH_CHECK();
      SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  p->vla_built = true;
  return SPMV_OK;
}

// (tile, groups) pairs with compiled kernels.
#define SPMV_COO_CONFIGS(X) X(1024, 1) X(2048, 1) X(1536, 1) X(1536, 6) X(1536, 7)
static bool coo_config_known(int64_t tile, int groups) {
#define X(TL, GR) if (tile == TL && groups == GR) return true;
  SPMV_COO_CONFIGS(X)
#undef X
  return false;
}

// irp[r] = first entry of row r in non-decreasing rows (binary search).
__global__ void row_bounds_kernel(const uint32_t* __restrict__ rows, int64_t nnz, int64_t nrows,
                                  uint32_t* __restrict__ irp) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= nrows; r += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (int64_t(rows[mid]) < r) lo = mid + 1; else hi = mid;
    }
    irp[r] = uint32_t(lo);
  }
}

__global__ void count_long_runs_kernel(const uint32_t* __restrict__ run_start, int64_t n_runs,
                                       unsigned long long* __restrict__ n_long) {
  unsigned long long c = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_runs; i += int64_t(gridDim.x) * blockDim.x)
    c += (run_start[i + 1] - run_start[i]) > uint32_t(kExactLen);
  for (int o = 16; o >= 1; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(n_long, c);
}

template <typename K>
static int coo_ctas_per_sm(K kernel, int threads, size_t smem, int cap, int* per_sm) {
  SPMV_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  SPMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kernel, threads, smem));
  *per_sm = cap_ctas(*per_sm, cap);
  return SPMV_OK;
}

template <typename T, int TILE, int G>
static int coo_launch_config(spmv_coo_plan* p) {
  using S1 = CooSmem<T, TILE, 1>;
  int per_sm = 0, per_sm1 = 0, rc;
  const int cta_cap = p->cfg.ctas_per_sm;
  if ((rc = coo_ctas_per_sm(coo_tile_kernel<T, true, TILE, G>, G * coo_group_threads<G>(),
                            CooSmem<T, TILE, G>::total, cta_cap, &per_sm)))
    return rc;
  if ((rc = coo_ctas_per_sm(coo_tile_kernel<T, true, TILE, 1>, kTileThreads, S1::total, cta_cap, &per_sm1))) return rc;
  if ((rc = coo_ctas_per_sm(coo_tile_kernel<T, false, TILE, 1>, kTileThreads, S1::total, cta_cap, &per_sm1))) return rc;
  const int64_t cap = int64_t(sm_count()) * per_sm, cap1 = int64_t(sm_count()) * per_sm1;
  p->grid = int(p->ntiles < cap ? p->ntiles : cap);
  p->grid_direct = int(p->ntiles < cap1 ? p->ntiles : cap1);
  return SPMV_OK;
}

// Warp-stream plan: entry ranges snapped to run starts (short runs stay
// whole), split long runs listed for the fix-up.  spmv_plan_config.warp_stream overrides
// the choice (plans with long runs).
static int coo_ws_build(spmv_coo_plan* p, cudaStream_t st) {
  const int mode = p->cfg.warp_stream;
  p->ws = mode < 0 ? p->n_long > 0 : mode > 0;
  if (!p->ws) return SPMV_OK;
  int rc, per_sm = 0;
  if (p->dtype == SPMV_F64)
    SPMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coo_wstream_kernel<double>, kWsWarps * 32, 0));
  else
    SPMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coo_wstream_kernel<float>, kWsWarps * 32, 0));
  per_sm = cap_ctas(per_sm, p->cfg.ctas_per_sm);
  p->ws_nwarps = std::max<int64_t>(1, std::min<int64_t>(int64_t(sm_count()) * per_sm * kWsWarps, p->nnz / kWsChunk));
  p->ws_nranges =
      std::max<int64_t>(p->ws_nwarps, std::min<int64_t>(p->ws_nwarps * p->ws_ranges_per_warp, p->nnz / kWsChunk));
  const int64_t nr = p->ws_nranges;
  if ((rc = p->ws_bounds.alloc(4 * (nr + 1))) || (rc = p->ws_row0.alloc(4 * nr))) return rc;
  const uint32_t* rs = p->run_start.as<uint32_t>();
  const int64_t gw = std::min<int64_t>((nr + 256) / 256, int64_t(sm_count()) * 16);
  ws_bounds_kernel<<<unsigned(gw), 256, 0, st>>>(rs, p->n_runs, p->nnz, nr, kExactLen, p->ws_bounds.as<uint32_t>(),
                                                 p->ws_row0.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  DevBuf ctr;
  if ((rc = ctr.alloc(8))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 8, st));
  const int64_t g_runs = std::min<int64_t>((p->n_runs + 255) / 256, int64_t(sm_count()) * 16);
  ws_span_list_kernel<<<unsigned(g_runs), 256, 0, st>>>(rs, p->n_runs, kExactLen, p->ws_bounds.as<uint32_t>(), nr,
                                                        nullptr, nullptr, nullptr, ctr.as<unsigned long long>());
  SPMV_LAUNCH_CHECK();
  unsigned long long h = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&h, ctr.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  p->ws_n_span = int64_t(h);
  if (p->ws_n_span > 0) {
    if ((rc = p->ws_span_run.alloc(4 * p->ws_n_span)) || (rc = p->ws_span_w0.alloc(4 * p->ws_n_span)) ||
        (rc = p->ws_span_w1.alloc(4 * p->ws_n_span)))
      return rc;
    SPMV_CUDA_TRY(cudaMemsetAsync(ctr.ptr, 0, 8, st));
    ws_span_list_kernel<<<unsigned(g_runs), 256, 0, st>>>(rs, p->n_runs, kExactLen, p->ws_bounds.as<uint32_t>(), nr,
                                                          p->ws_span_run.as<uint32_t>(), p->ws_span_w0.as<uint32_t>(),
                                                          p->ws_span_w1.as<uint32_t>(), ctr.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  }
  return SPMV_OK;
}

static int coo_plan_build(spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const void* av,
                          cudaStream_t st) {
  const int64_t nnz = p->nnz;
  const int tb = 256;
  const int64_t grid = std::min<int64_t>((nnz + tb - 1) / tb, int64_t(sm_count()) * 32);
  int rc;
  DevBuf flag;
  if ((rc = flag.alloc(sizeof(int)))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(int), st));
  rows_descending_kernel<<<unsigned(grid), tb, 0, st>>>(ai, nnz, flag.as<int>());
  SPMV_LAUNCH_CHECK();
  int h_flag = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&h_flag, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  p->row_sorted = h_flag == 0;
  const uint32_t* rows = ai;
  if (!p->row_sorted) {
    // Stable LSD radix sort on the row key keeps storage order inside rows.
    const size_t vs = value_size(p->dtype);
    DevBuf perm_in, perm_out, tmp;
    if ((rc = perm_in.alloc(4 * nnz)) || (rc = perm_out.alloc(4 * nnz)) || (rc = p->sorted_ai.alloc(4 * nnz)) ||
        (rc = p->sorted_aj.alloc(4 * nnz)) || (rc = p->sorted_av.alloc(vs * nnz)))
      return rc;
    iota_kernel<<<unsigned(grid), tb, 0, st>>>(perm_in.as<uint32_t>(), nnz);
    SPMV_LAUNCH_CHECK();
    int end_bit = 1;
    while (end_bit < 32 && (int64_t(1) << end_bit) < p->nrows) ++end_bit;
    size_t tmp_bytes = 0;
    SPMV_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ai, p->sorted_ai.as<uint32_t>(),
                                                  perm_in.as<uint32_t>(), perm_out.as<uint32_t>(), nnz, 0, end_bit,
                                                  st));
    if ((rc = tmp.alloc(tmp_bytes))) return rc;
    SPMV_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.ptr, tmp_bytes, ai, p->sorted_ai.as<uint32_t>(),
                                                  perm_in.as<uint32_t>(), perm_out.as<uint32_t>(), nnz, 0, end_bit,
                                                  st));
    if (p->dtype == SPMV_F64)
      gather_triples_kernel<double><<<unsigned(grid), tb, 0, st>>>(perm_out.as<uint32_t>(), nnz, aj,
                                                                  static_cast<const double*>(av),
                                                                  p->sorted_aj.as<uint32_t>(),
                                                                  p->sorted_av.as<double>());
    else
      gather_triples_kernel<float><<<unsigned(grid), tb, 0, st>>>(perm_out.as<uint32_t>(), nnz, aj,
                                                                 static_cast<const float*>(av),
                                                                 p->sorted_aj.as<uint32_t>(),
                                                                 p->sorted_av.as<float>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    rows = p->sorted_ai.as<uint32_t>();
  }
  // Run-length encode the (now non-decreasing) rows.
  DevBuf head, pos, tmp;
  if ((rc = head.alloc(4 * nnz)) || (rc = pos.alloc(4 * nnz))) return rc;
  run_heads_kernel<<<unsigned(grid), tb, 0, st>>>(rows, nnz, head.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  SPMV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, head.as<uint32_t>(), pos.as<uint32_t>(), nnz, st));
  if ((rc = tmp.alloc(tmp_bytes))) return rc;
  SPMV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, head.as<uint32_t>(), pos.as<uint32_t>(), nnz, st));
  uint32_t last_pos = 0, last_head = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&last_pos, pos.as<uint32_t>() + nnz - 1, 4, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(&last_head, head.as<uint32_t>() + nnz - 1, 4, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  p->n_runs = int64_t(last_pos) + last_head;
  if ((rc = p->run_start.alloc(4 * (p->n_runs + 1))) || (rc = p->run_row.alloc(4 * p->n_runs))) return rc;
  run_scatter_kernel<<<unsigned(grid), tb, 0, st>>>(rows, nnz, head.as<uint32_t>(), pos.as<uint32_t>(),
                                                    p->run_start.as<uint32_t>(), p->run_row.as<uint32_t>());
  SPMV_LAUNCH_CHECK();
  const uint32_t nnz32 = uint32_t(nnz);
  SPMV_CUDA_TRY(cudaMemcpyAsync(p->run_start.as<uint32_t>() + p->n_runs, &nnz32, 4, cudaMemcpyHostToDevice, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  DevBuf nl;
  if ((rc = nl.alloc(8))) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(nl.ptr, 0, 8, st));
  count_long_runs_kernel<<<unsigned(std::min<int64_t>((p->n_runs + 255) / 256, int64_t(sm_count()) * 16)), 256, 0,
                           st>>>(p->run_start.as<uint32_t>(), p->n_runs, nl.as<unsigned long long>());
  SPMV_LAUNCH_CHECK();
  unsigned long long h = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&h, nl.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  p->n_long = int64_t(h);
  // 1536-entry tiles; 7 consumer groups over 8 stages (one CTA per SM; no
  // long-row scratch, so they fit) for short runs, one group (4 CTAs/SM)
  // when long runs exist.  Measured on B200: 256^3 stencil 533 -> 711
  // GFLOP/s, Zipf 173 -> 222.
  p->tile = 1536;
  p->groups = p->n_long > 0 ? 1 : 7;
  const int t = p->cfg.tile;
  if (t == 1024 || t == 1536 || t == 2048) {
    p->tile = t;
    p->groups = 1;
  }
  if (p->cfg.groups > 0) p->groups = p->cfg.groups;
  if (p->n_long > 0) p->groups = 1;  // multi-group kernels carry no long-row scratch
  if (!coo_config_known(p->tile, p->groups)) {
    p->groups = 1;
    if (!coo_config_known(p->tile, 1)) p->tile = 2048;
  }
  p->ntiles = (nnz + p->tile - 1) / p->tile;
  // A CSR view of the plan's row-sorted triples (row pointers over the
  // sorted rows; the same column and value arrays): whole-matrix products
  // then stream 4 bytes per row instead of 4 bytes per entry of row indices
  // (16 -> 12 bytes per f64 entry: 256^3 COO 735 -> the CSR kernel's rate),
  // rows summed from +0.0 in storage order: np.add.at order (kernels.py:65),
  // bit-exact.  With long runs the view is kept if its plan takes the
  // column-panel path; without, unless the caller configured the COO tile
  // kernels (tile / groups / warp_stream) or turned views off (panels = 0).
  const bool view_long = p->n_long > 0 && p->cfg.panels != 0;
  const bool view_short = p->n_long == 0 && p->cfg.panels != 0 && p->cfg.tile == 0 && p->cfg.groups == 0 &&
                          p->cfg.warp_stream < 0 && p->nrows > 0 && nnz > 0 && p->nrows < int64_t(UINT32_MAX) - 1 &&
                          p->nrows <= 4 * nnz;  // hypersparse: the COO kernels' work follows the entries, not the rows
  if (view_long || view_short) {
    const uint32_t* vaj = p->row_sorted ? aj : p->sorted_aj.as<uint32_t>();
    const void* vav = p->row_sorted ? av : p->sorted_av.ptr;
    if ((rc = p->view_irp.alloc(4 * (p->nrows + 1)))) return rc;
    const int64_t gr = std::min<int64_t>((p->nrows + 256) / 256, int64_t(sm_count()) * 16);
    row_bounds_kernel<<<unsigned(gr), 256, 0, st>>>(rows, nnz, p->nrows, p->view_irp.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    spmv_plan_config vc = p->cfg;
    vc.flags |= 4;
    spmv_csr_plan* v = nullptr;
    if ((rc = spmv_csr_plan_create_ex(p->dtype, p->nrows, p->ncols, nnz, p->view_irp.as<uint32_t>(), vaj, vav, &vc,
                                      st, &v)))
      return rc;
    int path = 0;
    spmv_csr_plan_path(v, &path, nullptr);
    if (path == 2 || view_short) {
      p->csr_view = v;
      p->view_panel = path == 2;
      p->view_ai = ai;
      p->view_aj = aj;
      p->view_av = av;
    } else {
      spmv_csr_plan_destroy(v);
      p->view_irp.release();
    }
  }
  p->tma_hint = p->cfg.tma_hint != 0;  // COO: evict_first on the matrix stream unless turned off
  p->ws_ranges_per_warp = p->cfg.ranges_per_warp >= 1 && p->cfg.ranges_per_warp <= 64 ? p->cfg.ranges_per_warp : 8;
  if ((rc = coo_ws_build(p, st))) return rc;
  const size_t vs = value_size(p->dtype);
  SlotLayout lay;
  p->off_head_row = lay.add(4 * p->ntiles);
  p->off_tail_row = lay.add(4 * p->ntiles);
  p->off_pass = lay.add(4 * p->ntiles);
  p->off_head_val = lay.add(vs * p->ntiles);
  p->off_tail_val = lay.add(vs * p->ntiles);
  p->off_ws_head = lay.add(8 * p->ws_nranges);
  p->off_ws_tail = lay.add(8 * p->ws_nranges);
  p->off_ws_ctr = lay.add(8);
  p->off_steps = lay.add(8);
  p->scratch.bytes = lay.total;
#define X(TL, GR)                                                                                    \
  if (p->tile == TL && p->groups == GR)                                                             \
    return p->dtype == SPMV_F64 ? coo_launch_config<double, TL, GR>(p) : coo_launch_config<float, TL, GR>(p);
  SPMV_COO_CONFIGS(X)
#undef X
  return fail(SPMV_INVALID_ARG, "no COO kernel for tile %lld x %d groups", (long long)p->tile, p->groups);
}

template <typename T, int TILE, int G, int VW = 0>
static int coo_run_tiled(const spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const T* av, const T* x,
                   int64_t col_base, T* y, cudaStream_t st, int vla = 0) {
  if (p->nrows == 0) return SPMV_OK;
  if (p->nnz == 0) {
    SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(T) * p->nrows, st));
    return SPMV_OK;
  }
  if (!p->row_sorted) {
    ai = p->sorted_ai.as<uint32_t>();
    aj = p->sorted_aj.as<uint32_t>();
    av = p->sorted_av.as<T>();
  }
  unsigned char* scr = nullptr;
  int rc = p->scratch.get(st, reinterpret_cast<void**>(&scr));
  if (rc) return rc;
  CooParams<T> P;
  P.ai = ai;
  P.aj = aj;
  P.av = av;
  P.x = x;
  P.y = y;
  P.head_row = reinterpret_cast<uint32_t*>(scr + p->off_head_row);
  P.tail_row = reinterpret_cast<uint32_t*>(scr + p->off_tail_row);
  P.pass = reinterpret_cast<uint32_t*>(scr + p->off_pass);
  P.head_val = reinterpret_cast<T*>(scr + p->off_head_val);
  P.tail_val = reinterpret_cast<T*>(scr + p->off_tail_val);
  P.nrows = p->nrows;
  P.nnz = p->nnz;
  P.col_base = col_base;
  P.ntiles = p->ntiles;
  P.tile_begin = 0;
  P.mode = (p->cfg.flags & 3) | (p->tma_hint ? 4 : 0);
  P.vla = vla;
  if (p->n_runs < p->nrows) {  // empty rows exist: one memset instead of per-gap loops
    SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(T) * p->nrows, st));
    P.mode |= 8;
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(ai) % 16 == 0) && (reinterpret_cast<uintptr_t>(aj) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(av) % 16 == 0);
  P.n_bulk = aligned ? bulk_tiles(p->nnz, p->ntiles, TILE) : 0;
  const size_t smem1 = CooSmem<T, TILE, 1>::total;
  if constexpr (VW > 0) {
    // vla instantiations are not touched by the plan's occupancy queries
    static bool attrs = [] {
      cudaFuncSetAttribute(coo_tile_kernel<T, false, TILE, 1, VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(CooSmem<T, TILE, 1>::total));
      cudaFuncSetAttribute(coo_tile_kernel<T, true, TILE, 1, VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(CooSmem<T, TILE, 1>::total));
      cudaFuncSetAttribute(coo_tile_kernel<T, true, TILE, G, VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(CooSmem<T, TILE, G>::total));
      return true;
    }();
    (void)attrs;
  }
  if (!aligned) {
    coo_tile_kernel<T, false, TILE, 1, VW><<<unsigned(p->grid_direct), kTileThreads, smem1, st>>>(P);
  } else if (G == 1) {
    coo_tile_kernel<T, true, TILE, 1, VW><<<unsigned(p->grid), kTileThreads, smem1, st>>>(P);
  } else {
    if (P.n_bulk > 0)
      coo_tile_kernel<T, true, TILE, G, VW>
          <<<unsigned(std::min<int64_t>(p->grid, P.n_bulk)), G * coo_group_threads<G>(), CooSmem<T, TILE, G>::total,
             st>>>(P);
    if (P.n_bulk < p->ntiles) {  // tail tiles the bulk engine cannot address
      CooParams<T> Q = P;
      Q.tile_begin = P.n_bulk;
      const int64_t g1 = std::min<int64_t>(p->grid_direct, p->ntiles - P.n_bulk);
      coo_tile_kernel<T, false, TILE, 1, VW><<<unsigned(g1), kTileThreads, smem1, st>>>(Q);
    }
  }
  SPMV_LAUNCH_CHECK();
  if (p->n_long > 0) {
    const int64_t g = std::min<int64_t>((p->ntiles + 255) / 256, int64_t(sm_count()) * 8);
    coo_fixup_kernel<T><<<unsigned(g), 256, 0, st>>>(P);
    SPMV_LAUNCH_CHECK();
  }
  return SPMV_OK;
}

template <typename T>
static int coo_run_ws(const spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const T* av, const T* x,
                      int64_t col_base, T* y, cudaStream_t st) {
  if (!p->row_sorted) {
    ai = p->sorted_ai.as<uint32_t>();
    aj = p->sorted_aj.as<uint32_t>();
    av = p->sorted_av.as<T>();
  }
  unsigned char* scr = nullptr;
  int rc = p->scratch.get(st, reinterpret_cast<void**>(&scr));
  if (rc) return rc;
  if (p->n_runs < p->nrows) SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(T) * p->nrows, st));  // empty rows
  CooWsParams<T> P;
  P.ai = ai;
  P.aj = aj;
  P.av = av;
  P.x = x;
  P.y = y;
  P.bounds = p->ws_bounds.as<uint32_t>();
  P.head = reinterpret_cast<double*>(scr + p->off_ws_head);
  P.tail = reinterpret_cast<double*>(scr + p->off_ws_tail);
  P.ctr = reinterpret_cast<uint32_t*>(scr + p->off_ws_ctr);
  P.col_base = col_base;
  P.nwarps = p->ws_nwarps;
  P.nranges = p->ws_nranges;
  P.nnz = p->nnz;
  P.exact_len = uint32_t(kExactLen);
  const int64_t grid = (p->ws_nwarps + kWsWarps - 1) / kWsWarps;
  coo_wstream_kernel<T><<<unsigned(grid), kWsWarps * 32, 0, st>>>(P);
  SPMV_LAUNCH_CHECK();
  if (p->ws_n_span > 0) {
    const int64_t g = std::min<int64_t>((p->ws_n_span + 7) / 8, int64_t(sm_count()) * 8);  // a warp per row
    ws_span_fixup_kernel<T><<<unsigned(g), 256, 0, st>>>(p->ws_span_run.as<uint32_t>(), p->ws_span_w0.as<uint32_t>(),
                                                         p->ws_span_w1.as<uint32_t>(), p->ws_n_span, P.head, P.tail, y,
                                                         p->run_row.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
  }
  return SPMV_OK;
}

template <typename T>
static int coo_run(const spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const T* av, const T* x,
                   int64_t col_base, T* y, cudaStream_t st, int64_t x_len = -1) {
  if (p->csr_view && ai == p->view_ai && aj == p->view_aj && av == p->view_av)
    return spmv_csr(p->csr_view, p->view_irp.as<uint32_t>(), p->row_sorted ? aj : p->sorted_aj.as<uint32_t>(),
                    p->row_sorted ? static_cast<const void*>(av) : p->sorted_av.ptr, x, col_base,
                    x_len < 0 ? p->ncols - col_base : x_len, y, st);
  if (p->ws && p->nrows > 0 && p->nnz > 0) return coo_run_ws<T>(p, ai, aj, av, x, col_base, y, st);
#define X(TL, GR) \
  if (p->tile == TL && p->groups == GR) return coo_run_tiled<T, TL, GR>(p, ai, aj, av, x, col_base, y, st);
  SPMV_COO_CONFIGS(X)
#undef X
  return fail(SPMV_INVALID_ARG, "no COO kernel for tile %lld x %d groups", (long long)p->tile, p->groups);
}

// vla through the tile kernels (row-per-lane vla, tile.cuh row_vla_coo):
// plans without runs over 32 entries whose tile configuration has vla
// instantiations (any lane count).
#define SPMV_COO_VLA_CONFIGS(X) X(1536, 7)
template <typename T>
static int coo_run_vla_tiles(const spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const T* av,
                             const T* x, int64_t col_base, T* y, int lanes, cudaStream_t st, bool* done) {
  *done = false;
  if (p->n_long > 0 || lanes < 1) return SPMV_OK;
  const int w = lanes <= 1 ? 1 : lanes <= 2 ? 2 : lanes <= 4 ? 4 : lanes <= 8 ? 8 : lanes <= 16 ? 16 : 32;
#define X(TL, GR)                                                                              \
  if (p->tile == TL && p->groups == GR) {                                                      \
    *done = true;                                                                              \
    switch (w) {                                                                               \
      case 1: return coo_run_tiled<T, TL, GR, 1>(p, ai, aj, av, x, col_base, y, st, lanes);     \
      case 2: return coo_run_tiled<T, TL, GR, 2>(p, ai, aj, av, x, col_base, y, st, lanes);     \
      case 4: return coo_run_tiled<T, TL, GR, 4>(p, ai, aj, av, x, col_base, y, st, lanes);     \
      case 8: return coo_run_tiled<T, TL, GR, 8>(p, ai, aj, av, x, col_base, y, st, lanes);      \
      case 16: return coo_run_tiled<T, TL, GR, 16>(p, ai, aj, av, x, col_base, y, st, lanes);    \
      default: return coo_run_tiled<T, TL, GR, 32>(p, ai, aj, av, x, col_base, y, st, lanes);    \
    }                                                                                          \
  }
  SPMV_COO_VLA_CONFIGS(X)
#undef X
  return SPMV_OK;
}

// outer_steps of spmv_coo_vla: ceil(run length / L) per run.
__global__ void coo_vla_count_steps_kernel(const uint32_t* __restrict__ run_start, int64_t n_runs, int lanes,
                                           unsigned long long* __restrict__ steps) {
  unsigned long long c = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_runs; i += int64_t(gridDim.x) * blockDim.x)
    c += (run_start[i + 1] - run_start[i] + uint32_t(lanes) - 1) / uint32_t(lanes);
  for (int o = 16; o >= 1; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(steps, c);
}

namespace spmv {
int debug_counts_coo(unsigned long long* out4) { return debug_read_tu(out4); }
}  // namespace spmv

// The vla step counter of the stream's scratch slot.
static int steps_slot(const spmv_coo_plan* p, cudaStream_t st, unsigned long long** out) {
  unsigned char* scr = nullptr;
  int rc = p->scratch.get(st, reinterpret_cast<void**>(&scr));
  if (rc) return rc;
  if (!scr) return fail(SPMV_INVALID_ARG, "COO plan without scratch");
  *out = reinterpret_cast<unsigned long long*>(scr + p->off_steps);
  return SPMV_OK;
}

extern "C" {

int spmv_coo_plan_create(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* ai,
                         const uint32_t* aj, const void* av, void* stream, spmv_coo_plan** out) {
  return spmv_coo_plan_create_ex(dtype, nrows, ncols, nnz, ai, aj, av, nullptr, stream, out);
}

int spmv_coo_plan_config(const spmv_coo_plan* p, spmv_plan_config* out) {
  if (!p || !out) return fail(SPMV_INVALID_ARG, "NULL argument");
  *out = p->cfg;
  out->tile = int32_t(p->tile);
  out->groups = p->groups;
  out->exact_len = kExactLen;
  out->warp_stream = p->ws ? 1 : 0;
  out->ranges_per_warp = int32_t(p->ws_ranges_per_warp);
  out->tma_hint = p->tma_hint ? 1 : 0;
  out->panels = p->csr_view && p->view_panel ? 1 : 0;
  return SPMV_OK;
}

int spmv_coo_plan_create_ex(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* ai,
                            const uint32_t* aj, const void* av, const spmv_plan_config* cfg, void* stream,
                            spmv_coo_plan** out) {
  if (!out) return fail(SPMV_INVALID_ARG, "spmv_coo_plan_create: out is NULL");
  if (cfg && cfg->version != SPMV_PLAN_CONFIG_VERSION)
    return fail(SPMV_INVALID_ARG, "spmv_plan_config version %d, expected %d", cfg->version, SPMV_PLAN_CONFIG_VERSION);
  *out = nullptr;
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows < 0 || ncols < 0 || nnz < 0 || nnz > int64_t(UINT32_MAX) || nrows >= int64_t(UINT32_MAX))
    return fail(SPMV_INVALID_ARG, "bad COO sizes");
  if (nnz && (!ai || !aj || !av)) return fail(SPMV_INVALID_ARG, "NULL pointer");
  auto* p = new spmv_coo_plan();
  p->dtype = dtype;
  p->nrows = nrows;
  p->ncols = ncols;
  p->nnz = nnz;
  p->cfg = config_or_default(cfg);
  int rc = SPMV_OK;
  if (nnz) rc = coo_plan_build(p, ai, aj, av, as_stream(stream));
  // the vla step counter lives in the scratch slot even without entries
  if (!rc && !nnz) {
    SlotLayout lay;
    p->off_steps = lay.add(8);
    p->scratch.bytes = lay.total;
  }
  if (rc) {
    delete p;
    return rc;
  }
  *out = p;
  return SPMV_OK;
}

int spmv_coo_plan_destroy(spmv_coo_plan* p) {
  delete p;
  return SPMV_OK;
}

int spmv_coo_plan_info(const spmv_coo_plan* p, int64_t* n_runs, int64_t* n_long_runs, int64_t* n_items,
                       int* row_sorted, int64_t* launches) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (n_runs) *n_runs = p->n_runs;
  if (n_long_runs) *n_long_runs = p->n_long;
  if (n_items) *n_items = p->tile;
  if (row_sorted) *row_sorted = p->row_sorted ? 1 : 0;
  if (launches && p->csr_view)
    spmv_csr_plan_info(p->csr_view, nullptr, nullptr, launches);
  else if (launches && p->ws)
    *launches = 1 + (p->ws_n_span > 0 ? 1 : 0);
  else if (launches)
    *launches = (p->nrows > 0 ? 1 : 0) + (p->n_long > 0 ? 1 : 0) +
                (p->groups > 1 && p->nnz > 0 && bulk_tiles(p->nnz, p->ntiles, p->tile) < p->ntiles ? 1 : 0);
  return SPMV_OK;
}

int spmv_coo_plan_path(const spmv_coo_plan* p, int* warp_stream, int64_t* nwarps) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (warp_stream) *warp_stream = p->csr_view ? (p->view_panel ? 2 : 3) : p->ws ? 1 : 0;
  if (nwarps) {
    *nwarps = p->ws_nwarps;
    if (p->csr_view) spmv_csr_plan_path(p->csr_view, nullptr, nwarps);
  }
  return SPMV_OK;
}

int spmv_coo_plan_groups(const spmv_coo_plan* p, int* groups) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (groups) *groups = p->groups;
  return SPMV_OK;
}

int spmv_coo(const spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const void* av, const void* x,
             int64_t col_base, int64_t x_len, void* y, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (p->nrows && !y) return fail(SPMV_INVALID_ARG, "y is NULL");
  if (p->nnz && (!ai || !aj || !av || !x)) return fail(SPMV_INVALID_ARG, "NULL pointer");
  if (x_len < 0 || col_base < 0) return fail(SPMV_DIMENSION_MISMATCH, "bad x window");
  cudaStream_t st = as_stream(stream);
  if (p->dtype == SPMV_F64)
    return coo_run<double>(p, ai, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base,
                           static_cast<double*>(y), st, x_len);
  return coo_run<float>(p, ai, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
                        static_cast<float*>(y), st, x_len);
}

// Host x -> host y: x goes up in chunks, the product runs once all of x is
// on the device (COO rows are not tied to column prefixes), y comes down.
int spmv_coo_host(spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const void* av, const void* x_host,
                  void* y_host, int chunks, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (!x_host || !y_host) return fail(SPMV_INVALID_ARG, "NULL host buffer");
  if (p->nrows == 0 || p->ncols == 0) return fail(SPMV_INVALID_ARG, "host pipeline needs a non-empty matrix");
  if (chunks <= 0) chunks = 16;
  if (chunks > 1024) chunks = 1024;
  cudaStream_t st = as_stream(stream);
  const std::vector<int64_t> xb = host_x_chunks(p->ncols, chunks);
  const int nx = int(xb.size()) - 1;
  const size_t esz = value_size(p->dtype);
  auto compute = [&](int j, char* xd, char* yd, cudaStream_t s) -> int64_t {
    if (j < nx - 1) return 0;
    const int rc = p->dtype == SPMV_F64
                       ? coo_run<double>(p, ai, aj, static_cast<const double*>(av), reinterpret_cast<const double*>(xd),
                                         0, reinterpret_cast<double*>(yd), s, p->ncols)
                       : coo_run<float>(p, ai, aj, static_cast<const float*>(av), reinterpret_cast<const float*>(xd), 0,
                                        reinterpret_cast<float*>(yd), s, p->ncols);
    return rc ? -rc : p->nrows;
  };
  return run_host_pipeline(p->host, x_host, y_host, esz, p->ncols, p->nrows, xb, compute, true, st);
}

int spmv_coo_vla(spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const void* av, const void* x,
                 int64_t col_base, int64_t x_len, void* y, int lanes, int64_t* outer_steps, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (lanes < 1) return fail(SPMV_INVALID_ARG, "lane count must be >= 1");
  if (lanes > 1024) return fail(SPMV_UNSUPPORTED, "vla COO supports at most 1024 lanes, got %d", lanes);
  if (x_len < 0 || col_base < 0) return fail(SPMV_DIMENSION_MISMATCH, "bad x window");
  cudaStream_t st = as_stream(stream);
  if (outer_steps) *outer_steps = 0;
  if (p->nrows == 0) return SPMV_OK;
  if (p->nnz > 0) {
    bool done = false;
    if (p->csr_view && !p->view_panel && ai == p->view_ai && aj == p->view_aj && av == p->view_av) {
      // the row-pointer view: the CSR tile kernel with the COO step order
      int d = 0;
      const int rcv = spmvi_csr_vla_tiles(p->csr_view, p->view_irp.as<uint32_t>(),
                                         p->row_sorted ? aj : p->sorted_aj.as<uint32_t>(),
                                         p->row_sorted ? av : p->sorted_av.ptr, x, col_base, y, lanes, stream, &d);
      if (rcv) return rcv;
      done = d != 0;
    }
    const int rc = done ? SPMV_OK : p->dtype == SPMV_F64
                       ? coo_run_vla_tiles<double>(p, ai, aj, static_cast<const double*>(av),
                                                   static_cast<const double*>(x), col_base, static_cast<double*>(y),
                                                   lanes, st, &done)
                       : coo_run_vla_tiles<float>(p, ai, aj, static_cast<const float*>(av),
                                                  static_cast<const float*>(x), col_base, static_cast<float*>(y), lanes,
                                                  st, &done);
    if (rc) return rc;
    if (done) {
      if (outer_steps) {
        unsigned long long* steps = nullptr;
        int rc2 = steps_slot(p, st, &steps);
        if (rc2) return rc2;
        unsigned long long h = 0;
        SPMV_CUDA_TRY(cudaMemsetAsync(steps, 0, sizeof(h), st));
        const int64_t g = std::min<int64_t>((p->n_runs + 255) / 256, int64_t(sm_count()) * 16);
        coo_vla_count_steps_kernel<<<unsigned(g), 256, 0, st>>>(p->run_start.as<uint32_t>(), p->n_runs, lanes, steps);
        SPMV_LAUNCH_CHECK();
        SPMV_CUDA_TRY(cudaMemcpyAsync(&h, steps, sizeof(h), cudaMemcpyDeviceToHost, st));
        SPMV_CUDA_TRY(cudaStreamSynchronize(st));
        *outer_steps = int64_t(h);
      }
      return SPMV_OK;
    }
  }
  SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, value_size(p->dtype) * p->nrows, st));
  if (p->nnz == 0) return SPMV_OK;
  if (!p->row_sorted) {
    aj = p->sorted_aj.as<uint32_t>();
    av = p->sorted_av.ptr;
  }
  unsigned long long* steps = nullptr;
  if (outer_steps) {
    int rc2 = steps_slot(p, st, &steps);
    if (rc2) return rc2;
  }
  unsigned long long* steps_out = steps;
  if (steps) SPMV_CUDA_TRY(cudaMemsetAsync(steps, 0, sizeof(unsigned long long), st));
  int width = 1;
  while (width < lanes) width <<= 1;
  const int64_t cap = int64_t(sm_count()) * 16;
  const uint32_t* rs = p->run_start.as<uint32_t>();
  const uint32_t* rr = p->run_row.as<uint32_t>();
  if (width <= 32) {
    const int tb = 256;
    int64_t grid = (p->n_runs * width + tb - 1) / tb;
    if (grid > cap) grid = cap;
    const bool long_runs = p->n_long > 0;  // runs over 32 entries exist, so maybe over kVlaLong
    auto warp_kernel = [&](auto skip) {
      constexpr bool SKIP = decltype(skip)::value;
      if (p->dtype == SPMV_F64)
        coo_vla_warp_kernel<double, SKIP><<<unsigned(grid), tb, 0, st>>>(
            rs, rr, p->n_runs, aj, static_cast<const double*>(av), static_cast<const double*>(x), col_base,
            static_cast<double*>(y), lanes, width, steps);
      else
        coo_vla_warp_kernel<float, SKIP><<<unsigned(grid), tb, 0, st>>>(
            rs, rr, p->n_runs, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
            static_cast<float*>(y), lanes, width, steps);
    };
    // long runs, L <= 8: runs <= 32 one thread each, runs of 33..kVlaLong
    // by sub-warp groups over the plan's list, longer ones two-phase; the
    // step count then comes from the run lengths
    const bool split = long_runs && lanes <= 8;
    if (split) {
      int rc;
      {
        std::lock_guard<std::mutex> lock(p->build_mu);
        if (!p->vla_built && (rc = coo_vla_build(p, st))) return rc;
      }
      const int64_t gs = std::min<int64_t>((p->n_runs + 255) / 256, cap);
      auto short_kernel = [&](auto* tag) {
        using TT = std::remove_pointer_t<decltype(tag)>;
        const TT* avt = static_cast<const TT*>(av);
        const TT* xt = static_cast<const TT*>(x);
        TT* yt = static_cast<TT*>(y);
        switch (lanes <= 1 ? 1 : lanes <= 2 ? 2 : lanes <= 4 ? 4 : 8) {
          case 1: coo_vla_short_kernel<TT, 1><<<unsigned(gs), 256, 0, st>>>(rs, rr, p->n_runs, aj, avt, xt, col_base, yt, lanes); break;
          case 2: coo_vla_short_kernel<TT, 2><<<unsigned(gs), 256, 0, st>>>(rs, rr, p->n_runs, aj, avt, xt, col_base, yt, lanes); break;
          case 4: coo_vla_short_kernel<TT, 4><<<unsigned(gs), 256, 0, st>>>(rs, rr, p->n_runs, aj, avt, xt, col_base, yt, lanes); break;
          default: coo_vla_short_kernel<TT, 8><<<unsigned(gs), 256, 0, st>>>(rs, rr, p->n_runs, aj, avt, xt, col_base, yt, lanes);
        }
        if (p->vla_n_mid > 0) {
          const int64_t gm = std::min<int64_t>((p->vla_n_mid * width + tb - 1) / tb, cap);
          coo_vla_warp_kernel<TT, true><<<unsigned(gm), tb, 0, st>>>(rs, rr, p->vla_n_mid, aj, avt, xt, col_base, yt,
                                                                     lanes, width, nullptr, p->vla_mid.as<uint32_t>());
        }
      };
      if (p->dtype == SPMV_F64)
        short_kernel(static_cast<double*>(nullptr));
      else
        short_kernel(static_cast<float*>(nullptr));
      SPMV_LAUNCH_CHECK();
      if (steps) {
        const int64_t g = std::min<int64_t>((p->n_runs + 255) / 256, cap);
        coo_vla_count_steps_kernel<<<unsigned(g), 256, 0, st>>>(rs, p->n_runs, lanes, steps);
        SPMV_LAUNCH_CHECK();
        steps = nullptr;  // counted: the two-phase kernels below must not add theirs
      }
    } else if (long_runs) {
      warp_kernel(std::true_type{});
    } else {
      warp_kernel(std::false_type{});
    }
    if (long_runs) {  // runs over 32 entries exist: two-phase path for those over kVlaLong
      int rc;
      {
        std::lock_guard<std::mutex> lock(p->build_mu);
        if (!p->vla_built && (rc = coo_vla_build(p, st))) return rc;
      }
      void* sbuf = nullptr;
      if (p->vla_n > 0 && (rc = p->vla_scratch.get(st, &sbuf))) return rc;
      if (p->vla_n > 0) {
        const int64_t g1 = std::min<int64_t>((p->vla_chunks * 32 + tb - 1) / tb, cap);
        const int64_t g2 = std::min<int64_t>((p->vla_n * 32 + tb - 1) / tb, cap);
        const uint32_t* runs = p->vla_runs.as<uint32_t>();
        if (p->dtype == SPMV_F64) {
          double* S = static_cast<double*>(sbuf);
          coo_vla_steps_kernel<double><<<unsigned(g1), tb, 0, st>>>(
              rs, runs, p->vla_pre.as<uint32_t>(), p->vla_chunk_run.as<uint32_t>(), p->vla_chunks, aj,
              static_cast<const double*>(av), static_cast<const double*>(x), col_base, lanes, width, S);
          coo_vla_fold_kernel<double><<<unsigned(g2), tb, 0, st>>>(rs, rr, runs, p->vla_n, S, lanes,
                                                                    static_cast<double*>(y), steps);
        } else {
          float* S = static_cast<float*>(sbuf);
          coo_vla_steps_kernel<float><<<unsigned(g1), tb, 0, st>>>(
              rs, runs, p->vla_pre.as<uint32_t>(), p->vla_chunk_run.as<uint32_t>(), p->vla_chunks, aj,
              static_cast<const float*>(av), static_cast<const float*>(x), col_base, lanes, width, S);
          coo_vla_fold_kernel<float><<<unsigned(g2), tb, 0, st>>>(rs, rr, runs, p->vla_n, S, lanes,
                                                                   static_cast<float*>(y), steps);
        }
      }
    }
  } else {
    int64_t grid = p->n_runs < cap ? p->n_runs : cap;
    const size_t sm = value_size(p->dtype) * width;
    if (p->dtype == SPMV_F64)
      coo_vla_block_kernel<double><<<unsigned(grid), width, sm, st>>>(rs, rr, p->n_runs, aj,
                                                                       static_cast<const double*>(av),
                                                                       static_cast<const double*>(x), col_base,
                                                                       static_cast<double*>(y), lanes, steps);
    else
      coo_vla_block_kernel<float><<<unsigned(grid), width, sm, st>>>(rs, rr, p->n_runs, aj,
                                                                      static_cast<const float*>(av),
                                                                      static_cast<const float*>(x), col_base,
                                                                      static_cast<float*>(y), lanes, steps);
  }
  SPMV_LAUNCH_CHECK();
  if (outer_steps) {
    unsigned long long h = 0;
    SPMV_CUDA_TRY(cudaMemcpyAsync(&h, steps_out, sizeof(h), cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    *outer_steps = int64_t(h);
  }
  return SPMV_OK;
}

}  // extern "C"
