// On-device format conversions, bit-exact with convert.py.
//
//   coo_to_csr  (convert.py:87-94)   boundary scatter of a sorted row array
//   csr_to_coo  (convert.py:97-110)  row expansion + strictly-increasing check
//   coo_to_dia  (convert.py:113-144) diagonal-id bitmap, scan, scatter
//   dia_to_coo  (convert.py:147-177) per-row compaction of nonzero cells
//   sort_coo    (convert.py:60-84)   stable row sort (radix on the row only,
//                                    columns ride along), column sort inside
//                                    each row, duplicate runs summed in
//                                    np.add.reduceat order
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace spmv {

static int64_t grid_for(int64_t n, int tb = 256) {
  int64_t g = (n + tb - 1) / tb;
  const int64_t cap = int64_t(sm_count()) * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return g;
}

#define GRID_STRIDE(k, n) \
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < (n); k += int64_t(gridDim.x) * blockDim.x)

// ---- coo -> csr: irp[r] = first entry with row >= r -----------------------
// One pass: the row boundaries and the column / value copies (convert.py
// copies AJ and AV) share the read of each entry.
template <typename T>
__global__ void coo_to_csr_kernel(const uint32_t* __restrict__ ai, const uint32_t* __restrict__ aj,
                                  const T* __restrict__ av, int64_t nnz, int64_t nrows, uint32_t* __restrict__ irp,
                                  uint32_t* __restrict__ aj_out, T* __restrict__ av_out, int* __restrict__ descending) {
  GRID_STRIDE(k, nnz) {
    const int64_t rk = ai[k];
    const int64_t rp = k == 0 ? -1 : int64_t(ai[k - 1]);
    if (rk < rp) *descending = 1;  // a mis-flagged input: irp is rebuilt from counts
    for (int64_t r = rp + 1; r <= rk; ++r) irp[r] = uint32_t(k);
    if (k == nnz - 1)
      for (int64_t r = rk + 1; r <= nrows; ++r) irp[r] = uint32_t(nnz);
    aj_out[k] = aj[k];
    av_out[k] = av[k];
  }
}

// Four entries per thread with 16-byte loads and stores (16-byte aligned
// arrays): twice the bytes in flight per thread of the scalar kernel.
template <typename T> struct Vec4;
template <> struct Vec4<double> {
  double2 a, b;
  __device__ static Vec4 load(const double* p) {
    Vec4 v;
    v.a = __ldcs(reinterpret_cast<const double2*>(p));
    v.b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
    return v;
  }
  __device__ void store(double* p) const {
    __stcs(reinterpret_cast<double2*>(p), a);
    __stcs(reinterpret_cast<double2*>(p) + 1, b);
  }
};
template <> struct Vec4<float> {
  float4 a;
  __device__ static Vec4 load(const float* p) {
    Vec4 v;
    v.a = __ldcs(reinterpret_cast<const float4*>(p));
    return v;
  }
  __device__ void store(float* p) const { __stcs(reinterpret_cast<float4*>(p), a); }
};

template <typename T>
__global__ void __launch_bounds__(256) coo_to_csr_vec_kernel(const uint32_t* __restrict__ ai,
                                                             const uint32_t* __restrict__ aj,
                                                             const T* __restrict__ av, int64_t nnz, int64_t nrows,
                                                             uint32_t* __restrict__ irp, uint32_t* __restrict__ aj_out,
                                                             T* __restrict__ av_out, int* __restrict__ descending) {
  const int64_t n4 = nnz / 4;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = q * 4;
    const uint4 r = __ldcs(reinterpret_cast<const uint4*>(ai + k));
    const uint4 c = __ldcs(reinterpret_cast<const uint4*>(aj + k));
    const Vec4<T> v = Vec4<T>::load(av + k);
    int64_t rp = k == 0 ? -1 : int64_t(__ldg(ai + k - 1));
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t rk = rr[j];
      if (rk < rp) *descending = 1;  // a mis-flagged input: irp is rebuilt from counts
      for (int64_t row = rp + 1; row <= rk; ++row) irp[row] = uint32_t(k + j);
      rp = rk;
    }
    if (k + 4 == nnz)
      for (int64_t row = rp + 1; row <= nrows; ++row) irp[row] = uint32_t(nnz);
    __stcs(reinterpret_cast<uint4*>(aj_out + k), c);
    v.store(av_out + k);
  }
  // the last nnz % 4 entries
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int64_t k = n4 * 4; k < nnz; ++k) {
      const int64_t rk = ai[k], rp = k == 0 ? -1 : int64_t(ai[k - 1]);
      if (rk < rp) *descending = 1;
      for (int64_t row = rp + 1; row <= rk; ++row) irp[row] = uint32_t(k);
      if (k == nnz - 1)
        for (int64_t row = rk + 1; row <= nrows; ++row) irp[row] = uint32_t(nnz);
      aj_out[k] = aj[k];
      av_out[k] = av[k];
    }
}

// irp from per-row counts (np.bincount + cumsum, convert.py:92-93): the
// reference's result for any row order, used when the sorted flag is wrong.
__global__ void row_count_kernel(const uint32_t* __restrict__ ai, int64_t nnz, uint32_t* __restrict__ cnt) {
  GRID_STRIDE(k, nnz) atomicAdd(cnt + ai[k], 1u);
}

// ---- csr -> coo ------------------------------------------------------------
// A block takes kExpandRows rows, stages their row pointers in shared memory
// and walks the rows' entries entry-parallel: every thread finds its entry's
// row by binary search, so the row, column and value streams are read and
// written coalesced whatever the row lengths.  The column copy doubles as the
// strictly-increasing check (convert.py:104-108).
constexpr int kExpandRows = 256;

template <typename T>
__global__ void __launch_bounds__(256) csr_expand_kernel(const uint32_t* __restrict__ irp,
                                                         const uint32_t* __restrict__ aj, const T* __restrict__ av,
                                                         int64_t nrows, uint32_t* __restrict__ ai_out,
                                                         uint32_t* __restrict__ aj_out, T* __restrict__ av_out,
                                                         int* __restrict__ unsorted) {
  __shared__ uint32_t s_irp[kExpandRows + 1];
  bool bad = false;
  for (int64_t r0 = int64_t(blockIdx.x) * kExpandRows; r0 < nrows; r0 += int64_t(gridDim.x) * kExpandRows) {
    const int nr = int(min(int64_t(kExpandRows), nrows - r0));
    for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_irp[i] = irp[r0 + i];
    __syncthreads();
    const uint32_t e0 = s_irp[0], e1 = s_irp[nr];
    for (uint32_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      int lo = 0, hi = nr - 1;  // last local row with s_irp[row] <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_irp[mid] <= e) lo = mid; else hi = mid - 1;
      }
      const uint32_t c = aj[e];
      if (e > s_irp[lo] && c <= aj[e - 1]) bad = true;
      ai_out[e] = uint32_t(r0 + lo);
      aj_out[e] = c;
      av_out[e] = av[e];
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *unsorted = 1;
}

// Four consecutive entries per thread (16-byte aligned arrays): one binary
// search for the first, the row then advances while the next row pointer is
// reached; 16-byte loads and stores.
template <typename T>
__global__ void __launch_bounds__(256) csr_expand_vec_kernel(const uint32_t* __restrict__ irp,
                                                             const uint32_t* __restrict__ aj,
                                                             const T* __restrict__ av, int64_t nrows,
                                                             uint32_t* __restrict__ ai_out,
                                                             uint32_t* __restrict__ aj_out, T* __restrict__ av_out,
                                                             int* __restrict__ unsorted) {
  __shared__ uint32_t s_irp[kExpandRows + 1];
  bool bad = false;
  for (int64_t r0 = int64_t(blockIdx.x) * kExpandRows; r0 < nrows; r0 += int64_t(gridDim.x) * kExpandRows) {
    const int nr = int(min(int64_t(kExpandRows), nrows - r0));
    for (int i = threadIdx.x; i <= nr; i += blockDim.x) s_irp[i] = irp[r0 + i];
    __syncthreads();
    const uint32_t e0 = s_irp[0], e1 = s_irp[nr];
    // entries [e0, e1): an unaligned head and tail entry by entry, the
    // aligned middle four at a time
    const uint32_t m0 = min(e1, (e0 + 3u) & ~3u), m1 = max(m0, e1 & ~3u);
    auto row_of = [&](uint32_t e) {
      int lo = 0, hi = nr - 1;  // last local row with s_irp[row] <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_irp[mid] <= e) lo = mid; else hi = mid - 1;
      }
      return lo;
    };
    for (uint32_t e = (threadIdx.x < m0 - e0 ? e0 + threadIdx.x : m1 + (threadIdx.x - (m0 - e0)));
         threadIdx.x < (m0 - e0) + (e1 - m1) && e < e1; e = e1) {
      const int lo = row_of(e);
      const uint32_t c = aj[e];
      if (e > s_irp[lo] && c <= aj[e - 1]) bad = true;
      ai_out[e] = uint32_t(r0 + lo);
      aj_out[e] = c;
      av_out[e] = av[e];
    }
    for (uint32_t e = m0 + 4u * threadIdx.x; e < m1; e += 4u * blockDim.x) {
      int lo = row_of(e);
      const uint4 c = __ldcs(reinterpret_cast<const uint4*>(aj + e));
      const Vec4<T> v = Vec4<T>::load(av + e);
      const uint32_t cc[4] = {c.x, c.y, c.z, c.w};
      uint32_t rows[4];
      uint32_t prev = e > s_irp[lo] ? __ldg(aj + e - 1) : 0u;
      bool first = e == s_irp[lo];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        while (lo + 1 < nr && s_irp[lo + 1] <= e + j) {  // (empty rows are skipped)
          ++lo;
          first = true;
        }
        if (s_irp[lo] == e + j) first = true;
        if (!first && cc[j] <= prev) bad = true;
        rows[j] = uint32_t(r0 + lo);
        prev = cc[j];
        first = false;
      }
      __stcs(reinterpret_cast<uint4*>(ai_out + e), make_uint4(rows[0], rows[1], rows[2], rows[3]));
      __stcs(reinterpret_cast<uint4*>(aj_out + e), c);
      v.store(av_out + e);
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *unsorted = 1;
}

// ---- coo -> dia --------------------------------------------------------------
__global__ void diag_mark_kernel(const uint32_t* __restrict__ ai, const uint32_t* __restrict__ aj, int64_t nnz,
                                 int64_t nrows, uint32_t* __restrict__ flags) {
  // A matrix has few distinct diagonals: reading first (through L1) keeps
  // the flag lines shared instead of storing to the same words nnz times.
  GRID_STRIDE(k, nnz) {
    uint32_t* f = flags + (int64_t(aj[k]) - int64_t(ai[k]) + nrows - 1);
    if (__ldg(f) == 0u) *f = 1u;  // a stale 0 only repeats an idempotent store
  }
}

__global__ void diag_offsets_kernel(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ pos, int64_t nd_all,
                                    int64_t nrows, int32_t* __restrict__ offsets) {
  GRID_STRIDE(d, nd_all) if (flags[d]) offsets[pos[d]] = int32_t(d - (nrows - 1));
}

template <typename T>
__global__ void diag_scatter_kernel(const uint32_t* __restrict__ ai, const uint32_t* __restrict__ aj,
                                    const T* __restrict__ av, int64_t nnz, int64_t nrows, int64_t ndiags,
                                    const uint32_t* __restrict__ pos, T* __restrict__ out) {
  GRID_STRIDE(k, nnz) {
    const int64_t r = ai[k];
    const int64_t d = pos[int64_t(aj[k]) - r + nrows - 1];
    out[r * ndiags + d] = av[k];
  }
}

// ---- dia -> coo --------------------------------------------------------------
// Groups of W = next_pow2(ndiags) <= 32 lanes take one row each; lane d reads
// diagonal d (d + 32k when ndiags > 32), so a group reads its row's cells as
// one contiguous run and the kept cells (in-bounds, != 0: -0.0 dropped, NaN
// kept, convert.py:155-163) are compacted with a ballot: the emit pass writes
// each row's entries as a contiguous run in (row, col) order.  Four rows per
// group are loaded before they are compacted.
constexpr int kDiaRowsInFlight = 4;
inline int dia_group_width(int64_t nd) {
  int w = 1;
  while (w < nd && w < 32) w <<= 1;
  return w;
}

template <typename T, bool EMIT>
__global__ void __launch_bounds__(256) dia_rows_kernel(const int32_t* __restrict__ offs, const T* __restrict__ vals,
                                                       int64_t nrows, int64_t ncols, int nd, int W,
                                                       unsigned long long* __restrict__ counts,
                                                       const unsigned long long* __restrict__ starts,
                                                       uint32_t* __restrict__ ai, uint32_t* __restrict__ aj,
                                                       T* __restrict__ av) {
  const int lane = threadIdx.x & 31, sub = lane / W, gl = lane % W;
  const int gpw = 32 / W;  // groups (rows) per warp
  const unsigned gmask = W == 32 ? 0xffffffffu : ((1u << W) - 1u) << (sub * W);
  const unsigned below = (1u << lane) - 1u;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  constexpr int U = kDiaRowsInFlight;
  for (int64_t base = warp * gpw * U; base < nrows; base += nwarps * gpw * U) {
    unsigned long long o[U];  // EMIT: next output slot of each row; else its count
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + int64_t(u) * gpw + sub;
      o[u] = EMIT && i < nrows ? starts[i] : 0ull;
    }
    for (int d0 = 0; d0 < nd; d0 += W) {
      const int d = d0 + gl;
      const int64_t off = d < nd ? int64_t(__ldg(offs + d)) : 0;
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = base + int64_t(u) * gpw + sub;
        v[u] = (i < nrows && d < nd) ? vals[i * nd + d] : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = base + int64_t(u) * gpw + sub;
        const int64_t col = i + off;
        const bool keep = i < nrows && d < nd && col >= 0 && col < ncols && v[u] != T(0);
        const unsigned bal = __ballot_sync(0xffffffffu, keep) & gmask;
        if (EMIT && keep) {
          const unsigned long long q = o[u] + __popc(bal & below);
          ai[q] = uint32_t(i);
          aj[q] = uint32_t(col);
          av[q] = v[u];
        }
        o[u] += __popc(bal);
      }
    }
    if (!EMIT && gl == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = base + int64_t(u) * gpw + sub;
        if (i < nrows) counts[i] = o[u];
      }
    }
  }
}

// ndiags <= 32: tile kernels.  A CTA takes a tile of rows, 16 rows per lane
// group in registers (16 independent loads in flight per thread).  The count
// pass writes one count per TILE (no per-row arrays: 16-byte per-row counts and
// starts were 0.5 GB of extra traffic at 256^3); the emit pass reloads the
// tile, recomputes its ballots and places every kept cell from the tile's
// scanned start: a warp's ballot orders its kept cells by (sub, lane) = (row,
// diagonal) and u by row, so popc(ballot & lanes below) is the cell's slot in
// (row, col) order.  Row i of warp w: i = tile0 + (w * U + u) * gpw + sub.
// (A single pass that kept the tile in registers and found its start by a
// decoupled look-back over per-tile status words was slower than the two
// passes, 3.89 vs 3.47 ms at 256^3: with ~440 tiles of 28 KB in flight every
// tile walks back through most of the resident tiles' aggregates.)
constexpr int kDiaTileU = 16;        // rows per lane group held in registers
constexpr int kDiaTileThreads = 256;
inline int64_t dia_tile_rows(int W) { return int64_t(kDiaTileThreads / 32) * kDiaTileU * (32 / W); }

template <typename T, bool EMIT>
__global__ void __launch_bounds__(kDiaTileThreads, 3)
    dia_tiles_kernel(const int32_t* __restrict__ offs, const T* __restrict__ vals, int64_t nrows, int64_t ncols,
                     int nd, int W, unsigned long long* __restrict__ tile_count,
                     const unsigned long long* __restrict__ tile_start, uint32_t* __restrict__ ai,
                     uint32_t* __restrict__ aj, T* __restrict__ av) {
  constexpr int U = kDiaTileU, NW = kDiaTileThreads / 32;
  __shared__ unsigned long long s_warp[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane / W, gl = lane % W;
  const int gpw = 32 / W;
  const unsigned below = (1u << lane) - 1u;
  const int64_t tile = blockIdx.x;
  const int64_t row0 = tile * (int64_t(NW) * U * gpw) + int64_t(warp) * U * gpw;
  const int64_t off = gl < nd ? int64_t(__ldg(offs + gl)) : 0;
  // this lane's rows are i_u = i0 + u * gpw; the first nu of them exist; the
  // rows whose cell on the lane's diagonal lies inside the matrix are
  // [lo_i, lo_i + span) (one unsigned compare per cell; lanes past ndiags: none)
  const int64_t i0 = row0 + sub;
  const int nu = gl < nd ? int(min(int64_t(U), max(int64_t(0), (nrows - i0 + gpw - 1) / gpw))) : 0;
  const int64_t lo_i = max(int64_t(0), -off), hi_i = min(nrows, ncols - off);
  const uint64_t span = gl < nd && hi_i > lo_i ? uint64_t(hi_i - lo_i) : 0;
  const T* __restrict__ p = vals + i0 * nd + gl;
  const int64_t pstride = int64_t(gpw) * nd;
  T v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = u < nu ? (EMIT ? __ldcs(p + u * pstride) : __ldg(p + u * pstride)) : T(0);
  unsigned keepbits = 0;  // bit u: this lane's cell of row u is kept
  unsigned cnt = 0;       // the warp's kept cells
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool keep = uint64_t(i0 + u * gpw - lo_i) < span && v[u] != T(0);
    keepbits |= keep ? 1u << u : 0u;
    cnt += __popc(__ballot_sync(0xffffffffu, keep));
  }
  if (lane == 0) s_warp[warp] = cnt;
  __syncthreads();
  if (!EMIT) {
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t += s_warp[w];
      tile_count[tile] = t;
    }
    return;
  }
  unsigned long long q0 = tile_start[tile];
  for (int w = 0; w < warp; ++w) q0 += s_warp[w];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool keep = (keepbits >> u) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const unsigned long long q = q0 + __popc(bal & below);
      const int64_t i = row0 + int64_t(u) * gpw + sub;
      ai[q] = uint32_t(i);
      aj[q] = uint32_t(i + off);
      av[q] = v[u];
    }
    q0 += __popc(bal);
  }
}

// ---- sort_coo ------------------------------------------------------------------
// Unsorted rows take the group path further down (values ride along the
// radix sort, 256-row groups sorted in shared memory); matrices with groups
// too large for it, and inputs whose rows are already in order, take the
// per-row stage: Stage 1: a stable LSD radix sort of the row keys: each row's
// entries in storage order.  Stage 2: per row, its columns and values
// sorted by (column, storage index) — the reference's stable
// lexsort((cols, rows)) (convert.py:70) — written straight to the output
// positions (a warp per row of <= 32 entries: a bitonic sort in registers;
// longer rows: a segmented sort).  Stage 3, only when some (row, column)
// repeats: duplicate runs summed in np.add.reduceat order and compacted.

// flag = 1 if some row index is smaller than the one before it
// (a thread stops after the batch holding its first descent and stores once:
// on shuffled rows every thread used to store on every step, 1.5 ms of
// same-address traffic at 256^3; batches of 8 independent loads keep the
// ordered case a plain stream)
__global__ void rows_descend_kernel(const uint32_t* __restrict__ ai, int64_t nnz, int* __restrict__ flag) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  bool bad = false;
  for (int64_t k0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k0 < nnz && !bad; k0 += 8 * stride) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t k = k0 + u * stride;
      if (k > 0 && k < nnz) bad |= __ldg(ai + k) < __ldg(ai + k - 1);
    }
    if (!bad && *reinterpret_cast<volatile int*>(flag)) break;  // another thread found one
  }
  if (bad) *flag = 1;
}

// A row of m <= 32 entries, one column per lane (lanes >= m: `in` false):
// each lane's rank in ascending column order, by a bitonic sort of the bare
// 32-bit columns and a 5-step binary search of the lane's own column in the
// sorted registers — a third of the instructions of sorting 64-bit (column,
// index) keys, which bound these kernels (ncu: ALU pipe).  Equal columns
// (duplicates, rare) are reported instead: the caller then sorts the full
// keys, whose index part is the stable tie-break.
__device__ __forceinline__ int warp_col_rank(uint32_t c, bool in, uint32_t m, int lane, bool& has_dup) {
  uint32_t k = in ? c : 0xffffffffu;
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
    for (int j = kk >> 1; j >= 1; j >>= 1) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, k, j);
      const bool take_min = ((lane & j) == 0) == ((lane & kk) == 0);
      k = take_min ? min(k, o) : max(k, o);
    }
  const uint32_t prev = __shfl_up_sync(0xffffffffu, k, 1);
  has_dup = __any_sync(0xffffffffu, lane > 0 && uint32_t(lane) < m && prev == k);
  int lo = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const uint32_t probe = __shfl_sync(0xffffffffu, k, lo + step - 1);
    if (probe < c) lo += step;
  }
  return lo;  // sorted columns below c
}

// Two rows at once (two independent shuffle / compare chains in flight per
// warp: the kernels using this are bound by shuffle and load latency, not by
// issue slots).  dup: one of the two rows repeats a column.
__device__ __forceinline__ void warp_col_rank2(const uint32_t (&c)[2], const bool (&in)[2], const uint32_t (&m)[2],
                                               int lane, int (&rank)[2], bool& dup) {
  uint32_t k[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) k[u] = in[u] ? c[u] : 0xffffffffu;
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
    for (int j = kk >> 1; j >= 1; j >>= 1) {
      const bool take_min = ((lane & j) == 0) == ((lane & kk) == 0);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, k[u], j);
        k[u] = take_min ? min(k[u], o) : max(k[u], o);
      }
    }
  bool d = false;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint32_t prev = __shfl_up_sync(0xffffffffu, k[u], 1);
    d |= lane > 0 && uint32_t(lane) < m[u] && prev == k[u];
  }
  dup = __any_sync(0xffffffffu, d);
  rank[0] = rank[1] = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t probe = __shfl_sync(0xffffffffu, k[u], rank[u] + step - 1);
      if (probe < c[u]) rank[u] += step;
    }
}

// Rows of <= 32 entries: lane k holds entry k of the row, its payload
// (col << 32 | storage index); a bitonic sort of the payloads, then the
// value gathered through the storage index.  `pay` null: the rows were
// already in order, entry k's payload is built from aj[k] and k itself
// (no gathers at all).  Duplicate columns counted.
// (32 registers, 8 CTAs of 256 threads per SM: the kernel waits on its row's
// dependent loads, so rows in flight decide its speed: 256^3 rows-ordered
// sort 7.1 -> 6.3 ms against 6 CTAs per SM)
template <typename T>
__global__ void __launch_bounds__(256, 8) sort_rows_kernel(const uint32_t* __restrict__ rows_s, const unsigned long long* __restrict__ pay,
                                 const uint32_t* __restrict__ seg, int64_t nseg, const uint32_t* __restrict__ aj,
                                 const T* __restrict__ av, uint32_t* __restrict__ ai_out,
                                 uint32_t* __restrict__ aj_out, T* __restrict__ av_out, uint32_t* __restrict__ ucnt,
                                 unsigned long long* __restrict__ ndup) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long dups = 0;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < nseg; i += nw) {
    const uint32_t a = seg[i], n = seg[i + 1] - a;
    if (n > 32) continue;  // warp-uniform
    const bool in = uint32_t(lane) < n;
    unsigned long long key = ~0ull;
    if (in) key = pay ? pay[a + lane] : (static_cast<unsigned long long>(aj[a + lane]) << 32) | (a + lane);
    bool has_dup;
    const int rank = warp_col_rank(uint32_t(key >> 32), in, n, lane, has_dup);
    if (!has_dup) {  // distinct columns: every lane stores its own entry at its rank
      if (in) {
        ai_out[a + lane] = rows_s[a];
        aj_out[a + rank] = uint32_t(key >> 32);
        av_out[a + rank] = av[uint32_t(key)];
      }
      if (lane == 0) ucnt[i] = n;
      continue;
    }
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j >= 1; j >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, j);
        const bool take_min = ((lane & j) == 0) == ((lane & k) == 0);
        key = (take_min ? ok < key : ok > key) ? ok : key;
      }
    const unsigned long long prev = __shfl_up_sync(0xffffffffu, key, 1);
    const bool head = in && (lane == 0 || (prev >> 32) != (key >> 32));
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    if (in) {
      ai_out[a + lane] = rows_s[a];
      aj_out[a + lane] = uint32_t(key >> 32);
      av_out[a + lane] = av[uint32_t(key)];
    }
    if (lane == 0) {
      ucnt[i] = __popc(heads);
      dups += n - __popc(heads);
    }
  }
  if (lane == 0 && dups) atomicAdd(ndup, dups);
}

// Rows over 32 entries: (begin, end) of each (count only when lb is null).
__global__ void list_long_segments_kernel(const uint32_t* __restrict__ seg, int64_t nseg, uint32_t* __restrict__ lb,
                                          uint32_t* __restrict__ le, unsigned long long* __restrict__ n) {
  GRID_STRIDE(i, nseg) {
    const uint32_t a = seg[i], b = seg[i + 1];
    if (b - a <= 32) continue;
    const unsigned long long k = atomicAdd(n, 1ull);
    if (lb) {
      lb[k] = a;
      le[k] = b;
    }
  }
}

// Long rows, before their segmented sort: key = (col << 32 | storage
// index), from the stage-1 payloads or (rows already in order) built.
__global__ void long_keys_kernel(const unsigned long long* __restrict__ pay, const uint32_t* __restrict__ aj,
                                 const uint32_t* __restrict__ lb, const uint32_t* __restrict__ le, int64_t nl,
                                 unsigned long long* __restrict__ key) {
  for (int64_t i = blockIdx.x; i < nl; i += gridDim.x)
    for (uint32_t k = lb[i] + threadIdx.x; k < le[i]; k += blockDim.x)
      key[k] = pay ? pay[k] : (static_cast<unsigned long long>(aj[k]) << 32) | k;
}

// Long rows after the segmented sort: outputs in place, duplicates counted.
template <typename T>
__global__ void long_emit_kernel(const uint32_t* __restrict__ rows_s, const unsigned long long* __restrict__ key,
                                 const uint32_t* __restrict__ seg, int64_t nseg, const T* __restrict__ av,
                                 uint32_t* __restrict__ ai_out, uint32_t* __restrict__ aj_out,
                                 T* __restrict__ av_out, uint32_t* __restrict__ ucnt,
                                 unsigned long long* __restrict__ ndup) {
  GRID_STRIDE(i, nseg) {
    const uint32_t a = seg[i], b = seg[i + 1];
    if (b - a <= 32) continue;
    uint32_t u = 0;
    for (uint32_t k = a; k < b; ++k) {
      ai_out[k] = rows_s[a];
      aj_out[k] = uint32_t(key[k] >> 32);
      av_out[k] = av[uint32_t(key[k])];
      u += (k == a || (key[k] >> 32) != (key[k - 1] >> 32));
    }
    ucnt[i] = u;
    if (b - a > u) atomicAdd(ndup, static_cast<unsigned long long>(b - a - u));
  }
}

// ---- sort_coo, unsorted rows: values ride along, 256-row groups ---------------
// The stage-1 sort above fetched every value through a random storage
// index afterwards (a 32-byte DRAM sector per 8-byte value: ~10 ms at
// 256^3).  Here the (column, value) pair is the radix sort's payload and the
// sort stops 8 bits short: a stable LSD sort on row bits [8, bits(nrows))
// leaves every group of 256 consecutive rows contiguous, its entries in
// storage order.  One CTA then sorts a group in shared memory: a counting
// sort on the low 8 row bits, a warp bitonic sort of each row's (column,
// local index) keys — the local index is the storage order, i.e. the
// stable tie-break of lexsort((cols, rows)) (convert.py:70) — and coalesced
// stores of the finished rows.  One radix pass fewer, no random fetch.
// Sort key of the radix passes: row << 32 | column (only row bits are sorted on).
__global__ void sort_pack_kernel(const uint32_t* __restrict__ ai, const uint32_t* __restrict__ aj, int64_t nnz,
                                 unsigned long long* __restrict__ key) {
  GRID_STRIDE(k, nnz) key[k] = (static_cast<unsigned long long>(ai[k]) << 32) | aj[k];
}

// start[q] = first sorted entry whose key >> shift is >= q, q = 0..ngroups.
// One binary search per group over the sorted keys (a few thousand random
// reads) instead of a pass over all of them.
__global__ void group_bounds_kernel(const unsigned long long* __restrict__ key_s, int64_t nnz, int shift,
                                    int64_t ngroups, uint32_t* __restrict__ start) {
  GRID_STRIDE(q, ngroups + 1) {
    int64_t lo = 0, hi = nnz;  // first i in [0, nnz] with key_s[i] >> shift >= q
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (int64_t(__ldg(key_s + mid) >> shift) < q) lo = mid + 1; else hi = mid;
    }
    start[q] = uint32_t(lo);
  }
}

__global__ void max_diff_kernel(const uint32_t* __restrict__ start, int64_t n, uint32_t* __restrict__ out) {
  uint32_t m = 0;
  GRID_STRIDE(i, n) m = max(m, start[i + 1] - start[i]);
  for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

constexpr int kGroupBits = 8;       // low row bits sorted inside a group, at most
constexpr int kGroupRows = 1 << kGroupBits;
constexpr int kGroupMax = 7168;     // entries per group the shared-memory sort takes (two CTAs per SM for f64)
constexpr int kGroupThreads = 512;
static_assert(kGroupMax <= 8192, "local index in 13 bits");
template <typename T> constexpr size_t group_smem_bytes() {
  return size_t(kGroupMax) * (sizeof(T) + 4 + 2 + 1) + (kGroupRows + 4) * 4 * 2;
}

// (column, local index) order of two entries of a group.
__device__ __forceinline__ bool group_less(const uint32_t* scol, uint32_t i, uint32_t l) {
  const uint32_t ci = scol[i], cl = scol[l];
  return ci < cl || (ci == cl && i < l);
}

template <typename T>
__global__ void __launch_bounds__(kGroupThreads, 2)
    group_sort_kernel(const unsigned long long* __restrict__ key_s, const T* __restrict__ val_s,
                      const uint32_t* __restrict__ gstart, int64_t ngroups, int lo, uint32_t* __restrict__ ai_out,
                      uint32_t* __restrict__ aj_out, T* __restrict__ av_out, uint32_t* __restrict__ seg,
                      uint32_t* __restrict__ ucnt, unsigned long long* __restrict__ ndup) {
  extern __shared__ __align__(16) unsigned char group_smem[];
  T* sval = reinterpret_cast<T*>(group_smem);
  uint32_t* scol = reinterpret_cast<uint32_t*>(sval + kGroupMax);
  uint32_t* cnt = scol + kGroupMax;            // kGroupRows + 1 (+ pad): counts, then row starts
  uint32_t* cur = cnt + kGroupRows + 4;        // scatter cursors
  uint16_t* sord = reinterpret_cast<uint16_t*>(cur + kGroupRows + 4);  // local indices grouped by row
  uint8_t* srow = reinterpret_cast<uint8_t*>(sord + kGroupMax);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grows = 1 << lo;  // rows per group
  const uint32_t rmask = uint32_t(grows - 1);
  unsigned long long dups = 0;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const uint32_t a = gstart[g], n = gstart[g + 1] - a;
    if (tid < kGroupRows) cnt[tid] = 0;
    __syncthreads();
    // the group's entries into shared memory, 7 loads in flight per thread
    for (uint32_t i0 = 0; i0 < n; i0 += 7 * kGroupThreads) {
      unsigned long long k[7];
      T v[7];
#pragma unroll
      for (int u = 0; u < 7; ++u) {
        const uint32_t i = i0 + u * kGroupThreads + tid;
        if (i < n) {
          k[u] = __ldcs(key_s + a + i);
          v[u] = __ldcs(val_s + a + i);
        }
      }
#pragma unroll
      for (int u = 0; u < 7; ++u) {
        const uint32_t i = i0 + u * kGroupThreads + tid;
        if (i < n) {
          const uint32_t r = uint32_t(k[u] >> 32) & rmask;
          srow[i] = uint8_t(r);
          scol[i] = uint32_t(k[u]);
          sval[i] = v[u];
          atomicAdd(&cnt[r], 1u);
        }
      }
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 256 row counts: 8 per lane
      uint32_t c[8], sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        c[k] = cnt[lane * 8 + k];
        sum += c[k];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t up = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += up;
      }
      uint32_t run = inc - sum;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        cnt[lane * 8 + k] = run;
        cur[lane * 8 + k] = run;
        run += c[k];
      }
      if (lane == 31) cnt[kGroupRows] = run;
    }
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kGroupThreads) sord[atomicAdd(&cur[srow[i]], 1u)] = uint16_t(i);
    __syncthreads();
    constexpr int NWG = kGroupThreads / 32;
    for (int rp = warp; rp < grows; rp += 2 * NWG) {
      // two rows per step (rp and rp + NWG) when both hold 1..32 entries with
      // distinct columns: two rank networks in flight per warp
      if (rp + NWG < grows) {
        uint32_t s2[2], m2[2], i2[2] = {0u, 0u}, c2[2] = {0u, 0u};
        bool in2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          s2[u] = cnt[rp + u * NWG];
          m2[u] = cnt[rp + u * NWG + 1] - s2[u];
        }
        if (m2[0] - 1u < 32u && m2[1] - 1u < 32u) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            in2[u] = uint32_t(lane) < m2[u];
            if (in2[u]) {
              i2[u] = sord[s2[u] + lane];
              c2[u] = scol[i2[u]];
            }
          }
          int rank2[2];
          bool dup2;
          warp_col_rank2(c2, in2, m2, lane, rank2, dup2);
          if (!dup2) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int64_t sidx = g * grows + rp + u * NWG;
              if (in2[u]) {
                ai_out[a + s2[u] + lane] = uint32_t(sidx);
                aj_out[a + s2[u] + rank2[u]] = c2[u];
                av_out[a + s2[u] + rank2[u]] = sval[i2[u]];
              }
              if (lane == 0) {
                seg[sidx] = a + s2[u];
                ucnt[sidx] = m2[u];
              }
            }
            continue;
          }
        }
      }
      // one row at a time: a pair with an empty, long or repeated-column row, and the last odd row
      for (int r = rp; r < grows && r <= rp + NWG; r += NWG) {
        const uint32_t s0 = cnt[r], m = cnt[r + 1] - s0;
        const int64_t sidx = g * grows + r;
        const uint32_t row = uint32_t(sidx);
        if (lane == 0) seg[sidx] = a + s0;
        if (m == 0) continue;
        uint32_t heads_n = 0;
        if (m <= 32) {
          const bool in = uint32_t(lane) < m;
          unsigned long long key = ~0ull;
          uint32_t i = 0, c = 0;
          if (in) {
            i = sord[s0 + lane];
            c = scol[i];
            key = (static_cast<unsigned long long>(c) << 13) | i;
          }
          bool has_dup;
          const int rank = warp_col_rank(c, in, m, lane, has_dup);
          if (!has_dup) {  // distinct columns: every lane stores its own entry at its rank
            if (in) {
              ai_out[a + s0 + lane] = row;
              aj_out[a + s0 + rank] = c;
              av_out[a + s0 + rank] = sval[i];
            }
            if (lane == 0) ucnt[sidx] = m;
            continue;
          }
#pragma unroll
          for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j >= 1; j >>= 1) {
              const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, j);
              const bool take_min = ((lane & j) == 0) == ((lane & k) == 0);
              key = (take_min ? ok < key : ok > key) ? ok : key;
            }
          const unsigned long long prev = __shfl_up_sync(0xffffffffu, key, 1);
          const bool head = in && (lane == 0 || (prev >> 13) != (key >> 13));
          heads_n = __popc(__ballot_sync(0xffffffffu, head));
          if (in) {
            ai_out[a + s0 + lane] = row;
            aj_out[a + s0 + lane] = uint32_t(key >> 13);
            av_out[a + s0 + lane] = sval[uint32_t(key) & 8191u];
          }
        } else {
          // a longer row: its local indices sorted in place by (column, index),
          // a bitonic network with every merge ascending (entries past m act as
          // +infinity and never move)
          uint32_t N = 64;
          while (N < m) N <<= 1;
          for (uint32_t k = 2; k <= N; k <<= 1) {
            for (uint32_t j = k >> 1; j >= 1; j >>= 1) {
              for (uint32_t t = lane; t < N / 2; t += 32) {
                uint32_t i, l;
                if (j == (k >> 1)) {  // mirror step
                  const uint32_t blk = t / j, off = t % j;
                  i = blk * k + off;
                  l = blk * k + k - 1 - off;
                } else {
                  const uint32_t blk = t / j, off = t % j;
                  i = blk * 2 * j + off;
                  l = i + j;
                }
                if (l < m) {
                  const uint32_t x = sord[s0 + i], y = sord[s0 + l];
                  if (group_less(scol, y, x)) {
                    sord[s0 + i] = uint16_t(y);
                    sord[s0 + l] = uint16_t(x);
                  }
                }
              }
              __syncwarp();
            }
          }
          for (uint32_t t0 = 0; t0 < m; t0 += 32) {
            const uint32_t t = t0 + lane;
            const bool in = t < m;
            uint32_t i = 0;
            bool head = false;
            if (in) {
              i = sord[s0 + t];
              head = t == 0 || scol[sord[s0 + t - 1]] != scol[i];
              ai_out[a + s0 + t] = row;
              aj_out[a + s0 + t] = scol[i];
              av_out[a + s0 + t] = sval[i];
            }
            heads_n += __popc(__ballot_sync(0xffffffffu, head));
          }
        }
        if (lane == 0) {
          ucnt[sidx] = heads_n;
          dups += m - heads_n;
        }
      }
    }
    __syncthreads();
  }
  if (lane == 0 && dups) atomicAdd(ndup, dups);
}

// Fallback after a full row sort: stage-2 inputs from the sorted keys.
__global__ void sort_unpack_kernel(const unsigned long long* __restrict__ key_s, int64_t nnz,
                                   uint32_t* __restrict__ rows, unsigned long long* __restrict__ pay) {
  GRID_STRIDE(k, nnz) {
    const unsigned long long key = key_s[k];
    rows[k] = uint32_t(key >> 32);
    pay[k] = (key << 32) | static_cast<unsigned long long>(k);
  }
}

// numpy 2.3 pairwise_sum (loops_utils.h): < 8 terms sequential from -0.0,
// <= 128 terms eight interleaved accumulators, else split at n/2 rounded
// down to a multiple of 8.  Verified bit-for-bit against np.add.reduceat
// (tests/golden/make_golden.py pins it).
template <typename T>
__device__ T np_pairwise(const T* __restrict__ v, uint32_t n) {
  if (n < 8) {
    T res = T(-0.0);
    for (uint32_t i = 0; i < n; ++i) res = add_rn(res, v[i]);
    return res;
  }
  if (n <= 128) {
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = v[j];
    uint32_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = add_rn(r[j], v[i + j]);
    T res = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])), add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
    for (; i < n; ++i) res = add_rn(res, v[i]);
    return res;
  }
  uint32_t n2 = n / 2;
  n2 -= n2 % 8;
  return add_rn(np_pairwise(v, n2), np_pairwise(v + n2, n - n2));
}

// Duplicate runs (some (row, column) repeats): each run of equal columns in
// a row, already in storage order, becomes first + pairwise sum of the rest
// (np.add.reduceat, convert.py:80; zero sums kept), written compacted at
// opos[i] into the second buffers.
template <typename T>
__global__ void merge_runs_kernel(const uint32_t* __restrict__ seg, const uint32_t* __restrict__ opos, int64_t nseg,
                                  const uint32_t* __restrict__ ai_s, const uint32_t* __restrict__ aj_s,
                                  const T* __restrict__ av_s, uint32_t* __restrict__ ai_o, uint32_t* __restrict__ aj_o,
                                  T* __restrict__ av_o) {
  GRID_STRIDE(i, nseg) {
    const uint32_t a = seg[i], b = seg[i + 1];
    uint32_t o = opos[i];
    for (uint32_t k = a; k < b;) {
      uint32_t e = k + 1;
      while (e < b && aj_s[e] == aj_s[k]) ++e;
      T v = av_s[k];
      if (e - k > 1) v = add_rn(v, np_pairwise(av_s + k + 1, e - k - 1));
      ai_o[o] = ai_s[k];
      aj_o[o] = aj_s[k];
      av_o[o] = v;
      ++o;
      k = e;
    }
  }
}

}  // namespace spmv

using namespace spmv;

struct spmv_dia_builder {
  int64_t nrows = 0, ncols = 0, nnz = 0, nd_all = 0, ndiags = 0;
  ScratchBuf flags, pos;
};

struct spmv_dia_collect {
  int64_t nrows = 0, ncols = 0, ndiags = 0, nnz = 0;
  int64_t units = 0;  // counts / starts hold one entry per row, or per row tile (ndiags <= 32)
  bool tiled = false;
  ScratchBuf counts, starts;
};

template <typename V>
static int excl_scan(const V* in, V* out, int64_t n, cudaStream_t st) {
  size_t tmp_bytes = 0;
  SPMV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, n, st));
  ScratchBuf tmp;
  int rc = tmp.alloc(tmp_bytes, st);
  if (rc) return rc;
  SPMV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, in, out, n, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  return SPMV_OK;
}

template <typename V>
static int scan_total(const V* flags, const V* pos, int64_t n, cudaStream_t st, int64_t* total) {
  V a = 0, b = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&a, flags + n - 1, sizeof(V), cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(&b, pos + n - 1, sizeof(V), cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  *total = int64_t(a) + int64_t(b);
  return SPMV_OK;
}

extern "C" {

int spmv_coo_to_csr(int dtype, int64_t nrows, int64_t nnz, const uint32_t* ai, const uint32_t* aj, const void* av,
                    uint32_t* irp, uint32_t* aj_out, void* av_out, void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows < 0 || nnz < 0 || nnz > int64_t(UINT32_MAX)) return fail(SPMV_INVALID_ARG, "bad sizes");
  if (!irp) return fail(SPMV_INVALID_ARG, "row_pointers_out is NULL");
  cudaStream_t st = as_stream(stream);
  if (nnz == 0) {
    SPMV_CUDA_TRY(cudaMemsetAsync(irp, 0, sizeof(uint32_t) * (nrows + 1), st));
    return SPMV_OK;
  }
  ScratchBuf flag;
  int rc = flag.alloc(sizeof(int), st);
  if (rc) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(int), st));
  const bool vec = ((reinterpret_cast<uintptr_t>(ai) | reinterpret_cast<uintptr_t>(aj) |
                     reinterpret_cast<uintptr_t>(av) | reinterpret_cast<uintptr_t>(aj_out) |
                     reinterpret_cast<uintptr_t>(av_out)) & 15) == 0 && nnz >= 4;
  if (vec && dtype == SPMV_F64)
    coo_to_csr_vec_kernel<double><<<unsigned(grid_for(nnz / 4)), 256, 0, st>>>(
        ai, aj, static_cast<const double*>(av), nnz, nrows, irp, aj_out, static_cast<double*>(av_out),
        flag.as<int>());
  else if (vec)
    coo_to_csr_vec_kernel<float><<<unsigned(grid_for(nnz / 4)), 256, 0, st>>>(
        ai, aj, static_cast<const float*>(av), nnz, nrows, irp, aj_out, static_cast<float*>(av_out),
        flag.as<int>());
  else if (dtype == SPMV_F64)
    coo_to_csr_kernel<double><<<unsigned(grid_for(nnz)), 256, 0, st>>>(
        ai, aj, static_cast<const double*>(av), nnz, nrows, irp, aj_out, static_cast<double*>(av_out),
        flag.as<int>());
  else
    coo_to_csr_kernel<float><<<unsigned(grid_for(nnz)), 256, 0, st>>>(
        ai, aj, static_cast<const float*>(av), nnz, nrows, irp, aj_out, static_cast<float*>(av_out),
        flag.as<int>());
  SPMV_LAUNCH_CHECK();
  int h = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&h, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  if (h) {  // rows not actually non-decreasing: counts + exclusive scan, like bincount/cumsum
    ScratchBuf cnt;
    if ((rc = cnt.alloc(sizeof(uint32_t) * (nrows + 1), st))) return rc;
    SPMV_CUDA_TRY(cudaMemsetAsync(cnt.ptr, 0, sizeof(uint32_t) * (nrows + 1), st));
    row_count_kernel<<<unsigned(grid_for(nnz)), 256, 0, st>>>(ai, nnz, cnt.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    if ((rc = excl_scan<uint32_t>(cnt.as<uint32_t>(), irp, nrows + 1, st))) return rc;
  }
  return SPMV_OK;
}

int spmv_csr_to_coo(int dtype, int64_t nrows, int64_t nnz, const uint32_t* irp, const uint32_t* aj, const void* av,
                    uint32_t* ai_out, uint32_t* aj_out, void* av_out, int* sorted_out, void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows < 0 || nnz < 0 || nnz > int64_t(UINT32_MAX)) return fail(SPMV_INVALID_ARG, "bad sizes");
  cudaStream_t st = as_stream(stream);
  if (sorted_out) *sorted_out = 1;
  if (nnz == 0 || nrows == 0) return SPMV_OK;
  ScratchBuf flag;
  int rc = flag.alloc(sizeof(int), st);
  if (rc) return rc;
  SPMV_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(int), st));
  {
    int64_t g = (nrows + kExpandRows - 1) / kExpandRows;
    const int64_t cap = int64_t(sm_count()) * 8;
    if (g > cap) g = cap;
    const bool vec = ((reinterpret_cast<uintptr_t>(aj) | reinterpret_cast<uintptr_t>(av) |
                       reinterpret_cast<uintptr_t>(ai_out) | reinterpret_cast<uintptr_t>(aj_out) |
                       reinterpret_cast<uintptr_t>(av_out)) & 15) == 0;
    if (vec && dtype == SPMV_F64)
      csr_expand_vec_kernel<double><<<unsigned(g), 256, 0, st>>>(irp, aj, static_cast<const double*>(av), nrows,
                                                                ai_out, aj_out, static_cast<double*>(av_out),
                                                                flag.as<int>());
    else if (vec)
      csr_expand_vec_kernel<float><<<unsigned(g), 256, 0, st>>>(irp, aj, static_cast<const float*>(av), nrows, ai_out,
                                                               aj_out, static_cast<float*>(av_out), flag.as<int>());
    else if (dtype == SPMV_F64)
      csr_expand_kernel<double><<<unsigned(g), 256, 0, st>>>(irp, aj, static_cast<const double*>(av), nrows, ai_out,
                                                            aj_out, static_cast<double*>(av_out), flag.as<int>());
    else
      csr_expand_kernel<float><<<unsigned(g), 256, 0, st>>>(irp, aj, static_cast<const float*>(av), nrows, ai_out,
                                                           aj_out, static_cast<float*>(av_out), flag.as<int>());
    SPMV_LAUNCH_CHECK();
  }
  int h = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&h, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  if (sorted_out) *sorted_out = h ? 0 : 1;
  return SPMV_OK;
}

int spmv_coo_to_dia_analyze(int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* ai, const uint32_t* aj,
                            void* stream, spmv_dia_builder** out, int64_t* ndiags_out) {
  if (!out || !ndiags_out) return fail(SPMV_INVALID_ARG, "NULL output");
  *out = nullptr;
  if (nrows < 0 || ncols < 0 || nnz < 0) return fail(SPMV_INVALID_ARG, "bad sizes");
  cudaStream_t st = as_stream(stream);
  auto* b = new spmv_dia_builder();
  b->nrows = nrows;
  b->ncols = ncols;
  b->nnz = nnz;
  int rc = SPMV_OK;
  if (nnz > 0) {
    b->nd_all = nrows + ncols - 1;
    if (!(rc = b->flags.alloc(4 * b->nd_all, st)) && !(rc = b->pos.alloc(4 * b->nd_all, st))) {
      cudaError_t e = cudaMemsetAsync(b->flags.ptr, 0, 4 * b->nd_all, st);
      if (e != cudaSuccess) rc = fail(SPMV_CUDA_ERROR, "memset: %s", cudaGetErrorString(e));
      if (!rc) {
        diag_mark_kernel<<<unsigned(grid_for(nnz)), 256, 0, st>>>(ai, aj, nnz, nrows, b->flags.as<uint32_t>());
        e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(SPMV_CUDA_ERROR, "diag_mark: %s", cudaGetErrorString(e));
      }
      if (!rc) rc = excl_scan<uint32_t>(b->flags.as<uint32_t>(), b->pos.as<uint32_t>(), b->nd_all, st);
      if (!rc) rc = scan_total<uint32_t>(b->flags.as<uint32_t>(), b->pos.as<uint32_t>(), b->nd_all, st, &b->ndiags);
    }
  }
  if (rc) {
    delete b;
    return rc;
  }
  *ndiags_out = b->ndiags;
  *out = b;
  return SPMV_OK;
}

int spmv_coo_to_dia_offsets(const spmv_dia_builder* b, int32_t* offsets_out, void* stream) {
  if (!b) return fail(SPMV_INVALID_ARG, "builder is NULL");
  if (b->ndiags == 0) return SPMV_OK;
  cudaStream_t st = as_stream(stream);
  diag_offsets_kernel<<<unsigned(grid_for(b->nd_all)), 256, 0, st>>>(b->flags.as<uint32_t>(), b->pos.as<uint32_t>(),
                                                                     b->nd_all, b->nrows, offsets_out);
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

int spmv_coo_to_dia_fill(const spmv_dia_builder* b, int dtype, int64_t padded_rows, const uint32_t* ai,
                         const uint32_t* aj, const void* av, void* values_out, void* stream) {
  if (!b) return fail(SPMV_INVALID_ARG, "builder is NULL");
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (padded_rows < b->nrows) return fail(SPMV_INVALID_ARG, "padded_rows < nrows");
  cudaStream_t st = as_stream(stream);
  const size_t bytes = value_size(dtype) * size_t(padded_rows) * size_t(b->ndiags);
  if (bytes) SPMV_CUDA_TRY(cudaMemsetAsync(values_out, 0, bytes, st));
  if (b->nnz == 0 || b->ndiags == 0) return SPMV_OK;
  if (dtype == SPMV_F64)
    diag_scatter_kernel<double><<<unsigned(grid_for(b->nnz)), 256, 0, st>>>(
        ai, aj, static_cast<const double*>(av), b->nnz, b->nrows, b->ndiags, b->pos.as<uint32_t>(),
        static_cast<double*>(values_out));
  else
    diag_scatter_kernel<float><<<unsigned(grid_for(b->nnz)), 256, 0, st>>>(
        ai, aj, static_cast<const float*>(av), b->nnz, b->nrows, b->ndiags, b->pos.as<uint32_t>(),
        static_cast<float*>(values_out));
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

int spmv_dia_builder_destroy(spmv_dia_builder* b) {
  delete b;
  return SPMV_OK;
}

int spmv_dia_to_coo_count(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags, const int32_t* offsets,
                          const void* values, void* stream, spmv_dia_collect** out, int64_t* nnz_out) {
  if (!out || !nnz_out) return fail(SPMV_INVALID_ARG, "NULL output");
  *out = nullptr;
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows < 0 || ncols < 0 || ndiags < 0) return fail(SPMV_INVALID_ARG, "bad sizes");
  cudaStream_t st = as_stream(stream);
  auto* c = new spmv_dia_collect();
  c->nrows = nrows;
  c->ncols = ncols;
  c->ndiags = ndiags;
  int rc = SPMV_OK;
  if (nrows > 0 && ndiags > 0) {
    const int W = dia_group_width(ndiags);
    c->tiled = ndiags <= 32 && (nrows + dia_tile_rows(W) - 1) / dia_tile_rows(W) <= int64_t(INT32_MAX);
    c->units = c->tiled ? (nrows + dia_tile_rows(W) - 1) / dia_tile_rows(W) : nrows;
    rc = c->counts.alloc(8 * c->units, st);
    if (!rc) rc = c->starts.alloc(8 * c->units, st);
    if (!rc && c->tiled) {
      if (dtype == SPMV_F64)
        dia_tiles_kernel<double, false><<<unsigned(c->units), kDiaTileThreads, 0, st>>>(
            offsets, static_cast<const double*>(values), nrows, ncols, int(ndiags), W,
            c->counts.as<unsigned long long>(), nullptr, nullptr, nullptr, nullptr);
      else
        dia_tiles_kernel<float, false><<<unsigned(c->units), kDiaTileThreads, 0, st>>>(
            offsets, static_cast<const float*>(values), nrows, ncols, int(ndiags), W,
            c->counts.as<unsigned long long>(), nullptr, nullptr, nullptr, nullptr);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) rc = fail(SPMV_CUDA_ERROR, "dia_count: %s", cudaGetErrorString(e));
    } else if (!rc) {
      const int64_t g = grid_for(nrows * W / kDiaRowsInFlight);
      if (dtype == SPMV_F64)
        dia_rows_kernel<double, false><<<unsigned(g), 256, 0, st>>>(
            offsets, static_cast<const double*>(values), nrows, ncols, int(ndiags), W,
            c->counts.as<unsigned long long>(), nullptr, nullptr, nullptr, nullptr);
      else
        dia_rows_kernel<float, false><<<unsigned(g), 256, 0, st>>>(
            offsets, static_cast<const float*>(values), nrows, ncols, int(ndiags), W,
            c->counts.as<unsigned long long>(), nullptr, nullptr, nullptr, nullptr);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) rc = fail(SPMV_CUDA_ERROR, "dia_count: %s", cudaGetErrorString(e));
    }
    if (!rc)
      rc = excl_scan<unsigned long long>(c->counts.as<unsigned long long>(), c->starts.as<unsigned long long>(),
                                         c->units, st);
    if (!rc)
      rc = scan_total<unsigned long long>(c->counts.as<unsigned long long>(), c->starts.as<unsigned long long>(),
                                          c->units, st, &c->nnz);
    if (!rc && c->nnz > int64_t(UINT32_MAX))
      rc = fail(SPMV_INDEX_OVERFLOW, "DIA holds %lld nonzeros, over the 32-bit index range", (long long)c->nnz);
  }
  if (rc) {
    delete c;
    return rc;
  }
  *nnz_out = c->nnz;
  *out = c;
  return SPMV_OK;
}

int spmv_dia_to_coo_fill(const spmv_dia_collect* c, int dtype, const int32_t* offsets, const void* values,
                         uint32_t* ai, uint32_t* aj, void* av, void* stream) {
  if (!c) return fail(SPMV_INVALID_ARG, "collector is NULL");
  if (c->nnz == 0) return SPMV_OK;
  cudaStream_t st = as_stream(stream);
  const int W = dia_group_width(c->ndiags);
  if (c->tiled) {
    if (dtype == SPMV_F64)
      dia_tiles_kernel<double, true><<<unsigned(c->units), kDiaTileThreads, 0, st>>>(
          offsets, static_cast<const double*>(values), c->nrows, c->ncols, int(c->ndiags), W, nullptr,
          c->starts.as<unsigned long long>(), ai, aj, static_cast<double*>(av));
    else
      dia_tiles_kernel<float, true><<<unsigned(c->units), kDiaTileThreads, 0, st>>>(
          offsets, static_cast<const float*>(values), c->nrows, c->ncols, int(c->ndiags), W, nullptr,
          c->starts.as<unsigned long long>(), ai, aj, static_cast<float*>(av));
    SPMV_LAUNCH_CHECK();
    return SPMV_OK;
  }
  const int64_t g = grid_for(c->nrows * W / kDiaRowsInFlight);
  if (dtype == SPMV_F64)
    dia_rows_kernel<double, true><<<unsigned(g), 256, 0, st>>>(
        offsets, static_cast<const double*>(values), c->nrows, c->ncols, int(c->ndiags), W, nullptr,
        c->starts.as<unsigned long long>(), ai, aj, static_cast<double*>(av));
  else
    dia_rows_kernel<float, true><<<unsigned(g), 256, 0, st>>>(
        offsets, static_cast<const float*>(values), c->nrows, c->ncols, int(c->ndiags), W, nullptr,
        c->starts.as<unsigned long long>(), ai, aj, static_cast<float*>(av));
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

int spmv_dia_collect_destroy(spmv_dia_collect* c) {
  delete c;
  return SPMV_OK;
}

static int bits_for(int64_t n) {  // bits holding 0 .. n-1 (at least 1)
  int b = 1;
  while (b < 32 && (int64_t(1) << b) < n) ++b;
  return b;
}

}  // extern "C"

// Stage 3: duplicate runs merged and compacted (through a copy: rows move to
// lower positions).  seg: nseg + 1 row starts; ucnt: unique columns per row.
template <typename T>
static int merge_duplicates(const uint32_t* seg, const uint32_t* ucnt, int64_t nseg, int64_t nnz, uint32_t* ai_out,
                            uint32_t* aj_out, T* av_out, cudaStream_t st) {
  int r;
  ScratchBuf opos, ai_s, aj_s, av_s;
  if ((r = opos.alloc(4 * (nseg + 1), st)) || (r = ai_s.alloc(4 * nnz, st)) || (r = aj_s.alloc(4 * nnz, st)) ||
      (r = av_s.alloc(sizeof(T) * nnz, st)))
    return r;
  if ((r = excl_scan<uint32_t>(ucnt, opos.as<uint32_t>(), nseg + 1, st))) return r;
  SPMV_CUDA_TRY(cudaMemcpyAsync(ai_s.ptr, ai_out, 4 * nnz, cudaMemcpyDeviceToDevice, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(aj_s.ptr, aj_out, 4 * nnz, cudaMemcpyDeviceToDevice, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(av_s.ptr, av_out, sizeof(T) * nnz, cudaMemcpyDeviceToDevice, st));
  merge_runs_kernel<T><<<unsigned(grid_for(nseg)), 256, 0, st>>>(seg, opos.as<uint32_t>(), nseg, ai_s.as<uint32_t>(),
                                                                 aj_s.as<uint32_t>(), av_s.as<T>(), ai_out, aj_out,
                                                                 av_out);
  SPMV_LAUNCH_CHECK();
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  return SPMV_OK;
}

// Onesweep tile shape of sort_coo's radix passes.  CUB's sm_100 policy for
// 8-byte keys is 384 threads x 24 items; tools/radix_tune.cu (B200, two
// passes + histogram over 449M (key, value) records, input kept) measures
// 9.06 ms for it with 64-bit offsets, 13.14 ms with 32-bit offsets (an
// occupancy cliff), and 8.36 ms for 256 threads x 30 items with either offset
// width (f32 values: 7.57 default, 7.55 at 256 x 32): profiles/r2d_radix_tune.txt.
// Everything else is CUB's own policy.
template <typename T>
struct SortHub {
  using Base = cub::detail::radix::policy_hub<unsigned long long, T, unsigned int>;
  using B = typename Base::Policy1000;
  struct Policy : cub::ChainedPolicy<500, Policy, Policy> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = 8;
    using HistogramPolicy = typename B::HistogramPolicy;
    using ExclusiveSumPolicy = typename B::ExclusiveSumPolicy;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<256, sizeof(T) == 8 ? 30 : 32, unsigned long long, 1,
                                          cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY, cub::BLOCK_SCAN_RAKING_MEMOIZE,
                                          cub::RADIX_SORT_STORE_DIRECT, 8>;
    using ScanPolicy = typename B::ScanPolicy;
    using DownsweepPolicy = typename B::DownsweepPolicy;
    using AltDownsweepPolicy = typename B::AltDownsweepPolicy;
    using UpsweepPolicy = typename B::UpsweepPolicy;
    using AltUpsweepPolicy = typename B::AltUpsweepPolicy;
    using SingleTilePolicy = typename B::SingleTilePolicy;
    using SegmentedPolicy = typename B::SegmentedPolicy;
    using AltSegmentedPolicy = typename B::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy;
};

template <typename T>
static int sort_coo_run(int64_t nrows, int64_t nnz, const uint32_t* ai, const uint32_t* aj, const T* av,
                        uint32_t* ai_out, uint32_t* aj_out, T* av_out, int64_t* n_out, cudaStream_t st) {
  *n_out = 0;
  if (nnz == 0) return SPMV_OK;
  int r;
  ScratchBuf rows_buf, pay_buf, tmp, flag;
  auto tmp_for = [&](size_t bytes) -> int { return bytes > tmp.bytes ? tmp.alloc(bytes, st) : SPMV_OK; };
  // rows already non-decreasing (a COO without its sorted flag): no stage 1
  if ((r = flag.alloc(sizeof(int), st))) return r;
  SPMV_CUDA_TRY(cudaMemsetAsync(flag.ptr, 0, sizeof(int), st));
  rows_descend_kernel<<<unsigned(grid_for(nnz)), 256, 0, st>>>(ai, nnz, flag.as<int>());
  SPMV_LAUNCH_CHECK();
  int hflag = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&hflag, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  const bool rows_sorted = hflag == 0;
  const uint32_t* rows_p = ai;
  const unsigned long long* pay_p = nullptr;
  const T* av_p = av;
  ScratchBuf av_buf;
  if (!rows_sorted) {
    // stage 1: stable radix sort on the row bits above the low `lo`, the
    // column (in the key's low half) and the value riding along; then groups
    // of 2^lo rows in shared memory.  lo: the most bits (<= 8) whose groups
    // should fit going by the mean row length (checked exactly after the sort).
    const int bits = bits_for(nrows);
    int lo = std::min(bits, kGroupBits);
    while (lo > 0 && double(nnz) / double(nrows) * double(1 << lo) * 1.03 > double(kGroupMax)) --lo;
    ScratchBuf key_in, key_s, val_s;
    if ((r = key_in.alloc(8 * nnz, st)) || (r = key_s.alloc(8 * nnz, st)) || (r = val_s.alloc(sizeof(T) * nnz, st)))
      return r;
    sort_pack_kernel<<<unsigned(grid_for(nnz)), 256, 0, st>>>(ai, aj, nnz, key_in.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    auto radix = [&](int b0, int b1) -> int {  // (key_in, av) -> (key_s, val_s), stable, on key bits [b0, b1)
      // DeviceRadixSort::SortPairs with the onesweep tile shape of SortHub (32-bit offsets: nnz < 2^32)
      using Dispatch = cub::DispatchRadixSort<false, unsigned long long, T, unsigned int, SortHub<T>>;
      cub::DoubleBuffer<unsigned long long> dk(key_in.as<unsigned long long>(), key_s.as<unsigned long long>());
      cub::DoubleBuffer<T> dv(const_cast<T*>(av), val_s.as<T>());  // not overwritten: is_overwrite_okay = false
      size_t tb = 0;
      SPMV_CUDA_TRY(Dispatch::Dispatch(nullptr, tb, dk, dv, static_cast<unsigned int>(nnz), b0, b1, false, st));
      int rr = tmp_for(tb);
      if (rr) return rr;
      SPMV_CUDA_TRY(Dispatch::Dispatch(tmp.ptr, tb, dk, dv, static_cast<unsigned int>(nnz), b0, b1, false, st));
      return SPMV_OK;
    };
    bool grouped = false;
    // (hypersparse matrices, far more rows than entries, skip the group path:
    // its per-row segment arrays would dwarf the entries)
    if (lo > 0 && nrows <= 4 * nnz + 65536) {
      const unsigned long long* ks = key_in.as<unsigned long long>();
      const T* vs = av;
      if (bits > lo) {
        if ((r = radix(32 + lo, 32 + bits))) return r;
        ks = key_s.as<unsigned long long>();
        vs = val_s.as<T>();
      }
      const int64_t ngroups = ((nrows - 1) >> lo) + 1;
      ScratchBuf gstart, gmax;
      if ((r = gstart.alloc(4 * (ngroups + 1), st)) || (r = gmax.alloc(4, st))) return r;
      SPMV_CUDA_TRY(cudaMemsetAsync(gmax.ptr, 0, 4, st));
      group_bounds_kernel<<<unsigned(grid_for(ngroups + 1)), 256, 0, st>>>(ks, nnz, 32 + lo, ngroups, gstart.as<uint32_t>());
      SPMV_LAUNCH_CHECK();
      max_diff_kernel<<<unsigned(grid_for(ngroups)), 256, 0, st>>>(gstart.as<uint32_t>(), ngroups, gmax.as<uint32_t>());
      SPMV_LAUNCH_CHECK();
      uint32_t hmax = 0;
      SPMV_CUDA_TRY(cudaMemcpyAsync(&hmax, gmax.ptr, 4, cudaMemcpyDeviceToHost, st));
      SPMV_CUDA_TRY(cudaStreamSynchronize(st));
      if (hmax <= uint32_t(kGroupMax)) {
        grouped = true;
        const int64_t nseg = ngroups << lo;
        ScratchBuf seg, ucnt, ndup;
        if ((r = seg.alloc(4 * (nseg + 1), st)) || (r = ucnt.alloc(4 * (nseg + 1), st)) || (r = ndup.alloc(8, st)))
          return r;
        SPMV_CUDA_TRY(cudaMemsetAsync(ucnt.ptr, 0, 4 * (nseg + 1), st));
        SPMV_CUDA_TRY(cudaMemsetAsync(ndup.ptr, 0, 8, st));
        const uint32_t nnz32 = uint32_t(nnz);
        SPMV_CUDA_TRY(cudaMemcpyAsync(seg.as<uint32_t>() + nseg, &nnz32, 4, cudaMemcpyHostToDevice, st));
        static bool attr = [] {
          cudaFuncSetAttribute(group_sort_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(group_smem_bytes<T>()));
          return true;
        }();
        (void)attr;
        const unsigned gg = unsigned(std::min<int64_t>(ngroups, int64_t(sm_count()) * 2));
        group_sort_kernel<T><<<gg, kGroupThreads, group_smem_bytes<T>(), st>>>(
            ks, vs, gstart.as<uint32_t>(), ngroups, lo, ai_out, aj_out, av_out, seg.as<uint32_t>(),
            ucnt.as<uint32_t>(), ndup.as<unsigned long long>());
        SPMV_LAUNCH_CHECK();
        unsigned long long hd = 0;
        SPMV_CUDA_TRY(cudaMemcpyAsync(&hd, ndup.ptr, 8, cudaMemcpyDeviceToHost, st));
        SPMV_CUDA_TRY(cudaStreamSynchronize(st));
        *n_out = nnz - int64_t(hd);
        if (hd == 0) return SPMV_OK;
        return merge_duplicates<T>(seg.as<uint32_t>(), ucnt.as<uint32_t>(), nseg, nnz, ai_out, aj_out, av_out, st);
      }
    }
    // groups too large for shared memory (long rows): the full stable row
    // sort, then the per-row stage below on the sorted (column, value) pairs
    (void)grouped;
    if ((r = radix(32, 32 + bits))) return r;
    if ((r = rows_buf.alloc(4 * nnz, st)) || (r = pay_buf.alloc(8 * nnz, st))) return r;
    sort_unpack_kernel<<<unsigned(grid_for(nnz)), 256, 0, st>>>(key_s.as<unsigned long long>(), nnz,
                                                                rows_buf.as<uint32_t>(),
                                                                pay_buf.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    key_in.release();
    key_s.release();
    av_buf.ptr = val_s.ptr;  // keeps the sorted values alive past this block
    av_buf.bytes = val_s.bytes;
    av_buf.st = st;
    val_s.ptr = nullptr;
    val_s.bytes = 0;
    rows_p = rows_buf.as<uint32_t>();
    pay_p = pay_buf.as<unsigned long long>();
    av_p = av_buf.as<T>();
  }
  size_t tb = 0;
  // row segments: run lengths of the sorted rows, scanned
  ScratchBuf uniq, counts, nseg_d, seg;
  if ((r = uniq.alloc(4 * nnz, st)) || (r = counts.alloc(4 * (nnz + 1), st)) || (r = nseg_d.alloc(8, st))) return r;
  SPMV_CUDA_TRY(cub::DeviceRunLengthEncode::Encode(nullptr, tb, rows_p, uniq.as<uint32_t>(),
                                                   counts.as<uint32_t>(), nseg_d.as<int64_t>(), nnz, st));
  if ((r = tmp_for(tb))) return r;
  SPMV_CUDA_TRY(cub::DeviceRunLengthEncode::Encode(tmp.ptr, tb, rows_p, uniq.as<uint32_t>(),
                                                   counts.as<uint32_t>(), nseg_d.as<int64_t>(), nnz, st));
  int64_t nseg = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&nseg, nseg_d.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  uniq.release();
  if ((r = seg.alloc(4 * (nseg + 1), st))) return r;
  SPMV_CUDA_TRY(cudaMemsetAsync(counts.as<uint32_t>() + nseg, 0, 4, st));
  if ((r = excl_scan<uint32_t>(counts.as<uint32_t>(), seg.as<uint32_t>(), nseg + 1, st))) return r;
  // stage 2: columns inside each row, straight to the output positions
  ScratchBuf ucnt, ndup;
  if ((r = ucnt.alloc(4 * (nseg + 1), st)) || (r = ndup.alloc(8, st))) return r;
  SPMV_CUDA_TRY(cudaMemsetAsync(ucnt.ptr, 0, 4 * (nseg + 1), st));
  SPMV_CUDA_TRY(cudaMemsetAsync(ndup.ptr, 0, 8, st));
  const int64_t gw = std::min<int64_t>((nseg * 32 + 255) / 256, int64_t(sm_count()) * 64);
  sort_rows_kernel<T><<<unsigned(gw), 256, 0, st>>>(rows_p, pay_p, seg.as<uint32_t>(), nseg, aj, av_p, ai_out, aj_out,
                                                    av_out, ucnt.as<uint32_t>(), ndup.as<unsigned long long>());
  SPMV_LAUNCH_CHECK();
  ScratchBuf nlong;
  if ((r = nlong.alloc(8, st))) return r;
  SPMV_CUDA_TRY(cudaMemsetAsync(nlong.ptr, 0, 8, st));
  list_long_segments_kernel<<<unsigned(grid_for(nseg)), 256, 0, st>>>(seg.as<uint32_t>(), nseg, nullptr, nullptr,
                                                                      nlong.as<unsigned long long>());
  SPMV_LAUNCH_CHECK();
  unsigned long long hl = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&hl, nlong.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  if (hl > 0) {  // rows over 32 entries: a segmented sort of their keys
    const int64_t nl = int64_t(hl);
    ScratchBuf lb, le, keys, sorted;
    if ((r = lb.alloc(4 * nl, st)) || (r = le.alloc(4 * nl, st)) || (r = keys.alloc(8 * nnz, st)) ||
        (r = sorted.alloc(8 * nnz, st)))
      return r;
    SPMV_CUDA_TRY(cudaMemsetAsync(nlong.ptr, 0, 8, st));
    list_long_segments_kernel<<<unsigned(grid_for(nseg)), 256, 0, st>>>(seg.as<uint32_t>(), nseg, lb.as<uint32_t>(),
                                                                        le.as<uint32_t>(),
                                                                        nlong.as<unsigned long long>());
    const unsigned gl = unsigned(std::min<int64_t>(nl, int64_t(sm_count()) * 16));
    long_keys_kernel<<<gl, 256, 0, st>>>(pay_p, aj, lb.as<uint32_t>(), le.as<uint32_t>(), nl,
                                         keys.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    tb = 0;
    SPMV_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, keys.as<unsigned long long>(),
                                                     sorted.as<unsigned long long>(), nnz, nl, lb.as<uint32_t>(),
                                                     le.as<uint32_t>(), st));
    if ((r = tmp_for(tb))) return r;
    SPMV_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(tmp.ptr, tb, keys.as<unsigned long long>(),
                                                     sorted.as<unsigned long long>(), nnz, nl, lb.as<uint32_t>(),
                                                     le.as<uint32_t>(), st));
    long_emit_kernel<T><<<unsigned(grid_for(nseg)), 256, 0, st>>>(rows_p, sorted.as<unsigned long long>(),
                                                                  seg.as<uint32_t>(), nseg, av_p, ai_out, aj_out, av_out,
                                                                  ucnt.as<uint32_t>(), ndup.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));  // temporaries leave scope
  }
  unsigned long long hd = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&hd, ndup.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  *n_out = nnz - int64_t(hd);
  if (hd == 0) return SPMV_OK;
  return merge_duplicates<T>(seg.as<uint32_t>(), ucnt.as<uint32_t>(), nseg, nnz, ai_out, aj_out, av_out, st);
}

extern "C" int spmv_sort_coo(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* ai, const uint32_t* aj,
                  const void* av, uint32_t* ai_out, uint32_t* aj_out, void* av_out, int64_t* nnz_out, void* stream) {
  if (!nnz_out) return fail(SPMV_INVALID_ARG, "NULL output");
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nnz < 0 || nnz > int64_t(UINT32_MAX) - 1) return fail(SPMV_INVALID_ARG, "bad nnz");
  if (nrows < 1 || ncols < 1 || nrows > (int64_t(1) << 32) || ncols > (int64_t(1) << 32))
    return fail(SPMV_INVALID_ARG, "bad COO shape");
  if (nnz > 0 && (!ai || !aj || !av || !ai_out || !aj_out || !av_out)) return fail(SPMV_INVALID_ARG, "NULL pointer");
  cudaStream_t st = as_stream(stream);
  if (dtype == SPMV_F64)
    return sort_coo_run<double>(nrows, nnz, ai, aj, static_cast<const double*>(av), ai_out, aj_out,
                                static_cast<double*>(av_out), nnz_out, st);
  return sort_coo_run<float>(nrows, nnz, ai, aj, static_cast<const float*>(av), ai_out, aj_out,
                             static_cast<float*>(av_out), nnz_out, st);
}




