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

// ---- sort_coo ------------------------------------------------------------------
// Stage 1: a stable LSD radix sort of the 32-bit row keys (bits(nrows)
// bits) carrying each entry's storage index: each row's entries in storage
// order.  Stage 2: per row, its columns and values gathered through those
// indices and sorted by (column, storage index) — the reference's stable
// lexsort((cols, rows)) (convert.py:70) — written straight to the output
// positions (a warp per row of <= 32 entries: a bitonic sort in registers;
// longer rows: a segmented sort).  Stage 3, only when some (row, column)
// repeats: duplicate runs summed in np.add.reduceat order and compacted.

// flag = 1 if some row index is smaller than the one before it
__global__ void rows_descend_kernel(const uint32_t* __restrict__ ai, int64_t nnz, int* __restrict__ flag) {
  GRID_STRIDE(k, nnz) if (k > 0 && ai[k] < ai[k - 1]) *flag = 1;
}

// Rows of <= 32 entries: lane k holds entry k of the row, its payload
// (col << 32 | storage index); a bitonic sort of the payloads, then the
// value gathered through the storage index.  `pay` null: the rows were
// already in order, entry k's payload is built from aj[k] and k itself
// (no gathers at all).  Duplicate columns counted.
template <typename T>
__global__ void sort_rows_kernel(const uint32_t* __restrict__ rows_s, const unsigned long long* __restrict__ pay,
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

// Stage-1 payload: (col << 32 | storage index).
__global__ void sort_payload_kernel(const uint32_t* __restrict__ aj, int64_t nnz,
                                    unsigned long long* __restrict__ pay) {
  GRID_STRIDE(k, nnz) pay[k] = (static_cast<unsigned long long>(aj[k]) << 32) | static_cast<unsigned long long>(k);
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
  if (dtype == SPMV_F64)
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
    if (dtype == SPMV_F64)
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
    rc = c->counts.alloc(8 * nrows, st);
    if (!rc) rc = c->starts.alloc(8 * nrows, st);
    if (!rc) {
      const int W = dia_group_width(ndiags);
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
                                         nrows, st);
    if (!rc)
      rc = scan_total<unsigned long long>(c->counts.as<unsigned long long>(), c->starts.as<unsigned long long>(),
                                          nrows, st, &c->nnz);
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

template <typename T>
static int sort_coo_run(int64_t nrows, int64_t nnz, const uint32_t* ai, const uint32_t* aj, const T* av,
                        uint32_t* ai_out, uint32_t* aj_out, T* av_out, int64_t* n_out, cudaStream_t st) {
  *n_out = 0;
  if (nnz == 0) return SPMV_OK;
  int r;
  ScratchBuf pay_in, rows_buf, pay_buf, tmp, flag;
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
  if (!rows_sorted) {
    // stage 1: stable sort on the row, (col, storage index) as the payload
    if ((r = pay_in.alloc(8 * nnz, st)) || (r = pay_buf.alloc(8 * nnz, st)) || (r = rows_buf.alloc(4 * nnz, st)))
      return r;
    sort_payload_kernel<<<unsigned(grid_for(nnz)), 256, 0, st>>>(aj, nnz, pay_in.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    size_t tb = 0;
    SPMV_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, ai, rows_buf.as<uint32_t>(),
                                                  pay_in.as<unsigned long long>(), pay_buf.as<unsigned long long>(),
                                                  nnz, 0, bits_for(nrows), st));
    if ((r = tmp_for(tb))) return r;
    SPMV_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, ai, rows_buf.as<uint32_t>(),
                                                  pay_in.as<unsigned long long>(), pay_buf.as<unsigned long long>(),
                                                  nnz, 0, bits_for(nrows), st));
    pay_in.release();
    rows_p = rows_buf.as<uint32_t>();
    pay_p = pay_buf.as<unsigned long long>();
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
  sort_rows_kernel<T><<<unsigned(gw), 256, 0, st>>>(rows_p, pay_p, seg.as<uint32_t>(), nseg, aj, av, ai_out, aj_out,
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
                                                                  seg.as<uint32_t>(), nseg, av, ai_out, aj_out, av_out,
                                                                  ucnt.as<uint32_t>(), ndup.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));  // temporaries leave scope
  }
  unsigned long long hd = 0;
  SPMV_CUDA_TRY(cudaMemcpyAsync(&hd, ndup.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  *n_out = nnz - int64_t(hd);
  if (hd == 0) return SPMV_OK;
  // stage 3: duplicate runs merged and compacted (through a copy: rows move
  // to lower positions)
  ScratchBuf opos, ai_s, aj_s, av_s;
  if ((r = opos.alloc(4 * (nseg + 1), st)) || (r = ai_s.alloc(4 * nnz, st)) || (r = aj_s.alloc(4 * nnz, st)) ||
      (r = av_s.alloc(sizeof(T) * nnz, st)))
    return r;
  if ((r = excl_scan<uint32_t>(ucnt.as<uint32_t>(), opos.as<uint32_t>(), nseg + 1, st))) return r;
  SPMV_CUDA_TRY(cudaMemcpyAsync(ai_s.ptr, ai_out, 4 * nnz, cudaMemcpyDeviceToDevice, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(aj_s.ptr, aj_out, 4 * nnz, cudaMemcpyDeviceToDevice, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(av_s.ptr, av_out, sizeof(T) * nnz, cudaMemcpyDeviceToDevice, st));
  merge_runs_kernel<T><<<unsigned(grid_for(nseg)), 256, 0, st>>>(seg.as<uint32_t>(), opos.as<uint32_t>(), nseg,
                                                                 ai_s.as<uint32_t>(), aj_s.as<uint32_t>(), av_s.as<T>(),
                                                                 ai_out, aj_out, av_out);
  SPMV_LAUNCH_CHECK();
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  return SPMV_OK;
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




