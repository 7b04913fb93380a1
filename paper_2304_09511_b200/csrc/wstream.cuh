// Warp-stream SpMV for matrices whose x gathers are random (long rows,
// uniformly scattered columns: the Zipf config C3).
//
// Such a matrix is bound by the L1tex wavefront queue, not by HBM: every x
// gather is a random 32-byte L2 sector, one wavefront per lane, and an SM
// retires about one wavefront per cycle (B300_MICROARCH "L1tex wavefront
// queue"; tools/gather_ceiling.cu measures 240-250 G gathers/s on a B200
// for an index stream + value stream + one gather per entry).  The kernel
// is therefore built to issue nothing but the gathers on the LSU path:
//   * no shared-memory staging of the stream and no CTA barriers: the
//     entries are cut into contiguous ranges [b_w, b_w+1) (a few per warp,
//     handed out by an atomic counter) and a warp walks a range in chunks
//     of 32 x DEPTH entries, entry-per-lane (coalesced index/value loads,
//     DEPTH gathers in flight per lane);
//   * the rounded products go to a per-warp shared-memory buffer and each
//     row is summed from there: one lane per row, left to right, continuing
//     across chunks from a carried partial — the reference order
//     (kernels.py:69-82), bit-exact for every row that stays inside one
//     warp's range and has no chunk segment over kWsSeq entries;
//   * range boundaries snap back to a row start unless the row is longer
//     than exact_len, so only long rows are split between warps; their
//     per-warp partials (head/tail slots) are added in warp order by the
//     span fix-up kernel — deterministic, within 1e-12 (north_star);
//   * a chunk segment over kWsSeq entries (only rows over kWsSeq entries
//     have one) is summed by the whole warp (lane-strided, xor tree) and
//     added to the row's carry.
#pragma once

#include "common.cuh"

namespace spmv {

#ifndef SPMV_WS_DEPTH
#define SPMV_WS_DEPTH 8
#endif
#ifndef SPMV_WS_SEQ
#define SPMV_WS_SEQ 64
#endif
// COO keeps row indices and run state in registers: at 4 CTAs/SM it spills
// (56 B); 3 CTAs/SM without spills is 8% faster on C3 (CSR is faster at 4)
#ifndef SPMV_WS_COO_MINB
#define SPMV_WS_COO_MINB 3
#endif
#ifndef SPMV_WS_MINB
#define SPMV_WS_MINB 4
#endif
// matrix stream loads (column indices, values): read once, no L1 allocation
// (`__ldg` streams were 7% slower on C3, profiles/r1_notes.md)
template <typename T> __device__ __forceinline__ T ws_ld(const T* p) { return ld_stream(p); }
constexpr int kWsDepth = SPMV_WS_DEPTH;        // gathers in flight per lane
constexpr int kWsChunk = 32 * kWsDepth;        // entries per warp step
constexpr int kWsWarps = 8;                    // warps per CTA
constexpr uint32_t kWsSeq = SPMV_WS_SEQ;       // longest segment a lane sums alone

template <typename T>
struct WsParams {
  const uint32_t* irp;
  const uint32_t* aj;
  const T* av;
  const T* x;
  T* y;
  const uint32_t* bounds;  // nranges + 1 entry boundaries
  const uint32_t* row0;    // nranges: row containing bounds[w]
  double* head;            // nranges: partial of a row that started before bounds[w]
  double* tail;            // nranges: partial of a row that continues past bounds[w+1]
  uint32_t* ctr;           // [next range - nwarps, warps done]; zero between launches
  int64_t nrows, col_base, nwarps, nranges;
  uint32_t exact_len;
  const uint32_t* ymap;    // row r is y[ymap[r]] (the panel path's short-row CSR); nullptr else
};

template <typename T>
__device__ __forceinline__ int64_t ws_yrow(const WsParams<T>& P, int64_t r) {
  return P.ymap ? int64_t(P.ymap[r]) : r;
}

// Row sums accumulate in double.  f64: the plain rounded sum.  f32: rows of
// at most exact_len entries add in float (every partial is a float, so this
// is the reference's f32 left-to-right sum, bit-exact); longer rows keep a
// double partial and round once at the end — no worse than the reference
// against the exact sum (the f32 bar is 1e-5 against the
// f64-evaluated product).
__device__ __forceinline__ double ws_add(double s, double p, bool) { return __dadd_rn(s, p); }
__device__ __forceinline__ double ws_add(double s, float p, bool exact) {
  return exact ? double(__fadd_rn(float(s), p)) : __dadd_rn(s, double(p));
}

// One entry range [bounds[w], bounds[w+1]) walked by one warp.
template <typename T>
__device__ __forceinline__ void csr_ws_range(const WsParams<T>& P, const int64_t w, T* __restrict__ prod,
                                             const int lane) {
  const uint32_t b0 = __ldg(P.bounds + w), b1 = __ldg(P.bounds + w + 1);
  if (b0 >= b1) return;
  const T* xb = P.x - P.col_base;
  const double neg0 = -0.0;

  int64_t r = __ldg(P.row0 + w);      // current row (contains entry c0)
  uint32_t rs = __ldg(P.irp + r);     // its start
  bool head = rs < b0;                // started in an earlier warp's range
  double carry = neg0;                // its partial over earlier chunks (see ws_add)

  // column indices run one chunk ahead: their HBM latency overlaps the
  // previous chunk's gathers and row sums
  uint32_t col[kWsDepth];
#pragma unroll
  for (int k = 0; k < kWsDepth; ++k) {
    const uint32_t e = b0 + k * 32 + lane;
    col[k] = e < b1 ? ws_ld(P.aj + e) : 0u;
  }
  for (uint32_t c0 = b0, c1; c0 < b1; c0 = c1) {
    c1 = b1 - c0 > uint32_t(kWsChunk) ? c0 + uint32_t(kWsChunk) : b1;  // no uint32 wrap near 2^32 entries
    // row ends of the next 32 rows: issued first, consumed after the gathers
    uint32_t end = r + lane < P.nrows ? __ldg(P.irp + r + lane + 1) : 0xffffffffu;
    T p[kWsDepth];
    {
      T val[kWsDepth];
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) {
        const uint32_t e = c0 + k * 32 + lane;
        val[k] = e < c1 ? ws_ld(P.av + e) : T(0);
      }
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) p[k] = (c0 + k * 32 + lane < c1) ? ldx(xb + col[k]) : T(0);
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) {
        const uint32_t e = c1 + k * 32 + lane;
        col[k] = (c1 < b1 && e < b1 && e >= c1) ? ws_ld(P.aj + e) : 0u;
      }
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) p[k] = mul_rn(val[k], p[k]);
    }
    const uint32_t end0 = __shfl_sync(0xffffffffu, end, 0);
    if (end0 >= c1 && c1 - c0 == uint32_t(kWsChunk)) {
      // the whole chunk lies in row r (so the row has over kWsChunk entries):
      // lane partials in k order, xor tree, added to the carry — no shared
      // memory round trip
      double part = p[0];
#pragma unroll
      for (int k = 1; k < kWsDepth; ++k) part = add_rn(part, double(p[k]));
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) part = add_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
      carry = add_rn(carry, part);
      if (end0 == c1) {  // row r ends exactly here
        if (lane == 0) {
          if (head)
            P.head[w] = carry;
          else
            P.y[ws_yrow(P, r)] = T(carry);
        }
        r += 1;
        rs = c1;
        head = false;
        carry = neg0;
      }
      continue;
    }
#pragma unroll
    for (int k = 0; k < kWsDepth; ++k) prod[k * 32 + lane] = p[k];
    __syncwarp();

    // rows of the chunk, 32 at a time: lane l sums row r + l's segment
    while (true) {
      uint32_t start = __shfl_up_sync(0xffffffffu, end, 1);
      if (lane == 0) start = rs;
      const bool fin = end <= c1;  // invalid lanes have end = UINT32_MAX
      const int nfin = __popc(__ballot_sync(0xffffffffu, fin));
      const bool active = lane <= nfin && r + lane < P.nrows;
      const uint32_t lo = max(start, c0), hi = min(end, c1);
      const uint32_t len = (active && hi > lo) ? hi - lo : 0u;
      const bool exact = end - start <= P.exact_len;
      double s = lane == 0 ? carry : neg0;
      if (len <= kWsSeq) {
        const T* pp = prod + (lo - c0);
        for (uint32_t i = 0; i < len; ++i) s = ws_add(s, pp[i], exact);
      }
      unsigned longs = __ballot_sync(0xffffffffu, len > kWsSeq);
      while (longs) {
        const int L = __ffs(longs) - 1;
        longs &= longs - 1;
        const uint32_t llo = __shfl_sync(0xffffffffu, lo, L) - c0;
        const uint32_t llen = __shfl_sync(0xffffffffu, len, L);
        double part = neg0;
        for (uint32_t i = lane; i < llen; i += 32) part = add_rn(part, double(prod[llo + i]));
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) part = add_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
        if (lane == L) s = add_rn(s, part);
      }
      if (fin && active && end > start) {
        if (lane == 0 && head)
          P.head[w] = s;
        else
          P.y[ws_yrow(P, r + lane)] = T(s);
      }
      if (nfin < 32) {
        // lane nfin's row continues into the next chunk (or is past nrows)
        carry = __shfl_sync(0xffffffffu, s, nfin);
        rs = __shfl_sync(0xffffffffu, start, nfin);
        if (nfin > 0) head = false;
        r += nfin;
        break;
      }
      // all 32 rows finished inside the chunk: next 32 rows
      rs = __shfl_sync(0xffffffffu, end, 31);
      r += 32;
      head = false;
      carry = neg0;
      if (rs >= c1 || r >= P.nrows) break;
      end = r + lane < P.nrows ? __ldg(P.irp + r + lane + 1) : 0xffffffffu;
    }
    __syncwarp();
  }
  // a row still open at the end of the range continues in the next warp
  if (lane == 0 && r < P.nrows && rs < b1) {
    const uint32_t re = __ldg(P.irp + r + 1);
    if (re > b1) {
      if (head)
        P.head[w] = carry;
      else
        P.tail[w] = carry;
    }
  }
}

// Persistent warps over nranges ranges: warp w starts on range w, then takes
// ranges nwarps, nwarps+1, ... from an atomic counter (uneven row work
// evens out).  The last warp to finish resets the counters for the next
// launch (stream order), so a plan must not run on two streams at once.
template <typename T>
__global__ void __launch_bounds__(kWsWarps * 32, SPMV_WS_MINB) csr_wstream_kernel(const __grid_constant__ WsParams<T> P) {
  __shared__ T s_prod[kWsWarps][kWsChunk];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t w = int64_t(blockIdx.x) * kWsWarps + wid;
  if (w >= P.nwarps) return;
  for (int64_t q = w; q < P.nranges;) {
    csr_ws_range(P, q, s_prod[wid], lane);
    uint32_t nq = 0;
    if (lane == 0) nq = atomicAdd(P.ctr, 1u);
    q = P.nwarps + int64_t(__shfl_sync(0xffffffffu, nq, 0));
  }
  if (lane == 0 && atomicAdd(P.ctr + 1, 1u) == uint32_t(P.nwarps - 1)) {
    atomicExch(P.ctr, 0u);
    atomicExch(P.ctr + 1, 0u);
  }
}

// Rows split between ranges: y = tail[w0] + head[w0+1] + ... + head[w1],
// one warp per row: lane l sums partials l, l+32, ... in order, then a fixed
// xor tree (deterministic; these rows are longer than exact_len).  COO plans
// list runs (run_row maps a run to its row); CSR passes nullptr.
template <typename T>
__global__ void ws_span_fixup_kernel(const uint32_t* __restrict__ span_row, const uint32_t* __restrict__ span_w0,
                                     const uint32_t* __restrict__ span_w1, int64_t n_span,
                                     const double* __restrict__ head, const double* __restrict__ tail,
                                     T* __restrict__ y, const uint32_t* __restrict__ run_row = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n_span; i += nw) {
    const uint32_t w0 = span_w0[i], w1 = span_w1[i];
    double sum = -0.0;
    for (uint32_t u = w0 + lane; u <= w1; u += 32) sum = __dadd_rn(sum, u == w0 ? tail[u] : head[u]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
    if (lane == 0) y[run_row ? run_row[span_row[i]] : span_row[i]] = T(sum);
  }
}

// Warp ranges: target entry t = w*nnz/nwarps, snapped back to the start of
// its row unless that row is longer than exact_len.  row0[w] is the row
// containing bounds[w] (the last row whose start is <= it).
static __global__ void ws_bounds_kernel(const uint32_t* __restrict__ irp, int64_t nrows, int64_t nnz, int64_t nwarps,
                                 int exact_len, uint32_t* __restrict__ bounds, uint32_t* __restrict__ row0) {
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w <= nwarps; w += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t t = uint64_t(w) * uint64_t(nnz) / uint64_t(nwarps);
    if (w == nwarps || t >= uint64_t(nnz)) {
      bounds[w] = uint32_t(nnz);
      if (w < nwarps) row0[w] = uint32_t(nrows);
      continue;
    }
    int64_t lo = 0, hi = nrows - 1;  // last r with irp[r] <= t
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (uint64_t(irp[mid]) <= t) lo = mid; else hi = mid - 1;
    }
    const uint32_t s = irp[lo], e = irp[lo + 1];
    bounds[w] = (e - s <= uint32_t(exact_len)) ? s : uint32_t(t);
    row0[w] = uint32_t(lo);
  }
}

// Long rows split between warp ranges: (row, first warp, last warp).
static __global__ void ws_span_list_kernel(const uint32_t* __restrict__ irp, int64_t nrows, int exact_len,
                                    const uint32_t* __restrict__ bounds, int64_t nwarps,
                                    uint32_t* __restrict__ span_row, uint32_t* __restrict__ span_w0,
                                    uint32_t* __restrict__ span_w1, unsigned long long* __restrict__ n_span) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = irp[r], e = irp[r + 1];
    if (e - s <= uint32_t(exact_len)) continue;
    // last w with bounds[w] <= key (skips empty ranges)
    auto warp_of = [&](uint32_t key) {
      int64_t lo = 0, hi = nwarps - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (bounds[mid] <= key) lo = mid; else hi = mid - 1;
      }
      return lo;
    };
    const int64_t w0 = warp_of(s), w1 = warp_of(e - 1);
    if (w0 == w1) continue;
    const unsigned long long k = atomicAdd(n_span, 1ull);
    if (span_row) {
      span_row[k] = uint32_t(r);
      span_w0[k] = uint32_t(w0);
      span_w1[k] = uint32_t(w1);
    }
  }
}

static __global__ void count_empty_rows_kernel(const uint32_t* __restrict__ irp, int64_t nrows,
                                        unsigned long long* __restrict__ n_empty) {
  unsigned long long c = 0;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x)
    c += irp[r + 1] == irp[r];
  for (int o = 16; o >= 1; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(n_empty, c);
}

// ---- COO ------------------------------------------------------------------
// The same warp-stream scheme over a row-sorted COO stream
// (spmv_coo_plain, kernels.py:56-66: y = 0, then y[ai[j]] += av[j]*x[aj[j]]
// in storage order).  Row boundaries come from the row indices themselves:
// per chunk, ballots over ai[j] != ai[j-1] give a 256-bit map of run
// starts; lane l takes the l-th run segment (__fns select), sums its
// products left to right from +0.0 (np.add.at order) or continues the
// carried run.  Ranges snap to run starts unless a run is longer than
// exact_len (plan: run_start / run_row), so short runs stay whole.
//
// f32: a run's length is only known at its end, so a segment sum keeps both
// a float (the reference's rounding, used when the run has <= exact_len
// entries: bit-exact) and a double partial (used for longer runs).
template <typename T>
struct RunAcc;
template <>
struct RunAcc<double> {
  double d;
  __device__ __forceinline__ void set(double v, double) { d = v; }
  __device__ __forceinline__ void add(double p) { d = __dadd_rn(d, p); }
  __device__ __forceinline__ void add_wide(double v) { d = __dadd_rn(d, v); }
  __device__ __forceinline__ double exact() const { return d; }
  __device__ __forceinline__ void shfl(int src) { d = __shfl_sync(0xffffffffu, d, src); }
};
template <>
struct RunAcc<float> {
  double d;
  float f;
  __device__ __forceinline__ void set(double v, float g) { d = v; f = g; }
  __device__ __forceinline__ void add(float p) { d = __dadd_rn(d, double(p)); f = __fadd_rn(f, p); }
  __device__ __forceinline__ void add_wide(double v) { d = __dadd_rn(d, v); }
  __device__ __forceinline__ float exact() const { return f; }
  __device__ __forceinline__ void shfl(int src) {
    d = __shfl_sync(0xffffffffu, d, src);
    f = __shfl_sync(0xffffffffu, f, src);
  }
};

template <typename T>
struct CooWsParams {
  const uint32_t* ai;
  const uint32_t* aj;
  const T* av;
  const T* x;
  T* y;
  const uint32_t* bounds;  // nranges + 1
  double* head;
  double* tail;
  uint32_t* ctr;
  int64_t col_base, nwarps, nranges, nnz;
  uint32_t exact_len;
};

// position of the i-th set bit of the 256-bit map m[0..7] (pre = prefix
// popcounts); i < total
template <int D>
__device__ __forceinline__ uint32_t ws_select(const unsigned (&m)[D], const int (&pre)[D], int i) {
  int k = 0;
#pragma unroll
  for (int q = 1; q < D; ++q) k += i >= pre[q];
  unsigned mk = m[0];
  int base = pre[0];
#pragma unroll
  for (int q = 1; q < D; ++q)
    if (k == q) {
      mk = m[q];
      base = pre[q];
    }
  return uint32_t(k * 32) + __fns(mk, 0, i - base + 1);
}

template <typename T>
__device__ __forceinline__ void coo_ws_range(const CooWsParams<T>& P, const int64_t w, T* __restrict__ prod,
                                             uint32_t* __restrict__ rows_s, const int lane) {
  const uint32_t b0 = __ldg(P.bounds + w), b1 = __ldg(P.bounds + w + 1);
  if (b0 >= b1) return;
  const T* xb = P.x - P.col_base;
  // carried run: row crow, partial acc over clen entries of this range;
  // chead = it started before b0 (its partial goes to head[w])
  uint32_t crow = b0 > 0 ? __ldg(P.ai + b0 - 1) : 0xffffffffu;
  bool chead = true;
  uint32_t clen = 0;
  RunAcc<T> acc;
  acc.set(0.0, T(0));

  uint32_t col[kWsDepth];
#pragma unroll
  for (int k = 0; k < kWsDepth; ++k) {
    const uint32_t e = b0 + k * 32 + lane;
    col[k] = e < b1 ? ws_ld(P.aj + e) : 0u;
  }
  for (uint32_t c0 = b0, c1; c0 < b1; c0 = c1) {
    c1 = b1 - c0 > uint32_t(kWsChunk) ? c0 + uint32_t(kWsChunk) : b1;
    const uint32_t n = c1 - c0;
    uint32_t row[kWsDepth];
    T p[kWsDepth];
    {
      T val[kWsDepth];
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) {
        const uint32_t e = c0 + k * 32 + lane;
        const bool ok = e < c1;
        row[k] = ok ? ws_ld(P.ai + e) : 0xffffffffu;
        val[k] = ok ? ws_ld(P.av + e) : T(0);
      }
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) p[k] = (c0 + k * 32 + lane < c1) ? ldx(xb + col[k]) : T(0);
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) {
        const uint32_t e = c1 + k * 32 + lane;
        col[k] = (c1 < b1 && e < b1 && e >= c1) ? ws_ld(P.aj + e) : 0u;
      }
#pragma unroll
      for (int k = 0; k < kWsDepth; ++k) p[k] = mul_rn(val[k], p[k]);
    }
    // run-start map; bit 0 is always a segment start (new run or the carry)
    unsigned m[kWsDepth];
    int pre[kWsDepth];
    int nseg = 0;
    const uint32_t last_prev = crow;
#pragma unroll
    for (int k = 0; k < kWsDepth; ++k) {
      uint32_t prev = __shfl_up_sync(0xffffffffu, row[k], 1);
      const uint32_t wrap = __shfl_sync(0xffffffffu, k == 0 ? last_prev : row[k > 0 ? k - 1 : 0], 31);
      if (lane == 0) prev = k == 0 ? last_prev : wrap;
      const bool ok = uint32_t(k * 32 + lane) < n;
      m[k] = __ballot_sync(0xffffffffu, ok && (row[k] != prev || (k == 0 && lane == 0)));
      pre[k] = nseg;
      nseg += __popc(m[k]);
    }
    const bool cont = __shfl_sync(0xffffffffu, row[0], 0) == crow;  // entry c0 continues the carried run
    if (!cont && clen > 0 && lane == 0) {
      // the carried run ended at c0
      const T v = clen <= P.exact_len ? T(acc.exact()) : T(acc.d);
      if (chead)
        P.head[w] = acc.d;
      else
        P.y[crow] = v;
    }
    if (nseg == 1 && cont && n == uint32_t(kWsChunk)) {
      // the whole chunk continues the carried run (> kWsChunk entries): lane
      // partials, xor tree, no shared memory
      double part = p[0];
#pragma unroll
      for (int k = 1; k < kWsDepth; ++k) part = __dadd_rn(part, double(p[k]));
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
      acc.add_wide(part);
      clen += n;
      continue;
    }
#pragma unroll
    for (int k = 0; k < kWsDepth; ++k) {
      prod[k * 32 + lane] = p[k];
      rows_s[k * 32 + lane] = row[k];
    }
    __syncwarp();
    for (int g0 = 0; g0 < nseg; g0 += 32) {
      const int i = g0 + lane;
      const bool valid = i < nseg;
      const uint32_t lo = valid ? ws_select(m, pre, i) : n;
      const uint32_t hi = i + 1 < nseg ? ws_select(m, pre, i + 1) : n;
      const uint32_t len = hi - lo;
      const bool carried = i == 0 && cont;
      RunAcc<T> s;
      s.set(0.0, T(0));
      if (carried) s = acc;
      const uint32_t rlen = (carried ? clen : 0u) + len;  // run length so far
      if (valid && len <= kWsSeq) {
        const T* pp = prod + lo;
        for (uint32_t t = 0; t < len; ++t) s.add(pp[t]);
      }
      unsigned longs = __ballot_sync(0xffffffffu, valid && len > kWsSeq);
      while (longs) {
        const int L = __ffs(longs) - 1;
        longs &= longs - 1;
        const uint32_t llo = __shfl_sync(0xffffffffu, lo, L), llen = __shfl_sync(0xffffffffu, len, L);
        double part = -0.0;
        for (uint32_t t = lane; t < llen; t += 32) part = __dadd_rn(part, double(prod[llo + t]));
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
        if (lane == L) s.add_wide(part);
      }
      const uint32_t srow = valid ? rows_s[lo] : 0u;
      if (valid && i + 1 < nseg) {  // the run ends inside the chunk
        if (carried && chead)
          P.head[w] = s.d;
        else
          P.y[srow] = rlen <= P.exact_len ? T(s.exact()) : T(s.d);
      }
      const int lastl = (nseg - 1) - g0;  // lane holding the last segment, if in this group
      if (lastl < 32) {
        s.shfl(lastl);
        acc = s;
        crow = __shfl_sync(0xffffffffu, srow, lastl);
        clen = __shfl_sync(0xffffffffu, rlen, lastl);
        if (nseg > 1 || !cont) chead = false;
      }
    }
    __syncwarp();
  }
  // the carried run: ends at b1 or continues into the next range
  if (lane == 0 && clen > 0) {
    const bool more = b1 < uint64_t(P.nnz) && __ldg(P.ai + b1) == crow;
    if (chead)
      P.head[w] = acc.d;
    else if (more)
      P.tail[w] = acc.d;
    else
      P.y[crow] = clen <= P.exact_len ? T(acc.exact()) : T(acc.d);
  }
}

template <typename T>
__global__ void __launch_bounds__(kWsWarps * 32, SPMV_WS_COO_MINB) coo_wstream_kernel(const __grid_constant__ CooWsParams<T> P) {
  __shared__ T s_prod[kWsWarps][kWsChunk];
  __shared__ uint32_t s_rows[kWsWarps][kWsChunk];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int64_t w = int64_t(blockIdx.x) * kWsWarps + wid;
  if (w >= P.nwarps) return;
  for (int64_t q = w; q < P.nranges;) {
    coo_ws_range(P, q, s_prod[wid], s_rows[wid], lane);
    uint32_t nq = 0;
    if (lane == 0) nq = atomicAdd(P.ctr, 1u);
    q = P.nwarps + int64_t(__shfl_sync(0xffffffffu, nq, 0));
  }
  if (lane == 0 && atomicAdd(P.ctr + 1, 1u) == uint32_t(P.nwarps - 1)) {
    atomicExch(P.ctr, 0u);
    atomicExch(P.ctr + 1, 0u);
  }
}

}  // namespace spmv
