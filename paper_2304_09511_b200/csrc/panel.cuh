// Column-panel kernel for the long rows of random-column matrices (the
// Zipf config C3): their x gathers move from random L2 sectors into shared
// memory.
//
// Why: with uniformly random columns every x gather of the row-order
// kernels is one random 32-byte L2 sector, one L1tex wavefront per lane
// (about one per cycle per SM: tools/gather_ceiling.cu, ~248 G gathers/s on
// a B200), so C3 ran at 0.40 of HBM bandwidth with HBM mostly idle.
// Shared memory serves a warp of 32 random 8-byte reads in a few
// bank-conflict wavefronts instead of 32.
//
// Layout (built once per matrix by the plan, csr.cu csr_panel_build): the
// entries of the long rows (over `row_len` entries, plan default 128; 78%
// of C3's entries) are grouped by column panel — panel q holds columns
// [q*W, (q+1)*W), W chosen by the plan so that the panel count divides (or
// is a multiple of) the SM count and the x panel plus the warps' stream
// stages fit shared memory.  A (row, panel) run is a segment; a segment of
// more than kPanelH entries is cut into sub-segments of kPanelH.  Inside a
// panel the sub-segments are sorted by length (longest first) and put side
// by side, 32 at a time, one per lane: a *slice* (sliced ELL, one warp
// wide).  A slice is as many entry-rows as its longest sub-segment;
// shorter lanes are padded with (value 0, column W) entries and xs[W] = 0.
// So a lane just adds its products left to right — no segment flags,
// selects or scans in the hot loop (the first version's flagged stream
// spent 377 instructions per 256 entries on them and was ALU-bound) — and
// at a slice's last entry-row the 32 lanes store their 32 partials side by
// side.
//
// Stream: a warp task's slices are laid end to end and padded to whole
// steps of kPanelK = 8 entry-rows (256 entries).  Per step: the values,
// entry-row k lane l at [k * 32 + l] (conflict-free LDS.64); the 16-bit
// panel columns lane-contiguous (lane l's 8 columns in one 16-byte word:
// one LDS.128) followed by a 16-byte header whose first byte has bit k set
// when entry-row k ends a slice.  Both pieces are TMA bulk copies into the
// warp's own stage ring (2-4 stages deep), refilled as soon as a step is in
// registers.
//
// Kernel: one CTA per SM, warp-specialised.  kPanelWarps panel warps take a
// contiguous range of slices (equal entry-rows; cuts snapped to panel
// boundaries when close, so with C3's 148 panels every CTA loads exactly
// one x panel); for each panel the range touches they load the x panel
// into shared memory (one TMA bulk copy) while prefetching their first
// steps.  This side is an HBM stream.  kGatherWarps gather warps compute
// the rows of at most `row_len` entries in row order at the same time:
// those rows, grouped by exact length into column-major ELL classes, go
// one thread per row, left to right, with x gathered through L1 —
// bit-exact with the reference order, and bound by the L1 sector rate, not
// HBM, so the two sides overlap instead of queueing (as separate launches
// they took 43 + 62 us on C3).  A 50-entry row would otherwise leave ~45
// one-entry segments in the panel stream, each with its own partial: rows
// of 33..128 entries hold 8% of C3's entries but made 45% of the partials.
// Blocks of rows are handed out longest class first by an atomic counter.
//
// Results: each long row = its sub-segments' partials added in panel order
// by csr_panel_finish_kernel (a warp per row), each partial a
// left-to-right sum — deterministic, within 1e-12 of the reference's
// left-to-right sum (north_star allows that for rows over 32 entries; rows
// of <= row_len entries never come here and stay bit-exact).  f32:
// products rounded to f32 as in the reference, partials and the final sum
// in double, rounded once (the same contract as the warp-stream path).
#pragma once

#include "tma.cuh"

namespace spmv {

constexpr int kPanelWarps = 12;           // panel (stream) warps per CTA (one CTA per SM)
constexpr int kGatherWarps = 12;          // gather (short-row) warps per CTA
constexpr int kPanelThreads = (kPanelWarps + kGatherWarps) * 32;
constexpr int kRowLenMax = 256;           // longest row the gather side can take
constexpr int kRowLenDefault = 128;
constexpr int kPanelK = 8;                // entry-rows per step
constexpr int kPanelStep = 32 * kPanelK;  // entries per warp step
constexpr int kPanelH = 32;               // entry-rows per slice at most (longer segments are cut)
constexpr int kPanelColBytes = kPanelStep * 2 + 16;  // a step's columns + header
constexpr int kPanelMaxStages = 4;
constexpr int kPanelHeader = 1024;  // mbarriers: [0] panel, [1 + w * kPanelMaxStages + s] warp w's stage s
constexpr int kPanelSmemMax = 232448;
static_assert((1 + kPanelWarps * kPanelMaxStages) * 8 <= kPanelHeader, "panel mbarriers");
static_assert(kPanelH <= 64, "sub-segment length in 6 key bits");
template <typename T> constexpr int panel_stage_bytes() {
  return int(align_up(kPanelStep * sizeof(T) + kPanelColBytes, 128));
}
// shared memory of a launch: header, stage rings, x panel of W columns + the zero slot
template <typename T> constexpr int64_t panel_smem_bytes(int64_t W, int nstg) {
  return kPanelHeader + int64_t(kPanelWarps) * nstg * panel_stage_bytes<T>() +
         int64_t(align_up(size_t(W + 1) * sizeof(T), 16));
}
// widest panel with `nstg` stages per warp (a multiple of 4, so panels start 16-byte aligned)
template <typename T> constexpr int64_t panel_max_cols(int nstg) {
  const int64_t w = (kPanelSmemMax - kPanelHeader - int64_t(kPanelWarps) * nstg * panel_stage_bytes<T>()) /
                        int64_t(sizeof(T)) - 4;
  return (w < 65532 ? w : 65532) / 4 * 4;
}

template <typename T>
struct PanelParams {
  const uint8_t* pcol;  // per step kPanelColBytes: 256 u16 panel columns (lane-contiguous), 16-byte header
  const T* pval;        // per step 256 values, entry-row k lane l at k * 32 + l
  const T* x;           // x window: global column c at x[c - col_base]
  int64_t col_base, x_len, ncols;
  int32_t panel_cols, nstg;
  const uint32_t* cta_item;    // CTA c: items [cta_item[c], cta_item[c+1])
  const uint32_t* item_panel;
  const uint32_t* task;        // kPanelWarps per item, 3 words each: first step, steps, first slice
  double* part;                // partials: slice s lane l at s * 32 + l
  T* y;
  // gather side: rows of <= row_len entries by exact length class L, class L
  // column-major from ebase[L] (entry j of the class's r-th row at
  // ebase[L] + j * n_L + r); srow: the rows, classes ascending
  const uint32_t* blk;    // per block, longest class first: L << 23 | (first row within the class) / 32
  const uint32_t* cls;    // [L]: first row of class L in srow; [row_len + 1] = end
  const uint32_t* ebase;  // [L]
  const uint32_t* scol;
  const T* sval;
  const uint32_t* srow;
  uint32_t nblk, gather_warps;  // blocks; gather warps in the grid
  uint32_t* ctr;                // [0] next block, [1] warps done (zero between launches)
  int32_t pos_seed;             // rows start from +0.0 (COO order) instead of -0.0
};

template <typename T> __device__ __forceinline__ double panel_prod(T v, T x) { return double(mul_rn(v, x)); }

// Position of entry-row k, lane l inside a step's column block (u16 index) / value block.
__host__ __device__ __forceinline__ uint32_t panel_col_pos(uint32_t k, uint32_t lane) { return lane * kPanelK + k; }
__host__ __device__ __forceinline__ uint32_t panel_val_pos(uint32_t k, uint32_t lane) { return k * 32 + lane; }

template <typename T>
__device__ __forceinline__ void panel_issue(unsigned char* stage, uint64_t* bar, const uint8_t* __restrict__ pcol,
                                            const T* __restrict__ pval, uint32_t step) {
  constexpr uint32_t vb = kPanelStep * sizeof(T);
  mbar_arrive_expect_tx(bar, vb + kPanelColBytes);
  bulk_g2s(stage, pval + size_t(step) * kPanelStep, vb, bar, true);
  bulk_g2s(stage + vb, pcol + size_t(step) * kPanelColBytes, kPanelColBytes, bar, true);
}

// One warp's task: steps [step0, step0 + n) of the stream, whole slices
// from slice0 on; its first min(n, nstg) steps were issued by the caller.
// (Storing the partials straight to row-major slots instead — scattered
// 8-byte stores — took the kernel from 62 to 115 us: profiles/r2_notes.md.)
template <typename T>
__device__ __forceinline__ void panel_task(const PanelParams<T>& P, const T* __restrict__ xs, unsigned char* stages,
                                           uint64_t* bars, uint32_t& phases, uint32_t step0, uint32_t n,
                                           uint32_t slice0, int lane) {
  constexpr uint32_t vb = kPanelStep * sizeof(T);
  const int nstg = P.nstg;
  double acc = -0.0;
  double* out = P.part + size_t(slice0) * 32 + lane;
  int s = 0;
  for (uint32_t i = 0; i < n; ++i) {
    unsigned char* stg = stages + s * panel_stage_bytes<T>();
    mbar_wait(&bars[s], (phases >> s) & 1u);
    phases ^= 1u << s;
#ifdef SPMV_DEBUG_CHECKS
    {  // the stage holds exactly this step (no ring race), columns inside the panel
      const T* gv = P.pval + size_t(step0 + i) * kPanelStep;
      const uint16_t* gc = reinterpret_cast<const uint16_t*>(P.pcol + size_t(step0 + i) * kPanelColBytes);
      const T* vs = reinterpret_cast<const T*>(stg);
      const uint16_t* cs = reinterpret_cast<const uint16_t*>(stg + vb);
      for (int k = lane; k < kPanelStep; k += 32) {
        SPMV_DCHECK(same_bits(vs[k], gv[k]), 0);
        SPMV_DCHECK(cs[k] == gc[k], 0);
        SPMV_DCHECK(int(cs[k]) <= P.panel_cols, 1);
      }
      SPMV_DCHECK(stg[vb + kPanelStep * 2] == P.pcol[size_t(step0 + i) * kPanelColBytes + kPanelStep * 2], 0);
    }
#endif
    T v[kPanelK];
    const T* vs = reinterpret_cast<const T*>(stg);
#pragma unroll
    for (int k = 0; k < kPanelK; ++k) v[k] = vs[k * 32 + lane];
    const uint4 cw = *reinterpret_cast<const uint4*>(stg + vb + lane * 16);
    const uint32_t hdr = stg[vb + kPanelStep * 2];
    __syncwarp();
    if (lane == 0 && i + uint32_t(nstg) < n) {
      fence_proxy_async();
      panel_issue<T>(stg, &bars[s], P.pcol, P.pval, step0 + i + uint32_t(nstg));
    }
    s = s + 1 == nstg ? 0 : s + 1;
    const uint32_t cc[4] = {cw.x, cw.y, cw.z, cw.w};
    double p[kPanelK];
#pragma unroll
    for (int k = 0; k < kPanelK; ++k) {
      const uint32_t c = (k & 1) ? (cc[k >> 1] >> 16) : (cc[k >> 1] & 0xffffu);
      p[k] = panel_prod(v[k], xs[c]);
    }
    if (hdr == 0) {
#pragma unroll
      for (int k = 0; k < kPanelK; ++k) acc = __dadd_rn(acc, p[k]);
    } else {
#pragma unroll
      for (int k = 0; k < kPanelK; ++k) {
        acc = __dadd_rn(acc, p[k]);
        if ((hdr >> k) & 1u) {
          *out = acc;
          out += 32;
          acc = -0.0;
        }
      }
    }
  }
}

__device__ __forceinline__ void panel_bar_sync() {  // the panel warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kPanelWarps * 32) : "memory");
}

// ---- gather side --------------------------------------------------------------
// Rows per thread: the 1-4 entry rows (most of a Zipf matrix's rows) keep 8
// gathers in flight per thread by taking several rows at once.
__host__ __device__ constexpr int short_rows_per_thread(int L) { return L <= 1 ? 8 : L == 2 ? 4 : L <= 4 ? 2 : 1; }

// U rows of LL entries per thread, everything in flight at once; each row
// summed left to right from `seed`.
template <typename T, int U, int LL>
__device__ __forceinline__ void short_rows_fixed(const uint32_t* __restrict__ cp, const T* __restrict__ vp,
                                                 const uint32_t* __restrict__ rows, uint32_t n, uint32_t r0, int lane,
                                                 const T* __restrict__ xb, T* __restrict__ y, T seed) {
  uint32_t c[U][LL], dst[U];
  T v[U][LL], xv[U][LL];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t r = min(r0 + uint32_t(u) * 32 + uint32_t(lane), n - 1);  // clamped: the store is predicated
    dst[u] = __ldcs(rows + r);
#pragma unroll
    for (int j = 0; j < LL; ++j) {
      c[u][j] = __ldcs(cp + uint32_t(j) * n + r);
      v[u][j] = __ldcs(vp + uint32_t(j) * n + r);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int j = 0; j < LL; ++j) xv[u][j] = ldx(xb + c[u][j]);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    T acc = seed;
#pragma unroll
    for (int j = 0; j < LL; ++j) acc = add_rn(acc, mul_rn(v[u][j], xv[u][j]));
    if (r0 + uint32_t(u) * 32 + uint32_t(lane) < n) y[dst[u]] = acc;
  }
}

// One block: 32 * short_rows_per_thread(L) rows of class L from row r0 of
// the class.  One thread per row, its entries left to right from -0.0
// (cumsum order, kernels.py:81: bit-exact) or, for COO plans (pos_seed),
// from +0.0 (np.add.at on a zeroed y, kernels.py:65); empty rows +0.0.  The
// warp's rows share their length, so its loops are uniform; loads are
// coalesced (column-major classes), 8 gathers in flight per thread.
template <typename T>
__device__ __forceinline__ void gather_block(const PanelParams<T>& P, uint32_t desc, int lane, const T* __restrict__ xb,
                                             T seed) {
  const int L = int(desc >> 23);
  const uint32_t r0 = (desc & 0x7fffffu) * 32u;
  const uint32_t c0 = __ldg(P.cls + L), n = __ldg(P.cls + L + 1) - c0, eb = __ldg(P.ebase + L);
  const uint32_t* cp = P.scol + eb;
  const T* vp = P.sval + eb;
  const uint32_t* rows = P.srow + c0;
  T* __restrict__ y = P.y;
  switch (L) {
    case 1: short_rows_fixed<T, 8, 1>(cp, vp, rows, n, r0, lane, xb, y, seed); return;
    case 2: short_rows_fixed<T, 4, 2>(cp, vp, rows, n, r0, lane, xb, y, seed); return;
    case 3: short_rows_fixed<T, 2, 3>(cp, vp, rows, n, r0, lane, xb, y, seed); return;
    case 4: short_rows_fixed<T, 2, 4>(cp, vp, rows, n, r0, lane, xb, y, seed); return;
    default: break;
  }
  const uint32_t r = r0 + uint32_t(lane);
  if (r >= n) return;
  cp += r;
  vp += r;
  const uint32_t dst = __ldcs(rows + r);
  T acc = seed;
  int j = 0;
  for (; j + 8 <= L; j += 8) {
    uint32_t c[8];
    T v[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      c[u] = __ldcs(cp + uint32_t(j + u) * n);
      v[u] = __ldcs(vp + uint32_t(j + u) * n);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = ldx(xb + c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
  }
  if (j < L) {  // the last 1..7 entries, all in flight (warp-uniform count)
    uint32_t c[7];
    T v[7], xv[7];
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (j + u < L) {
        c[u] = __ldcs(cp + uint32_t(j + u) * n);
        v[u] = __ldcs(vp + uint32_t(j + u) * n);
      }
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (j + u < L) xv[u] = ldx(xb + c[u]);
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (j + u < L) acc = add_rn(acc, mul_rn(v[u], xv[u]));
  }
  y[dst] = L == 0 ? T(0) : acc;
}

// A gather warp: blocks from the launch's counter until none is left; the
// last warp to finish zeroes the counters for the next launch on this
// stream (per-stream scratch).
template <typename T>
__device__ __forceinline__ void gather_warp(const PanelParams<T>& P, int lane) {
  const T* xb = P.x - P.col_base;
  const T seed = P.pos_seed ? T(0) : T(-0.0);
  auto fetch = [&]() {
    uint32_t b = 0;
    if (lane == 0) b = atomicAdd(P.ctr, 1u);
    return __shfl_sync(0xffffffffu, b, 0);
  };
  uint32_t b = fetch();
  while (b < P.nblk) {
    const uint32_t desc = __ldg(P.blk + b);
    const uint32_t nb = fetch();  // the next block's index arrives while this one runs
    gather_block<T>(P, desc, lane, xb, seed);
    b = nb;
  }
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(P.ctr + 1, 1u) == P.gather_warps - 1) {
      P.ctr[0] = 0;
      P.ctr[1] = 0;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kPanelThreads, 1) csr_panel_kernel(const __grid_constant__ PanelParams<T> P) {
  extern __shared__ __align__(128) unsigned char panel_smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(panel_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= kPanelWarps) {  // gather side: no shared memory, no CTA barriers
    gather_warp<T>(P, lane);
    return;
  }
  const uint32_t it0 = P.cta_item[blockIdx.x], it1 = P.cta_item[blockIdx.x + 1];
  if (it0 == it1) return;
  const int nstg = P.nstg;
  const int64_t W = P.panel_cols;
  unsigned char* stages = panel_smem + kPanelHeader + size_t(warp) * nstg * panel_stage_bytes<T>();
  T* xs = reinterpret_cast<T*>(panel_smem + kPanelHeader + size_t(kPanelWarps) * nstg * panel_stage_bytes<T>());
  uint64_t* wbar = bar + 1 + warp * kPanelMaxStages;
  if (threadIdx.x < 1 + kPanelWarps * kPanelMaxStages) mbar_init(&bar[threadIdx.x], 1);
  if (threadIdx.x == 0) {
    mbar_fence_init();
    xs[W] = T(0);  // the padding entries' column
  }
  panel_bar_sync();
  uint32_t phase = 0, wphases = 0;
  for (uint32_t it = it0; it < it1; ++it) {
    const int64_t c0 = int64_t(P.item_panel[it]) * W;  // global column of xs[0]
    const int64_t lo = max(c0, P.col_base), hi = min(min(c0 + W, P.col_base + P.x_len), P.ncols);
    const T* src = P.x + (lo - P.col_base);
    // the 16-byte aligned middle of the panel by one TMA bulk copy, the few
    // entries around it by plain loads
    constexpr int64_t V = 16 / int64_t(sizeof(T));
    const int64_t a0 = c0 + (lo - c0 + V - 1) / V * V;
    const int64_t a1 = a0 + max(int64_t(0), hi - a0) / V * V;
    const bool bulk = a1 > a0 && reinterpret_cast<uintptr_t>(src + (a0 - lo)) % 16 == 0;
    const uint32_t* tk = P.task + (size_t(it) * kPanelWarps + warp) * 3;
    const uint32_t step0 = tk[0], nsteps = tk[1], slice0 = tk[2];
    panel_bar_sync();  // every warp is done with the previous panel (and its own stages)
    if (bulk && threadIdx.x == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, uint32_t((a1 - a0) * sizeof(T)));
      bulk_g2s(xs + (a0 - c0), src + (a0 - lo), uint32_t((a1 - a0) * sizeof(T)), bar);
    }
    if (lane == 0) {  // the warp's first steps stream in while the panel loads
      fence_proxy_async();
      for (uint32_t s = 0; s < uint32_t(nstg) && s < nsteps; ++s)
        panel_issue<T>(stages + s * panel_stage_bytes<T>(), &wbar[s], P.pcol, P.pval, step0 + s);
    }
    for (int64_t c = lo + threadIdx.x; c < (bulk ? a0 : hi); c += kPanelWarps * 32) xs[c - c0] = __ldg(src + (c - lo));
    if (bulk)
      for (int64_t c = a1 + threadIdx.x; c < hi; c += kPanelWarps * 32) xs[c - c0] = __ldg(src + (c - lo));
    if (bulk) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    }
    panel_bar_sync();
#ifdef SPMV_DEBUG_CHECKS
    for (int64_t c = lo + threadIdx.x; c < hi; c += kPanelWarps * 32) SPMV_DCHECK(same_bits(xs[c - c0], src[c - lo]), 2);
    SPMV_DCHECK(same_bits(xs[W], T(0)), 2);
#endif
    panel_task<T>(P, xs, stages, wbar, wphases, step0, nsteps, slice0, lane);
  }
}

// y[row] = the row's partials in panel order: a warp per long row, lane l
// adds partials l, l+32, ... of the row's list (rseg: partial indices row by
// row, panels ascending, a segment's pieces in order; 8 gathers in flight
// per lane) then a fixed xor tree (deterministic).
template <typename T>
__global__ void csr_panel_finish_kernel(const uint32_t* __restrict__ lrow, const uint32_t* __restrict__ ptr,
                                        const uint32_t* __restrict__ rseg, int64_t n_long,
                                        const double* __restrict__ part, T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; k < n_long; k += nw) {
    const uint32_t p0 = __ldg(ptr + k), p1 = __ldg(ptr + k + 1);
    double s = -0.0;
    for (uint32_t i0 = p0 + lane; i0 < p1; i0 += 256) {
      uint32_t idx[8];
      double val[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) idx[u] = i0 + 32u * u < p1 ? __ldcs(rseg + i0 + 32u * u) : 0u;
#pragma unroll
      for (int u = 0; u < 8; ++u) val[u] = i0 + 32u * u < p1 ? __ldcs(part + idx[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + 32u * u < p1) s = __dadd_rn(s, val[u]);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) y[lrow[k]] = T(s);
  }
}

// ---- plan-time kernels ------------------------------------------------------
// Long row k's entries: key = panel of the column, value = long-entry index;
// erow / eidx map a long-entry index to its long row and CSR entry.
__global__ void panel_expand_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                                    const uint32_t* __restrict__ lrow, const uint32_t* __restrict__ lptr,
                                    int64_t n_long, uint32_t W, uint32_t* __restrict__ key,
                                    uint32_t* __restrict__ val, uint32_t* __restrict__ erow,
                                    uint32_t* __restrict__ eidx) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; k < n_long; k += nw) {
    const uint32_t s = irp[lrow[k]], l0 = lptr[k], n = lptr[k + 1] - l0;
    for (uint32_t i = lane; i < n; i += 32) {
      key[l0 + i] = aj[s + i] / W;
      val[l0 + i] = l0 + i;
      erow[l0 + i] = uint32_t(k);
      eidx[l0 + i] = s + i;
    }
  }
}

// flag[i] = 1 when panel-major entry i is the first of its (row, panel) segment.
__global__ void panel_flag_kernel(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ perm,
                                  const uint32_t* __restrict__ erow, int64_t nl, uint32_t* __restrict__ flag) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nl; i += int64_t(gridDim.x) * blockDim.x)
    flag[i] = (i == 0 || skey[i - 1] != skey[i] || erow[perm[i - 1]] != erow[perm[i]]) ? 1u : 0u;
}

// Per segment (at its first entry): first entry, long row, panel;
// seg_start[nseg] = nl.
__global__ void panel_segments_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ seg_of,
                                      const uint32_t* __restrict__ skey, const uint32_t* __restrict__ perm,
                                      const uint32_t* __restrict__ erow, int64_t nl, int64_t nseg,
                                      uint32_t* __restrict__ seg_start, uint32_t* __restrict__ seg_row,
                                      uint32_t* __restrict__ seg_panel) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nl; i += int64_t(gridDim.x) * blockDim.x) {
    if (i == 0) seg_start[nseg] = uint32_t(nl);
    if (!flag[i]) continue;
    const uint32_t s = seg_of[i];
    seg_start[s] = uint32_t(i);
    seg_row[s] = erow[perm[i]];
    seg_panel[s] = skey[i];
  }
}

// Pieces of at most kPanelH entries per segment (nsub[nseg] = 0 for the scan's total).
__global__ void panel_nsub_kernel(const uint32_t* __restrict__ seg_start, int64_t nseg, uint32_t* __restrict__ nsub) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s <= nseg; s += int64_t(gridDim.x) * blockDim.x)
    nsub[s] = s < nseg ? (seg_start[s + 1] - seg_start[s] + kPanelH - 1) / kPanelH : 0u;
}

// Sub-segment t = sub_base[s] + j: sort key (panel, longest first), its segment.
__global__ void panel_subs_kernel(const uint32_t* __restrict__ seg_start, const uint32_t* __restrict__ seg_panel,
                                  const uint32_t* __restrict__ sub_base, int64_t nseg, uint32_t* __restrict__ key,
                                  uint32_t* __restrict__ id, uint32_t* __restrict__ sub_seg) {
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < nseg; s += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t len = seg_start[s + 1] - seg_start[s], t0 = sub_base[s], q = seg_panel[s];
    for (uint32_t j = 0; j * kPanelH < len; ++j) {
      const uint32_t l = min(uint32_t(kPanelH), len - j * kPanelH);
      key[t0 + j] = (q << 6) | (uint32_t(kPanelH) - l);
      id[t0 + j] = t0 + j;
      sub_seg[t0 + j] = uint32_t(s);
    }
  }
}

// The last index q <= nq with base[q] <= i (base ascending, base[0] = 0).
__device__ __forceinline__ uint32_t panel_find(const uint32_t* __restrict__ base, uint32_t nq, uint32_t i) {
  uint32_t lo = 0, hi = nq;  // invariant: base[lo] <= i
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (base[mid] <= i)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Entry-rows of slice sl: the length of its first (longest) sub-segment.
__global__ void panel_slice_width_kernel(const uint32_t* __restrict__ skey_s, const uint32_t* __restrict__ sub_ptr,
                                         const uint32_t* __restrict__ slice_base, uint32_t npanels, int64_t nslices,
                                         uint32_t* __restrict__ width) {
  for (int64_t sl = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; sl <= nslices; sl += int64_t(gridDim.x) * blockDim.x) {
    if (sl == nslices) {
      width[sl] = 0;
      continue;
    }
    const uint32_t q = panel_find(slice_base, npanels, uint32_t(sl));
    const uint32_t p0 = sub_ptr[q] + (uint32_t(sl) - slice_base[q]) * 32;
    width[sl] = uint32_t(kPanelH) - (skey_s[p0] & 63u);
  }
}

// Every column = W (the zero slot), headers zero.
__global__ void panel_init_cols_kernel(uint16_t* __restrict__ pcol, int64_t nsteps, uint32_t W) {
  constexpr int64_t per = kPanelColBytes / 2;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nsteps * per; i += int64_t(gridDim.x) * blockDim.x)
    pcol[i] = (i % per) < kPanelStep ? uint16_t(W) : uint16_t(0);
}

// The sub-segment at sorted position p goes to lane (p - first of its
// panel) % 32 of the panel's slice ... / 32: its entries down the slice's
// entry-rows; its partial's index and long row for the row-major list.
template <typename T>
__global__ void panel_fill_kernel(const uint32_t* __restrict__ skey_s, const uint32_t* __restrict__ sperm,
                                  const uint32_t* __restrict__ sub_ptr, const uint32_t* __restrict__ slice_base,
                                  const uint32_t* __restrict__ slice_row, const uint32_t* __restrict__ sub_seg,
                                  const uint32_t* __restrict__ sub_base, const uint32_t* __restrict__ seg_start,
                                  const uint32_t* __restrict__ seg_row, const uint32_t* __restrict__ perm,
                                  const uint32_t* __restrict__ eidx, const uint32_t* __restrict__ aj,
                                  const T* __restrict__ av, int64_t nsubs, uint32_t W, uint8_t* __restrict__ pcol,
                                  T* __restrict__ pval, uint32_t* __restrict__ sub_part,
                                  uint32_t* __restrict__ sub_row) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < nsubs; p += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t key = skey_s[p], q = key >> 6, len = uint32_t(kPanelH) - (key & 63u);
    const uint32_t k = uint32_t(p) - sub_ptr[q], sl = slice_base[q] + k / 32, lane = k % 32;
    const uint32_t t = sperm[p], s = sub_seg[t], i0 = seg_start[s] + (t - sub_base[s]) * kPanelH;
    const uint32_t row0 = slice_row[sl];
    for (uint32_t r = 0; r < len; ++r) {
      const uint32_t e = eidx[perm[i0 + r]], row = row0 + r, step = row / kPanelK, kk = row % kPanelK;
      pval[size_t(step) * kPanelStep + panel_val_pos(kk, lane)] = av[e];
      reinterpret_cast<uint16_t*>(pcol + size_t(step) * kPanelColBytes)[panel_col_pos(kk, lane)] =
          uint16_t(aj[e] - q * W);
    }
    sub_part[t] = sl * 32 + lane;
    sub_row[t] = seg_row[s];
  }
}

// Header bit of every slice's last entry-row.
__global__ void panel_endbits_kernel(const uint32_t* __restrict__ slice_row, const uint32_t* __restrict__ width,
                                     int64_t nslices, uint8_t* __restrict__ pcol) {
  for (int64_t sl = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; sl < nslices; sl += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t row = slice_row[sl] + width[sl] - 1;
    atomicOr(reinterpret_cast<uint32_t*>(pcol + size_t(row / kPanelK) * kPanelColBytes + kPanelStep * 2),
             1u << (row % kPanelK));
  }
}

// Long rows (over `thr` entries) and short rows, each in ascending order.
__global__ void split_rows_flags_kernel(const uint32_t* __restrict__ irp, int64_t nrows, uint32_t thr,
                                        uint32_t* __restrict__ is_long) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x)
    is_long[r] = (irp[r + 1] - irp[r]) > thr ? 1u : 0u;
}

// rows[pos[r]] = r for rows whose flag == want (pos: exclusive scan of the
// flags, or of 1 - flags for want == 0).
__global__ void split_rows_scatter_kernel(const uint32_t* __restrict__ is_long, const uint32_t* __restrict__ pos_long,
                                          int64_t nrows, uint32_t* __restrict__ lrow, uint32_t* __restrict__ srow) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t pl = pos_long[r];
    if (is_long[r])
      lrow[pl] = uint32_t(r);
    else
      srow[uint32_t(r) - pl] = uint32_t(r);
  }
}

// Lengths of listed rows.
__global__ void listed_lengths_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ rows, int64_t n,
                                      uint32_t* __restrict__ len) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    len[i] = irp[rows[i] + 1] - irp[rows[i]];
}

// Class of sorted short row i: the last L with cls[L] <= i.
__device__ __forceinline__ int short_class(const uint32_t* __restrict__ cls, int nclasses, uint32_t i) {
  int lo = 0, hi = nclasses - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cls[mid] <= i)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Column-major copy of the short rows by length class (see PanelParams).
template <typename T>
__global__ void short_ell_fill_kernel(const uint32_t* __restrict__ cls, const uint32_t* __restrict__ ebase,
                                      int nclasses, const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                                      const T* __restrict__ av, const uint32_t* __restrict__ srow, int64_t ns,
                                      uint32_t* __restrict__ scol, T* __restrict__ sval) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ns; i += int64_t(gridDim.x) * blockDim.x) {
    const int L = short_class(cls, nclasses, uint32_t(i));
    const uint32_t r = uint32_t(i) - cls[L], n = cls[L + 1] - cls[L], s = irp[srow[i]], eb = ebase[L];
    for (int j = 0; j < L; ++j) {
      scol[eb + uint32_t(j) * n + r] = aj[s + j];
      sval[eb + uint32_t(j) * n + r] = av[s + j];
    }
  }
}


template <typename T>
__global__ void scatter_zero_kernel(const uint32_t* __restrict__ rows, int64_t n, T* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[rows[i]] = T(0);
}

}  // namespace spmv
