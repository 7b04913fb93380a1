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
// entries of the long rows (over kExactLen entries; 86% of C3's entries)
// are copied in panel-major order — panel q holds columns
// [q*W, (q+1)*W), W = kPanelCols, one panel = W values = 224 KB of f64 x —
// and inside a panel in row order, each row's entries in their original
// column order.  A (row, panel) run is a segment.  Per entry: a 16-bit word
// (column within the panel, bit 15 = first entry of a segment) and the
// value.  Segment s's partial sum goes to part[s]; rseg lists the segments
// row by row (panels ascending inside a row) for the final sums.
//
// Kernel: one 512-thread CTA per SM takes a contiguous range of the
// panel-major stream (equal entry counts, cut at segment starts); for each
// panel its range touches it loads the x panel into shared memory (one TMA
// bulk copy), then its 16 warps each walk one slice (cut at segment
// starts).  A warp step covers 32 x 8 entries, 8 consecutive per lane
// (16-byte vector loads of columns and values, streamed once from HBM, the
// next step's loads in flight during this step): each lane sums its entries
// left to right segment by segment, a warp segmented scan joins segments
// spanning lanes, completed segments are stored in segment order.
//
// Results: each long row = its panels' partials added in panel order by
// csr_panel_finish_kernel, each partial a left-to-right sum joined across
// lanes by the scan's fixed tree — deterministic, within 1e-12 of the
// reference's left-to-right sum (north_star allows that for rows over 32
// entries; rows of <= 32 entries never come here and stay bit-exact).
// f32: products rounded to f32 as in the reference, partials and the final
// sum in double, rounded once (the same contract as the warp-stream path).
#pragma once

#include "tma.cuh"

namespace spmv {

constexpr int kPanelCols = 28672;     // x entries per panel: 224 KB of f64 (+ the flag bit fits 16 bits)
constexpr int kPanelWarps = 16;       // warps per CTA (one CTA per SM)
constexpr int kPanelK = 8;            // consecutive entries per lane per step
static_assert(kPanelCols <= 0xffff, "panel column in 16 bits");

template <typename T>
struct PanelParams {
  const uint16_t* pcol;     // panel-major long-row entries: column in the panel
  const T* pval;
  const uint8_t* pflag;     // one byte per 8 entries: bit k = entry 8i+k starts a segment
  const T* x;               // x window: global column c at x[c - col_base]
  int64_t col_base, x_len, ncols;
  const uint32_t* cta_item;   // CTA c: items [cta_item[c], cta_item[c+1])
  const uint32_t* item_panel;
  const uint32_t* item_end;   // one past the item's last entry
  const uint32_t* task_begin; // kPanelWarps per item: warp w's first entry (a segment start)
  const uint32_t* task_seg0;  // segment index of task_begin
  double* part;               // partials, one per segment
};

template <typename T> __device__ __forceinline__ double panel_prod(T v, T x) { return double(mul_rn(v, x)); }

// Entries [j0, j0 + 8) of the panel stream, 16-byte vector loads (the
// arrays are padded, csr_panel_build).
__device__ __forceinline__ void panel_load(const uint16_t* __restrict__ pcol, const double* __restrict__ pval,
                                           uint32_t j0, uint16_t (&c)[kPanelK], double (&v)[kPanelK]) {
  const uint4 cw = __ldcs(reinterpret_cast<const uint4*>(pcol + j0));
  const uint32_t w[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c[2 * k] = uint16_t(w[k] & 0xffffu);
    c[2 * k + 1] = uint16_t(w[k] >> 16);
  }
  const double2* vp = reinterpret_cast<const double2*>(pval + j0);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 d = __ldcs(vp + k);
    v[2 * k] = d.x;
    v[2 * k + 1] = d.y;
  }
}
__device__ __forceinline__ void panel_load(const uint16_t* __restrict__ pcol, const float* __restrict__ pval,
                                           uint32_t j0, uint16_t (&c)[kPanelK], float (&v)[kPanelK]) {
  const uint4 cw = __ldcs(reinterpret_cast<const uint4*>(pcol + j0));
  const uint32_t w[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c[2 * k] = uint16_t(w[k] & 0xffffu);
    c[2 * k + 1] = uint16_t(w[k] >> 16);
  }
  const float4* vp = reinterpret_cast<const float4*>(pval + j0);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float4 d = __ldcs(vp + k);
    v[4 * k] = d.x;
    v[4 * k + 1] = d.y;
    v[4 * k + 2] = d.z;
    v[4 * k + 3] = d.w;
  }
}

__device__ __forceinline__ void st_if(double* p, double v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}" ::"l"(p), "d"(v),
               "r"(int(pred))
               : "memory");
}

// Columns (8 x 16 bit) and values of one lane's 8 entries, and the step's
// segment-start byte of this lane (bit k: entry k starts a segment).
template <typename T>
struct PanelRegs {
  uint16_t c[kPanelK];
  T v[kPanelK];
  unsigned fl;
};

template <typename T>
__device__ __forceinline__ void panel_fetch(const uint16_t* __restrict__ pcol, const T* __restrict__ pval,
                                            const uint8_t* __restrict__ pflag, uint32_t j0, PanelRegs<T>& r) {
  panel_load(pcol, pval, j0, r.c, r.v);
  r.fl = __ldcs(pflag + (j0 >> 3));
}

// One step of a warp slice: 32 lanes x kPanelK consecutive entries at
// j0 = base + lane * kPanelK (ok: the lane's entries inside the slice).
// A completed segment s is stored at part[s] (panel-major order: a step's
// stores go to neighbouring addresses); csr_panel_finish_kernel reads them
// row by row through the plan's row-major segment list.
template <typename T, bool FULL>
__device__ __forceinline__ void panel_step(const T* __restrict__ xs, const PanelRegs<T>& r, unsigned ok, int lane,
                                           int lo_ok, double* __restrict__ part_open, int& open_adv,
                                           double& carry) {
  const unsigned fl = FULL ? r.fl : (r.fl & ok);
  // segments started before this lane in the step (exclusive scan)
  const int nf = __popc(fl);
  int incl = nf;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  const int before = incl - nf;
  open_adv = __shfl_sync(0xffffffffu, incl, 31);
  double p[kPanelK];
#pragma unroll
  for (int k = 0; k < kPanelK; ++k) {
    p[k] = panel_prod(r.v[k], xs[r.c[k]]);  // invalid entries read a panel column too: masked below
    if (!FULL && !((ok >> k) & 1u)) p[k] = 0.0;
  }
  // lane pass, left to right: a segment complete inside the lane is stored
  // here; head = the part before the lane's first start
  int rel = before;  // segment open at this point, relative to `open`
  double run = 0.0, head = 0.0;
  bool started = false;
#pragma unroll
  for (int k = 0; k < kPanelK; ++k) {
    const bool f = (fl >> k) & 1u;
    st_if(part_open + rel, run, f && started && rel >= lo_ok);
    head = (f && !started) ? run : head;
    started = started || f;
    rel += f ? 1 : 0;
    run = __dadd_rn(f ? 0.0 : run, p[k]);
  }
  // segmented inclusive scan over lanes of (started, run); lane 0 first
  // takes the carried segment.  A lane adds the value d lanes up only while
  // no segment starts between (its last start at or before it: `ls`).
  if (lane == 0) {
    if (started)
      head = __dadd_rn(carry, head);
    else
      run = __dadd_rn(carry, run);
  }
  const unsigned smask = __ballot_sync(0xffffffffu, started) & ((2u << lane) - 1u);
  const int reach = smask ? lane - (31 - __clz(smask)) : lane + 1;  // lanes back to (not incl.) the last start
  double sc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double up = __shfl_up_sync(0xffffffffu, sc, d);
    if (reach >= d && lane >= d) sc = __dadd_rn(up, sc);
  }
  const double in = __shfl_up_sync(0xffffffffu, sc, 1);  // the segment open at this lane's start
  st_if(part_open + before, lane == 0 ? head : __dadd_rn(in, head), started && before >= lo_ok);
  carry = __shfl_sync(0xffffffffu, sc, 31);
}

// One warp's slice [b, e) of the panel stream (b is a segment start, seg0
// its segment index; the slice ends at a segment start or the item end).
// Software pipeline, one step ahead in two register sets: the next step's
// columns, values and start bits load while this step is reduced.
template <typename T>
__device__ __forceinline__ void panel_slice(const uint16_t* __restrict__ pcol, const T* __restrict__ pval,
                                            const uint8_t* __restrict__ pflag, double* __restrict__ part,
                                            const T* __restrict__ xs, uint32_t b, uint32_t e, uint32_t seg0,
                                            int lane) {
  if (b >= e) return;
  constexpr uint32_t STEP = 32 * kPanelK;
  double carry = 0.0;                // the open segment's sum over earlier steps
  int64_t open = int64_t(seg0) - 1;  // index of the segment open before this step (seg0 - 1: none)
  uint32_t base = b & ~(STEP - 1);
  PanelRegs<T> ra, rb;
  panel_fetch(pcol, pval, pflag, base + uint32_t(lane) * kPanelK, ra);
  auto run_step = [&](const PanelRegs<T>& cur, PanelRegs<T>& nxt) -> bool {
    const uint32_t j0 = base + uint32_t(lane) * kPanelK;
    const bool more = base + STEP < e;
    if (more) panel_fetch(pcol, pval, pflag, j0 + STEP, nxt);
    const int lo_ok = open < int64_t(seg0) ? 1 : 0;  // relative index 0 is seg0 - 1 (none) on the first step
    int adv = 0;
    if (base >= b && base + STEP <= e) {
      panel_step<T, true>(xs, cur, 0xffu, lane, lo_ok, part + open, adv, carry);
    } else {
      const int lo = min(max(int(int64_t(b) - int64_t(j0)), 0), kPanelK);
      const int hi = min(max(int(int64_t(e) - int64_t(j0)), 0), kPanelK);
      const unsigned ok = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
      panel_step<T, false>(xs, cur, ok, lane, lo_ok, part + open, adv, carry);
    }
    open += adv;
    base += STEP;
    return more;
  };
  while (run_step(ra, rb) && run_step(rb, ra)) {
  }
  if (lane == 0 && open >= int64_t(seg0)) part[open] = carry;  // the slice's last segment
}

template <typename T>
__global__ void __launch_bounds__(kPanelWarps * 32, 1) csr_panel_kernel(const __grid_constant__ PanelParams<T> P) {
  extern __shared__ __align__(128) unsigned char panel_smem[];
  T* xs = reinterpret_cast<T*>(panel_smem + 128);
  uint64_t* bar = reinterpret_cast<uint64_t*>(panel_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  for (uint32_t it = P.cta_item[blockIdx.x]; it < P.cta_item[blockIdx.x + 1]; ++it) {
    const int64_t c0 = int64_t(P.item_panel[it]) * kPanelCols;  // global column of xs[0]
    const int64_t lo = max(c0, P.col_base), hi = min(min(c0 + kPanelCols, P.col_base + P.x_len), P.ncols);
    const T* src = P.x + (lo - P.col_base);
    // the 16-byte aligned middle of the panel by one TMA bulk copy, the few
    // entries around it by plain loads
    constexpr int64_t V = 16 / int64_t(sizeof(T));
    const int64_t a0 = c0 + (lo - c0 + V - 1) / V * V;
    const int64_t a1 = a0 + max(int64_t(0), hi - a0) / V * V;
    const bool bulk = a1 > a0 && reinterpret_cast<uintptr_t>(src + (a0 - lo)) % 16 == 0;
    __syncthreads();  // every warp is done with the previous panel
    if (bulk && threadIdx.x == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, uint32_t((a1 - a0) * sizeof(T)));
      bulk_g2s(xs + (a0 - c0), src + (a0 - lo), uint32_t((a1 - a0) * sizeof(T)), bar);
    }
    for (int64_t c = lo + threadIdx.x; c < (bulk ? a0 : hi); c += blockDim.x) xs[c - c0] = __ldg(src + (c - lo));
    if (bulk)
      for (int64_t c = a1 + threadIdx.x; c < hi; c += blockDim.x) xs[c - c0] = __ldg(src + (c - lo));
    if (bulk) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    }
    __syncthreads();
    const uint32_t t = it * kPanelWarps + uint32_t(warp);
    const uint32_t b = P.task_begin[t];
    const uint32_t e = warp + 1 < kPanelWarps ? P.task_begin[t + 1] : P.item_end[it];
    panel_slice<T>(P.pcol, P.pval, P.pflag, P.part, xs, b, e, P.task_seg0[t], lane);
  }
}

// y[row] = the row's partials in panel order: 8 lanes per long row, lane
// l adds partials l, l+8, ... of the row's segment list (rseg: segment
// indices row by row, panels ascending) then a fixed xor tree
// (deterministic).
template <typename T>
__global__ void csr_panel_finish_kernel(const uint32_t* __restrict__ lrow, const uint32_t* __restrict__ ptr,
                                        const uint32_t* __restrict__ rseg, int64_t n_long,
                                        const double* __restrict__ part, T* __restrict__ y) {
  const int lane = threadIdx.x & 31, sub = lane & 7;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t kb = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 4; kb < n_long; kb += nw * 4) {
    const int64_t k = kb + (lane >> 3);
    double s = -0.0;
    if (k < n_long) {
      const uint32_t p0 = __ldg(ptr + k), p1 = __ldg(ptr + k + 1);
      for (uint32_t i = p0 + sub; i < p1; i += 8) s = __dadd_rn(s, __ldg(part + __ldg(rseg + i)));
    }
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (sub == 0 && k < n_long) y[lrow[k]] = T(s);
  }
}

// ---- plan-time kernels ------------------------------------------------------
// Long row k's entries: key = panel of the column, value = long-entry index;
// erow / eidx map a long-entry index to its long row and CSR entry.
__global__ void panel_expand_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                                    const uint32_t* __restrict__ lrow, const uint32_t* __restrict__ lptr,
                                    int64_t n_long, uint32_t* __restrict__ key, uint32_t* __restrict__ val,
                                    uint32_t* __restrict__ erow, uint32_t* __restrict__ eidx) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; k < n_long; k += nw) {
    const uint32_t s = irp[lrow[k]], l0 = lptr[k], n = lptr[k + 1] - l0;
    for (uint32_t i = lane; i < n; i += 32) {
      key[l0 + i] = aj[s + i] / uint32_t(kPanelCols);
      val[l0 + i] = l0 + i;
      erow[l0 + i] = uint32_t(k);
      eidx[l0 + i] = s + i;
    }
  }
}

// Panel-major copy: value, 16-bit column word with the segment flag, and
// the segment flag as a 0/1 word for the scan.
template <typename T>
__global__ void panel_gather_kernel(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ perm,
                                    const uint32_t* __restrict__ erow, const uint32_t* __restrict__ eidx,
                                    const uint32_t* __restrict__ aj, const T* __restrict__ av, int64_t nl,
                                    uint16_t* __restrict__ pcol, T* __restrict__ pval, uint32_t* __restrict__ flag) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nl; i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t le = perm[i], e = eidx[le], q = skey[i];
    const bool start = i == 0 || skey[i - 1] != q || erow[perm[i - 1]] != erow[le];
    pcol[i] = uint16_t(aj[e] - q * uint32_t(kPanelCols));
    pval[i] = av[e];
    flag[i] = start ? 1u : 0u;
  }
}

// Per segment (at its first entry): its long row and panel; per long row
// the number of segments (atomic counts, order-free).
__global__ void panel_segments_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ seg_of,
                                      const uint32_t* __restrict__ perm, const uint32_t* __restrict__ erow,
                                      int64_t nl, uint32_t* __restrict__ seg_row, uint32_t* __restrict__ row_cnt) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nl; i += int64_t(gridDim.x) * blockDim.x) {
    if (!flag[i]) continue;
    const uint32_t k = erow[perm[i]];
    seg_row[seg_of[i]] = k;
    atomicAdd(row_cnt + k, 1u);
  }
}

// Cut targets moved forward to the next segment start (or `limit`).
__global__ void panel_snap_kernel(const uint32_t* __restrict__ flag, uint32_t* __restrict__ pos, int64_t n,
                                  const uint32_t* __restrict__ limit) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t t = pos[i];
    const uint32_t lim = limit[i];
    while (t < lim && !flag[t]) ++t;
    pos[i] = t;
  }
}

// Segment-start bits, one byte per 8 entries.
__global__ void panel_flag_bytes_kernel(const uint32_t* __restrict__ flag, int64_t nl, uint8_t* __restrict__ out) {
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g * 8 < nl; g += int64_t(gridDim.x) * blockDim.x) {
    unsigned byte = 0;
    for (int k = 0; k < 8 && g * 8 + k < nl; ++k) byte |= (flag[g * 8 + k] ? 1u : 0u) << k;
    out[g] = uint8_t(byte);
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

// Lengths of listed rows (for the scans of lptr / the short CSR's IRP).
__global__ void listed_lengths_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ rows, int64_t n,
                                      uint32_t* __restrict__ len) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    len[i] = irp[rows[i] + 1] - irp[rows[i]];
}

// The short rows as their own CSR (a warp per row copies its entries).
template <typename T>
__global__ void short_copy_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                                  const T* __restrict__ av, const uint32_t* __restrict__ srow,
                                  const uint32_t* __restrict__ sirp, int64_t ns, uint32_t* __restrict__ saj,
                                  T* __restrict__ sav) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ns; i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t s = irp[srow[i]], d = sirp[i], n = sirp[i + 1] - d;
    for (uint32_t j = 0; j < n; ++j) {
      saj[d + j] = aj[s + j];
      sav[d + j] = av[s + j];
    }
  }
}

// Listed rows with no entries (the short CSR's empty rows), original ids.
__global__ void empty_listed_kernel(const uint32_t* __restrict__ sirp, const uint32_t* __restrict__ srow, int64_t ns,
                                    uint32_t* __restrict__ out, unsigned long long* __restrict__ n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ns; i += int64_t(gridDim.x) * blockDim.x)
    if (sirp[i + 1] == sirp[i]) {
      const unsigned long long k = atomicAdd(n, 1ull);
      if (out) out[k] = srow[i];
    }
}

template <typename T>
__global__ void scatter_zero_kernel(const uint32_t* __restrict__ rows, int64_t n, T* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[rows[i]] = T(0);
}

}  // namespace spmv
