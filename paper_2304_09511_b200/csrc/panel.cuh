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

constexpr int kPanelCols = 23552;     // x entries per panel: 184 KB of f64
constexpr int kPanelWarps = 16;       // warps per CTA (one CTA per SM)
constexpr int kPanelK = 8;            // consecutive entries per lane per step
constexpr int kPanelStep = 32 * kPanelK;  // entries per warp step
// per-warp staging of one step (TMA bulk copies): values, column pairs, start bits
template <typename T> constexpr int panel_stage_bytes() {
  return int(align_up(kPanelStep * sizeof(T) + kPanelStep * 2 + 32, 128));
}
constexpr int kPanelHeader = 256;  // mbarriers: [0] panel, [1 + w] warp w's stage
template <typename T> constexpr int panel_smem_bytes() {
  return kPanelHeader + kPanelWarps * panel_stage_bytes<T>() + kPanelCols * int(sizeof(T));
}
static_assert(panel_smem_bytes<double>() <= 232448, "panel kernel shared memory");
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

// Stream layout: within each 256-entry step (absolute entry index
// multiple of 256) the lane-contiguous order is transposed, so a lane's k-th
// entry sits at k * 32 + lane: values at step * 256 + k * 32 + lane, column
// pairs (entries 2m, 2m+1 of a lane in one 32-bit word) at word
// step * 128 + m * 32 + lane, and the lane's 8 start bits at byte
// step * 32 + lane.  Shared-memory reads of a staged step are then
// conflict-free.
__host__ __device__ __forceinline__ uint32_t panel_val_pos(uint32_t i) {
  const uint32_t r = i & (kPanelStep - 1);
  return (i - r) + (r & (kPanelK - 1)) * 32 + (r >> 3);
}
__host__ __device__ __forceinline__ uint32_t panel_col_pos(uint32_t i) {  // u16 index
  const uint32_t r = i & (kPanelStep - 1), k = r & (kPanelK - 1);
  return (i - r) + (k >> 1) * 64 + (r >> 3) * 2 + (k & 1);
}

__device__ __forceinline__ void st_if(double* p, double v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}" ::"l"(p), "d"(v),
               "r"(int(pred))
               : "memory");
}

// A lane's 8 entries of one step: columns, values, start bits (bit k: its
// entry k starts a segment).
template <typename T>
struct PanelRegs {
  uint16_t c[kPanelK];
  T v[kPanelK];
  unsigned fl;
};

// Warp stage: [0, 256 sizeof(T)) values, then 128 column-pair words, then
// 32 start-bit bytes.  Issued by lane 0 (three TMA bulk copies on the warp's
// mbarrier); read back into registers by every lane.
template <typename T>
__device__ __forceinline__ void panel_issue(unsigned char* stage, uint64_t* bar, const uint16_t* __restrict__ pcol,
                                            const T* __restrict__ pval, const uint8_t* __restrict__ pflag,
                                            uint32_t base) {
  constexpr uint32_t vb = kPanelStep * sizeof(T), cb = kPanelStep * 2;
  mbar_arrive_expect_tx(bar, vb + cb + 32);
  bulk_g2s(stage, pval + base, vb, bar, true);
  bulk_g2s(stage + vb, pcol + base, cb, bar, true);
  bulk_g2s(stage + vb + cb, pflag + base / 8, 32, bar, true);
}

template <typename T>
__device__ __forceinline__ void panel_read(const unsigned char* stage, int lane, PanelRegs<T>& r) {
  const T* vs = reinterpret_cast<const T*>(stage);
  const uint32_t* cs = reinterpret_cast<const uint32_t*>(stage + kPanelStep * sizeof(T));
#pragma unroll
  for (int k = 0; k < kPanelK; ++k) r.v[k] = vs[k * 32 + lane];
#pragma unroll
  for (int m = 0; m < kPanelK / 2; ++m) {
    const uint32_t w = cs[m * 32 + lane];
    r.c[2 * m] = uint16_t(w & 0xffffu);
    r.c[2 * m + 1] = uint16_t(w >> 16);
  }
  r.fl = stage[kPanelStep * sizeof(T) + kPanelStep * 2 + lane];
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
  // segments started before this lane in the step: the flag counts (<= 8)
  // summed bit-plane by bit-plane with ballots (no shuffles)
  const int nf = __popc(fl);
  const unsigned lt = (1u << lane) - 1u;
  int before = 0, total = 0;
#pragma unroll
  for (int bit = 0; bit < 4; ++bit) {
    const unsigned m = __ballot_sync(0xffffffffu, (nf >> bit) & 1);
    before += __popc(m & lt) << bit;
    total += __popc(m) << bit;
  }
  open_adv = total;
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
  // no segment starts between (its last start at or before it: `reach`).
  if (lane == 0) {
    if (started)
      head = __dadd_rn(carry, head);
    else
      run = __dadd_rn(carry, run);
  }
  const unsigned smask = __ballot_sync(0xffffffffu, started) & ((2u << lane) - 1u);
  const int reach = smask ? lane - (31 - __clz(smask)) : lane + 1;
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
// The warp's stage is refilled by TMA with the next step as soon as this
// step is in registers, so the copy runs while the step is reduced.
template <typename T>
__device__ __forceinline__ void panel_slice(const uint16_t* __restrict__ pcol, const T* __restrict__ pval,
                                            const uint8_t* __restrict__ pflag, double* __restrict__ part,
                                            const T* __restrict__ xs, unsigned char* stage, uint64_t* bar,
                                            uint32_t& phase, uint32_t b, uint32_t e, uint32_t seg0, int lane) {
  if (b >= e) return;
  double carry = 0.0;                // the open segment's sum over earlier steps
  int64_t open = int64_t(seg0) - 1;  // index of the segment open before this step (seg0 - 1: none)
  uint32_t base = b & ~uint32_t(kPanelStep - 1);
  if (lane == 0) panel_issue(stage, bar, pcol, pval, pflag, base);
  for (; base < e; base += kPanelStep) {
    const uint32_t j0 = base + uint32_t(lane) * kPanelK;
    const bool more = base + kPanelStep < e;
    PanelRegs<T> r;
    mbar_wait(bar, phase);
    phase ^= 1u;
#ifdef SPMV_DEBUG_CHECKS
    {  // the warp's stage holds exactly this step (no stage race)
      const T* vs = reinterpret_cast<const T*>(stage);
      const uint16_t* cs = reinterpret_cast<const uint16_t*>(stage + kPanelStep * sizeof(T));
      for (int k = lane; k < kPanelStep; k += 32) {
        SPMV_DCHECK(same_bits(vs[k], pval[base + k]), 0);
        SPMV_DCHECK(cs[k] == pcol[base + k], 0);
        SPMV_DCHECK(cs[k] < kPanelCols, 1);
      }
      SPMV_DCHECK(stage[kPanelStep * sizeof(T) + kPanelStep * 2 + lane] == pflag[base / 8 + lane], 0);
    }
#endif
    panel_read(stage, lane, r);
    __syncwarp();
    if (more && lane == 0) {
      fence_proxy_async();
      panel_issue(stage, bar, pcol, pval, pflag, base + kPanelStep);
    }
    const int lo_ok = open < int64_t(seg0) ? 1 : 0;  // relative index 0 is seg0 - 1 (none) on the first step
    int adv = 0;
    if (base >= b && base + kPanelStep <= e) {
      panel_step<T, true>(xs, r, 0xffu, lane, lo_ok, part + open, adv, carry);
    } else {
      const int lo = min(max(int(int64_t(b) - int64_t(j0)), 0), kPanelK);
      const int hi = min(max(int(int64_t(e) - int64_t(j0)), 0), kPanelK);
      const unsigned ok = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
      panel_step<T, false>(xs, r, ok, lane, lo_ok, part + open, adv, carry);
    }
    open += adv;
  }
  if (lane == 0 && open >= int64_t(seg0)) part[open] = carry;  // the slice's last segment
}

template <typename T>
__global__ void __launch_bounds__(kPanelWarps * 32, 1) csr_panel_kernel(const __grid_constant__ PanelParams<T> P) {
  extern __shared__ __align__(128) unsigned char panel_smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(panel_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* stage = panel_smem + kPanelHeader + warp * panel_stage_bytes<T>();
  T* xs = reinterpret_cast<T*>(panel_smem + kPanelHeader + kPanelWarps * panel_stage_bytes<T>());
  if (threadIdx.x < 1 + kPanelWarps) mbar_init(&bar[threadIdx.x], 1);
  if (threadIdx.x == 0) mbar_fence_init();
  __syncthreads();
  uint32_t phase = 0, wphase = 0;
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
#ifdef SPMV_DEBUG_CHECKS
    for (int64_t c = lo + threadIdx.x; c < hi; c += blockDim.x) SPMV_DCHECK(same_bits(xs[c - c0], src[c - lo]), 2);
#endif
    const uint32_t t = it * kPanelWarps + uint32_t(warp);
    const uint32_t b = P.task_begin[t];
    const uint32_t e = warp + 1 < kPanelWarps ? P.task_begin[t + 1] : P.item_end[it];
    panel_slice<T>(P.pcol, P.pval, P.pflag, P.part, xs, stage, &bar[1 + warp], wphase, b, e, P.task_seg0[t], lane);
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
      // batches of 8 partials per lane: indices, then values, all in
      // flight, then added in order
      for (uint32_t i0 = p0 + sub; i0 < p1; i0 += 64) {
        uint32_t idx[8];
        double val[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) idx[u] = i0 + 8u * u < p1 ? __ldg(rseg + i0 + 8u * u) : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) val[u] = i0 + 8u * u < p1 ? __ldg(part + idx[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + 8u * u < p1) s = __dadd_rn(s, val[u]);
      }
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
    pcol[panel_col_pos(uint32_t(i))] = uint16_t(aj[e] - q * uint32_t(kPanelCols));
    pval[panel_val_pos(uint32_t(i))] = av[e];
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

// Lengths of listed rows.
__global__ void listed_lengths_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ rows, int64_t n,
                                      uint32_t* __restrict__ len) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    len[i] = irp[rows[i] + 1] - irp[rows[i]];
}

// Short rows (<= 32 entries) grouped by exact length L: rows [cls[L],
// cls[L+1]) of the sorted list have L entries, stored column-major from
// ebase[L]: entry j of the class's r-th row at ebase[L] + j * n_L + r.
constexpr int kShortClasses = 33;  // lengths 0..32
struct ShortEll {
  uint32_t cls[kShortClasses + 1];
  uint32_t ebase[kShortClasses];
};

__device__ __forceinline__ int short_class(const ShortEll& P, uint32_t i) {
  int L = 0;  // the last class whose first row is <= i
#pragma unroll
  for (int step = 32; step >= 1; step >>= 1)
    if (L + step <= kShortClasses - 1 && P.cls[L + step] <= i) L += step;
  return L;
}

template <typename T>
__global__ void short_ell_fill_kernel(const __grid_constant__ ShortEll P, const uint32_t* __restrict__ irp,
                                      const uint32_t* __restrict__ aj, const T* __restrict__ av,
                                      const uint32_t* __restrict__ srow, int64_t ns, uint32_t* __restrict__ scol,
                                      T* __restrict__ sval) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ns; i += int64_t(gridDim.x) * blockDim.x) {
    const int L = short_class(P, uint32_t(i));
    const uint32_t r = uint32_t(i) - P.cls[L], n = P.cls[L + 1] - P.cls[L], s = irp[srow[i]];
    for (int j = 0; j < L; ++j) {
      scol[P.ebase[L] + uint32_t(j) * n + r] = aj[s + j];
      sval[P.ebase[L] + uint32_t(j) * n + r] = av[s + j];
    }
  }
}

// y of the short rows: one thread per row, its entries left to right from
// -0.0 (cumsum order, kernels.py:81: bit-exact) or, for COO plans
// (pos_seed), from +0.0 (np.add.at on a zeroed y, kernels.py:65); empty
// rows +0.0.  Rows of
// a warp share their length class, so the loop is uniform; loads are
// coalesced (column-major classes), gathers 4 in flight.
template <typename T>
__global__ void __launch_bounds__(256) short_ell_kernel(const __grid_constant__ ShortEll P,
                                                        const uint32_t* __restrict__ scol, const T* __restrict__ sval,
                                                        const uint32_t* __restrict__ srow, int64_t ns,
                                                        const T* __restrict__ x, int64_t col_base, T* __restrict__ y,
                                                        bool pos_seed) {
  const T* xb = x - col_base;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < ns; i += int64_t(gridDim.x) * blockDim.x) {
    const int L = short_class(P, uint32_t(i));
    const uint32_t n = P.cls[L + 1] - P.cls[L];
    const uint32_t o = P.ebase[L] + (uint32_t(i) - P.cls[L]);
    const uint32_t* cp = scol + o;
    const T* vp = sval + o;
    T acc = pos_seed ? T(0) : T(-0.0);
    int j = 0;
    for (; j + 4 <= L; j += 4) {
      uint32_t c[4];
      T v[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = __ldcs(cp + uint32_t(j + u) * n);
        v[u] = __ldcs(vp + uint32_t(j + u) * n);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = ldx(xb + c[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
    }
    for (; j < L; ++j) acc = add_rn(acc, mul_rn(__ldcs(vp + uint32_t(j) * n), ldx(xb + __ldcs(cp + uint32_t(j) * n))));
    y[srow[i]] = L == 0 ? T(0) : acc;
  }
}

template <typename T>
__global__ void scatter_zero_kernel(const uint32_t* __restrict__ rows, int64_t n, T* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[rows[i]] = T(0);
}

}  // namespace spmv
