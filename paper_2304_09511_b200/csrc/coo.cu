// COO SpMV for sm_100a.
//
// Reference: spmv_coo_plain (kernels.py:56-66) is np.add.at(y, rows,
// values * x[cols]) on a zeroed y — per row, a strictly sequential sum in
// storage order that starts from +0.0.  spmv_coo_vla (kernels.py:104-140)
// walks each row in L-entry steps, tree-reduces every step and adds it once
// into y[row].
//
// Plain path: fixed 2048-entry tiles (256 threads x 8 entries), so work per
// CTA does not depend on row lengths (Zipf rows up to 50k entries).  Inside
// a tile the row indices are segmented with a block scan; no atomics touch y.
//   * a row of <= 32 entries is "owned" by the tile holding its first entry;
//     one thread sums it left to right from +0.0 (shared-memory products,
//     plus at most 31 entries past the tile end) => bit-exact with np.add.at.
//     Whether a boundary row is short is decided from the 32 row indices on
//     either side of the tile, so both neighbouring tiles agree.
//   * rows of > 32 entries come from the plan's run table and go through
//     the shared long-row warp chunks (longrow.cuh).
//   * each tile zero-fills the empty rows between consecutive row starts,
//     so y needs no separate memset pass.
#include "longrow.cuh"

namespace spmv {

constexpr int kCooThreads = 256;
constexpr int kCooItems = 8;
constexpr int kCooTile = kCooThreads * kCooItems;
constexpr uint32_t kNoRow = 0xffffffffu;

template <typename T>
__global__ void __launch_bounds__(kCooThreads)
coo_tile_kernel(const uint32_t* __restrict__ ai, const uint32_t* __restrict__ aj, const T* __restrict__ av,
                const T* __restrict__ x, int64_t col_base, T* __restrict__ y, int64_t nnz, int64_t nrows) {
  using BlockScan = cub::BlockScan<int, kCooThreads>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  __shared__ uint32_t s_row[kCooTile];
  __shared__ T s_prod[kCooTile];
  __shared__ uint16_t s_seg[kCooTile];
  __shared__ uint16_t s_start[kCooTile + 1];
  __shared__ uint8_t s_owned[kCooTile];
  __shared__ uint32_t s_prev[32], s_next[32];
  __shared__ int s_nseg;

  const T* xb = x - col_base;
  const int tid = threadIdx.x;
  const int64_t base = int64_t(blockIdx.x) * kCooTile;
  const int cnt = int(min(int64_t(kCooTile), nnz - base));

  // 1. row indices of the tile (striped, coalesced) and the 32 on each side
  for (int k = tid; k < kCooTile; k += kCooThreads) s_row[k] = k < cnt ? ld_stream(ai + base + k) : kNoRow;
  if (tid < 32) {
    const int64_t g = base - 32 + tid;
    s_prev[tid] = g >= 0 ? ai[g] : kNoRow;
  } else if (tid < 64) {
    const int64_t g = base + cnt + (tid - 32);
    s_next[tid - 32] = g < nnz ? ai[g] : kNoRow;
  }
  __syncthreads();

  // 2. segment heads (blocked: thread owns entries tid*8 .. tid*8+7)
  bool head[kCooItems];
  int nh = 0;
#pragma unroll
  for (int i = 0; i < kCooItems; ++i) {
    const int k = tid * kCooItems + i;
    head[i] = k < cnt && (k == 0 || s_row[k] != s_row[k - 1]);
    nh += head[i];
  }
  int off = 0, total = 0;
  BlockScan(scan_tmp).ExclusiveSum(nh, off, total);
  {
    int cur = off - 1;
#pragma unroll
    for (int i = 0; i < kCooItems; ++i) {
      const int k = tid * kCooItems + i;
      if (head[i]) {
        ++cur;
        s_start[cur] = uint16_t(k);
      }
      if (k < cnt) s_seg[k] = uint16_t(cur);
    }
  }
  if (tid == 0) {
    s_nseg = total;
    s_start[total] = uint16_t(cnt);  // cnt <= 2048 fits
  }
  __syncthreads();
  const int nseg = s_nseg;

  // 3. classify segments; zero-fill empty rows before each row start
  for (int s = tid; s < nseg; s += kCooThreads) {
    const int k0 = s_start[s], k1 = s_start[s + 1];
    const uint32_t r = s_row[k0];
    const bool cont_before = (k0 == 0) && base > 0 && s_prev[31] == r;
    int before = 0, after = 0;
    if (cont_before)
      while (before < 32 && s_prev[31 - before] == r) ++before;
    if (k1 == cnt && base + cnt < nnz)
      while (after < 32 && s_next[after] == r) ++after;
    const int n = before + (k1 - k0) + after;
    const bool is_long = before == 32 || after == 32 || n > kExactLen;
    s_owned[s] = (!is_long && !cont_before) ? 1 : 0;
    if (!cont_before) {
      const int64_t prev = k0 > 0 ? int64_t(s_row[k0 - 1]) : (base > 0 ? int64_t(s_prev[31]) : int64_t(-1));
      for (int64_t q = prev + 1; q < int64_t(r); ++q) y[q] = T(0);
    }
    if (k1 == cnt && base + cnt == nnz)
      for (int64_t q = int64_t(r) + 1; q < nrows; ++q) y[q] = T(0);
  }
  __syncthreads();

  // 4. products of owned entries (striped, coalesced, 4 in flight)
  {
    int k = tid;
    for (; k + 3 * kCooThreads < cnt; k += 4 * kCooThreads) {
      const bool o0 = s_owned[s_seg[k]], o1 = s_owned[s_seg[k + kCooThreads]];
      const bool o2 = s_owned[s_seg[k + 2 * kCooThreads]], o3 = s_owned[s_seg[k + 3 * kCooThreads]];
      T v0 = T(0), v1 = T(0), v2 = T(0), v3 = T(0);
      uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
      if (o0) { c0 = ld_stream(aj + base + k); v0 = ld_stream(av + base + k); }
      if (o1) { c1 = ld_stream(aj + base + k + kCooThreads); v1 = ld_stream(av + base + k + kCooThreads); }
      if (o2) { c2 = ld_stream(aj + base + k + 2 * kCooThreads); v2 = ld_stream(av + base + k + 2 * kCooThreads); }
      if (o3) { c3 = ld_stream(aj + base + k + 3 * kCooThreads); v3 = ld_stream(av + base + k + 3 * kCooThreads); }
      if (o0) s_prod[k] = mul_rn(v0, __ldg(xb + c0));
      if (o1) s_prod[k + kCooThreads] = mul_rn(v1, __ldg(xb + c1));
      if (o2) s_prod[k + 2 * kCooThreads] = mul_rn(v2, __ldg(xb + c2));
      if (o3) s_prod[k + 3 * kCooThreads] = mul_rn(v3, __ldg(xb + c3));
    }
    for (; k < cnt; k += kCooThreads)
      if (s_owned[s_seg[k]]) s_prod[k] = mul_rn(ld_stream(av + base + k), __ldg(xb + ld_stream(aj + base + k)));
  }
  __syncthreads();

  // 5. one thread per owned row: left-to-right sum from +0.0
  for (int s = tid; s < nseg; s += kCooThreads) {
    if (!s_owned[s]) continue;
    const int k0 = s_start[s], k1 = s_start[s + 1];
    const uint32_t r = s_row[k0];
    T acc = T(0);
    for (int k = k0; k < k1; ++k) acc = add_rn(acc, s_prod[k]);
    if (k1 == cnt) {
      for (int j = 0; j < 32 && s_next[j] == r; ++j) {
        const int64_t g = base + cnt + j;
        acc = add_rn(acc, mul_rn(av[g], __ldg(xb + aj[g])));
      }
    }
    y[r] = acc;
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
template <typename T>
__global__ void __launch_bounds__(256)
coo_vla_warp_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ run_row, int64_t n_runs,
                    const uint32_t* __restrict__ aj, const T* __restrict__ av, const T* __restrict__ x,
                    int64_t col_base, T* __restrict__ y, int lanes, int width,
                    unsigned long long* __restrict__ steps_out) {
  const T* xb = x - col_base;
  const int lane = threadIdx.x % width;
  const int rows_per_warp = 32 / width;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long my_steps = 0;
  for (int64_t bidx = warp * rows_per_warp; bidx < n_runs; bidx += nwarps * rows_per_warp) {
    const int64_t ri = bidx + (threadIdx.x & 31) / width;
    uint32_t a = 0, b = 0, row = 0;
    if (ri < n_runs) {
      a = run_start[ri];
      b = run_start[ri + 1];
      row = run_row[ri];
    }
    const uint32_t nsteps = (b - a + uint32_t(lanes) - 1) / uint32_t(lanes);
    unsigned max_steps = __reduce_max_sync(0xffffffffu, nsteps);
    T yv = T(0);
    for (uint32_t st = 0; st < max_steps; ++st) {
      const uint32_t c0 = a + st * uint32_t(lanes);
      T p = T(0);
      if (st < nsteps && lane < lanes && c0 + lane < b) {
        const uint32_t j = c0 + lane;
        p = mul_rn(ld_stream(av + j), __ldg(xb + ld_stream(aj + j)));
      }
      p = tree_reduce_warp(p, width);
      if (st < nsteps) yv = add_rn(yv, p);
    }
    if (lane == 0 && ri < n_runs) {
      y[row] = yv;
      my_steps += nsteps;
    }
  }
  if (steps_out) {
    for (int o = 16; o >= 1; o >>= 1) my_steps += __shfl_down_sync(0xffffffffu, my_steps, o);
    if ((threadIdx.x & 31) == 0 && my_steps) atomicAdd(steps_out, my_steps);
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
      if (t < lanes && c0 + t < b) p = mul_rn(ld_stream(av + c0 + t), __ldg(xb + ld_stream(aj + c0 + t)));
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
  int64_t n_runs = 0;
  LongRows longrows;
  DevBuf steps;
};

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
  return p->longrows.build(p->run_start.as<uint32_t>(), p->run_row.as<uint32_t>(), p->n_runs, kExactLen,
                           value_size(p->dtype), st);
}

template <typename T>
static int coo_run(const spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const T* av, const T* x,
                   int64_t col_base, T* y, cudaStream_t st) {
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
  const int64_t tiles = (p->nnz + kCooTile - 1) / kCooTile;
  coo_tile_kernel<T><<<unsigned(tiles), kCooThreads, 0, st>>>(ai, aj, av, x, col_base, y, p->nnz, p->nrows);
  SPMV_LAUNCH_CHECK();
  return p->longrows.launch<T>(aj, av, x, col_base, y, st);
}

extern "C" {

int spmv_coo_plan_create(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* ai,
                         const uint32_t* aj, const void* av, void* stream, spmv_coo_plan** out) {
  if (!out) return fail(SPMV_INVALID_ARG, "spmv_coo_plan_create: out is NULL");
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
  int rc = SPMV_OK;
  if (nnz) rc = coo_plan_build(p, ai, aj, av, as_stream(stream));
  if (!rc) rc = p->steps.alloc(sizeof(unsigned long long));
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
  if (n_long_runs) *n_long_runs = p->longrows.n_long;
  if (n_items) *n_items = p->longrows.n_items;
  if (row_sorted) *row_sorted = p->row_sorted ? 1 : 0;
  if (launches) *launches = (p->nrows > 0 ? 1 : 0) + (p->longrows.n_items > 0 ? 1 : 0);
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
                           static_cast<double*>(y), st);
  return coo_run<float>(p, ai, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
                        static_cast<float*>(y), st);
}

int spmv_coo_vla(const spmv_coo_plan* p, const uint32_t* ai, const uint32_t* aj, const void* av, const void* x,
                 int64_t col_base, int64_t x_len, void* y, int lanes, int64_t* outer_steps, void* stream) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (lanes < 1) return fail(SPMV_INVALID_ARG, "lane count must be >= 1");
  if (lanes > 1024) return fail(SPMV_UNSUPPORTED, "vla COO supports at most 1024 lanes, got %d", lanes);
  if (x_len < 0 || col_base < 0) return fail(SPMV_DIMENSION_MISMATCH, "bad x window");
  (void)ai;
  cudaStream_t st = as_stream(stream);
  if (outer_steps) *outer_steps = 0;
  if (p->nrows == 0) return SPMV_OK;
  SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, value_size(p->dtype) * p->nrows, st));
  if (p->nnz == 0) return SPMV_OK;
  if (!p->row_sorted) {
    aj = p->sorted_aj.as<uint32_t>();
    av = p->sorted_av.ptr;
  }
  unsigned long long* steps = outer_steps ? p->steps.as<unsigned long long>() : nullptr;
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
    if (p->dtype == SPMV_F64)
      coo_vla_warp_kernel<double><<<unsigned(grid), tb, 0, st>>>(rs, rr, p->n_runs, aj,
                                                                  static_cast<const double*>(av),
                                                                  static_cast<const double*>(x), col_base,
                                                                  static_cast<double*>(y), lanes, width, steps);
    else
      coo_vla_warp_kernel<float><<<unsigned(grid), tb, 0, st>>>(rs, rr, p->n_runs, aj, static_cast<const float*>(av),
                                                                 static_cast<const float*>(x), col_base,
                                                                 static_cast<float*>(y), lanes, width, steps);
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
    SPMV_CUDA_TRY(cudaMemcpyAsync(&h, steps, sizeof(h), cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    *outer_steps = int64_t(h);
  }
  return SPMV_OK;
}

}  // extern "C"
