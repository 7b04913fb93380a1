// CSR SpMV for sm_100a.
//
// Reference: spmv_csr_plain (kernels.py:69-82) sums each row strictly left
// to right after rounding every product; spmv_csr_vla (kernels.py:143-171)
// uses L strided lane accumulators and a pairwise tree (lanes.py:107-128).
//
// Plain path = CSR-Adaptive style binning decided once in the plan:
//   * csr_stream_kernel: 128 consecutive rows per CTA.  When every row of
//     the group has <= exact_len entries (the stencil case) the group's
//     contiguous nnz range is streamed with coalesced loads, products are
//     formed in parallel into shared memory, and each thread then sums its
//     row from shared memory left to right — the reference order, so the
//     result is bit-exact.  Groups that contain long rows sum their short
//     rows per thread straight from global memory (still left to right) and
//     skip the long rows.
//   * long_rows_kernel (longrow.cuh): warp chunks for rows > exact_len.
#include "longrow.cuh"

namespace spmv {

constexpr int kGroupRows = 128;        // rows per CTA = threads per CTA
constexpr int kStreamCap = kGroupRows * kExactLen;  // staged products per CTA

template <typename T>
__global__ void __launch_bounds__(kGroupRows)
csr_stream_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                  const T* __restrict__ av, const T* __restrict__ x, int64_t col_base,
                  T* __restrict__ y, int64_t nrows, int exact_len) {
  __shared__ T prod[kStreamCap];
  const T* xb = x - col_base;
  const int tid = threadIdx.x;
  const int64_t r0 = int64_t(blockIdx.x) * kGroupRows;
  const int64_t r = r0 + tid;
  const int64_t rend = min(r0 + kGroupRows, nrows);
  uint32_t s = 0, e = 0;
  if (r < nrows) {
    s = irp[r];
    e = irp[r + 1];
  }
  const uint32_t len = e - s;
  const bool is_short = len <= uint32_t(exact_len);
  const uint32_t j0 = irp[r0];
  const uint32_t j1 = irp[rend];
  const uint32_t total = j1 - j0;
  const bool pure = __syncthreads_and(is_short) && total <= uint32_t(kStreamCap);
  if (pure) {
    // Coalesced stream of the group's [j0, j1): 4 products in flight/thread.
    uint32_t k = tid;
    for (; k + 3 * kGroupRows < total; k += 4 * kGroupRows) {
      const uint32_t c0 = ld_stream(aj + j0 + k), c1 = ld_stream(aj + j0 + k + kGroupRows);
      const uint32_t c2 = ld_stream(aj + j0 + k + 2 * kGroupRows), c3 = ld_stream(aj + j0 + k + 3 * kGroupRows);
      const T v0 = ld_stream(av + j0 + k), v1 = ld_stream(av + j0 + k + kGroupRows);
      const T v2 = ld_stream(av + j0 + k + 2 * kGroupRows), v3 = ld_stream(av + j0 + k + 3 * kGroupRows);
      prod[k] = mul_rn(v0, __ldg(xb + c0));
      prod[k + kGroupRows] = mul_rn(v1, __ldg(xb + c1));
      prod[k + 2 * kGroupRows] = mul_rn(v2, __ldg(xb + c2));
      prod[k + 3 * kGroupRows] = mul_rn(v3, __ldg(xb + c3));
    }
    for (; k < total; k += kGroupRows) prod[k] = mul_rn(ld_stream(av + j0 + k), __ldg(xb + ld_stream(aj + j0 + k)));
    __syncthreads();
    if (r < nrows) {
      T acc = T(0);
      if (len) {
        const T* p = prod + (s - j0);
        acc = p[0];  // cumsum starts from the first product (keeps -0.0)
        for (uint32_t i = 1; i < len; ++i) acc = add_rn(acc, p[i]);
      }
      y[r] = acc;
    }
  } else if (r < nrows && is_short) {
    T acc = T(0);
    if (len) {
      acc = mul_rn(ld_stream(av + s), __ldg(xb + ld_stream(aj + s)));
      for (uint32_t j = s + 1; j < e; ++j) acc = add_rn(acc, mul_rn(ld_stream(av + j), __ldg(xb + ld_stream(aj + j))));
    }
    y[r] = acc;
  }
}

// ---- vla: sub-warp (L <= 32) or CTA (32 < L <= 1024) per row ------------
template <typename T>
__global__ void __launch_bounds__(256)
csr_vla_warp_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj,
                    const T* __restrict__ av, const T* __restrict__ x, int64_t col_base,
                    T* __restrict__ y, int64_t nrows, int lanes, int width) {
  const T* xb = x - col_base;
  const int lane = threadIdx.x % width;
  const int rows_per_warp = 32 / width;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  // Uniform trip count per warp so the shuffles see every lane.
  for (int64_t base = warp * rows_per_warp; base < nrows; base += nwarps * rows_per_warp) {
    const int64_t r = base + (threadIdx.x & 31) / width;
    uint32_t s = 0, e = 0;
    if (r < nrows) {
      s = irp[r];
      e = irp[r + 1];
    }
    T acc = T(0);
    if (lane < lanes)
      for (uint32_t j = s + lane; j < e; j += uint32_t(lanes))
        acc = add_rn(acc, mul_rn(ld_stream(av + j), __ldg(xb + ld_stream(aj + j))));
    acc = tree_reduce_warp(acc, width);
    if (lane == 0 && r < nrows) y[r] = (s == e) ? T(0) : acc;
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
        acc = add_rn(acc, mul_rn(ld_stream(av + j), __ldg(xb + ld_stream(aj + j))));
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
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int exact_len = kExactLen;
  LongRows longrows;
};

template <typename T>
static int csr_run(const spmv_csr_plan* p, const uint32_t* irp, const uint32_t* aj, const T* av, const T* x,
                   int64_t col_base, T* y, cudaStream_t st) {
  if (p->nrows == 0) return SPMV_OK;
  const int64_t groups = (p->nrows + kGroupRows - 1) / kGroupRows;
  csr_stream_kernel<T><<<unsigned(groups), kGroupRows, 0, st>>>(irp, aj, av, x, col_base, y, p->nrows, p->exact_len);
  SPMV_LAUNCH_CHECK();
  return p->longrows.launch<T>(aj, av, x, col_base, y, st);
}

extern "C" {

int spmv_csr_plan_create(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* row_pointers,
                         int exact_len, void* stream, spmv_csr_plan** out) {
  if (!out) return fail(SPMV_INVALID_ARG, "spmv_csr_plan_create: out is NULL");
  *out = nullptr;
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows < 0 || ncols < 0 || nnz < 0 || nnz > int64_t(UINT32_MAX) || nrows >= int64_t(UINT32_MAX))
    return fail(SPMV_INVALID_ARG, "bad CSR sizes nrows=%lld ncols=%lld nnz=%lld", (long long)nrows,
                (long long)ncols, (long long)nnz);
  if (!row_pointers) return fail(SPMV_INVALID_ARG, "row_pointers is NULL");
  if (exact_len <= 0) exact_len = kExactLen;
  if (exact_len > kExactLen) exact_len = kExactLen;  // stream capacity is sized for 32
  auto* p = new spmv_csr_plan();
  p->dtype = dtype;
  p->nrows = nrows;
  p->ncols = ncols;
  p->nnz = nnz;
  p->exact_len = exact_len;
  int rc = p->longrows.build(row_pointers, nullptr, nrows, exact_len, value_size(dtype), as_stream(stream));
  if (rc) {
    delete p;
    return rc;
  }
  *out = p;
  return SPMV_OK;
}

int spmv_csr_plan_destroy(spmv_csr_plan* plan) {
  delete plan;
  return SPMV_OK;
}

int spmv_csr_plan_info(const spmv_csr_plan* p, int64_t* n_long_rows, int64_t* n_items, int64_t* launches) {
  if (!p) return fail(SPMV_INVALID_ARG, "plan is NULL");
  if (n_long_rows) *n_long_rows = p->longrows.n_long;
  if (n_items) *n_items = p->longrows.n_items;
  if (launches) *launches = (p->nrows > 0 ? 1 : 0) + (p->longrows.n_items > 0 ? 1 : 0);
  return SPMV_OK;
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
                           static_cast<double*>(y), st);
  return csr_run<float>(p, irp, aj, static_cast<const float*>(av), static_cast<const float*>(x), col_base,
                        static_cast<float*>(y), st);
}

int spmv_csr_vla(int dtype, int64_t nrows, int64_t ncols, int64_t nnz, const uint32_t* irp, const uint32_t* aj,
                 const void* av, const void* x, int64_t col_base, int64_t x_len, void* y, int lanes,
                 void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (lanes < 1) return fail(SPMV_INVALID_ARG, "lane count must be >= 1");
  if (lanes > 1024) return fail(SPMV_UNSUPPORTED, "vla CSR supports at most 1024 lanes, got %d", lanes);
  if (nrows < 0 || nnz < 0 || x_len < 0) return fail(SPMV_INVALID_ARG, "bad sizes");
  (void)ncols;
  if (nrows == 0) return SPMV_OK;
  int width = 1;
  while (width < lanes) width <<= 1;
  cudaStream_t st = as_stream(stream);
  const int64_t cap = int64_t(sm_count()) * 16;
  if (width <= 32) {
    const int tb = 256;
    int64_t grid = (nrows * width + tb - 1) / tb;
    if (grid > cap) grid = cap;
    if (dtype == SPMV_F64)
      csr_vla_warp_kernel<double><<<unsigned(grid), tb, 0, st>>>(irp, aj, static_cast<const double*>(av),
                                                                  static_cast<const double*>(x), col_base,
                                                                  static_cast<double*>(y), nrows, lanes, width);
    else
      csr_vla_warp_kernel<float><<<unsigned(grid), tb, 0, st>>>(irp, aj, static_cast<const float*>(av),
                                                                 static_cast<const float*>(x), col_base,
                                                                 static_cast<float*>(y), nrows, lanes, width);
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

}  // extern "C"
