// DIA SpMV for sm_100a.
//
// Reference: spmv_dia_plain (kernels.py:85-101) adds, for each diagonal in
// ascending offset order, values[i, d] * x[i + off] into y[i] for the rows
// whose column lies inside the matrix; spmv_dia_vla (kernels.py:174-210)
// visits each row's diagonals in the same order.  One thread per row that
// starts from +0.0 and adds its in-bounds products in diagonal order is
// therefore bit-exact with both.
//
// Data layout: the reference's row-major (padded_rows, ndiags) block
// (formats.py:166-207).  A tile of R consecutive rows is one contiguous
// R*ndiags*sizeof(T) byte range, so a single cp.async.bulk (TMA 1-D bulk
// copy, completion on an mbarrier) stages it into shared memory; a
// persistent CTA keeps STAGES tiles in flight while it computes on the
// oldest one.  Each thread then reads its row from shared memory (stride
// ndiags, odd strides are bank-conflict free for 8-byte words) and gathers
// x through L1: the x window of a tile is re-read by every diagonal with
// the same (dz, dy), so it stays L1/L2 resident.
#include "tma.cuh"

namespace spmv {

int dia_rows_per_tile();
int dia_stages();

constexpr int kDiaThreads = 256;
constexpr int kMaxSmemOffsets = 2048;

// One row: ascending diagonals, in-bounds cells only, from +0.0.  With ND
// known at compile time all ND x-gathers are issued before the first add
// (one L2 round trip per row instead of ND).
template <typename T, int ND>
__device__ __forceinline__ T dia_row(const T* __restrict__ v, const int32_t* __restrict__ offs, int nd, int64_t grow,
                                     int64_t ncols, const T* __restrict__ xb) {
  T acc = T(0);
  if constexpr (ND > 0) {
    T xv[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const int64_t col = grow + offs[d];
      xv[d] = (col >= 0 && col < ncols) ? ldx(xb + col) : T(0);
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const int64_t col = grow + offs[d];
      if (col >= 0 && col < ncols) acc = add_rn(acc, mul_rn(v[d], xv[d]));
    }
  } else {
#pragma unroll 9
    for (int d = 0; d < nd; ++d) {
      const int64_t col = grow + offs[d];
      if (col >= 0 && col < ncols) acc = add_rn(acc, mul_rn(v[d], ldx(xb + col)));
    }
  }
  return acc;
}

// Persistent TMA-pipelined kernel.  Tile t covers local rows
// [t*R, t*R + R) (the last tile is clipped to avail_rows).
template <typename T, int STAGES, int ND>
__global__ void __launch_bounds__(kDiaThreads)
dia_bulk_kernel(const T* __restrict__ vals, const int32_t* __restrict__ offsets, int nd, const T* __restrict__ x,
                T* __restrict__ y, int64_t nrows, int64_t avail_rows, int64_t ncols, int64_t row_base,
                int64_t col_base, int rows_per_tile, int64_t ntiles, uint32_t stage_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  int32_t* s_off = reinterpret_cast<int32_t*>(smem + 128);
  const size_t off_bytes = (size_t(nd) * 4 + 127) & ~size_t(127);
  unsigned char* bufs = smem + 128 + off_bytes;
  const int tid = threadIdx.x;
  const T* xb = x - col_base;

  for (int d = tid; d < nd; d += blockDim.x) s_off[d] = offsets[d];
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t first = blockIdx.x;
  const int64_t stride = gridDim.x;
  const int64_t my_tiles = first < ntiles ? (ntiles - 1 - first) / stride + 1 : 0;
  const size_t row_bytes = size_t(nd) * sizeof(T);

  auto issue = [&](int64_t i) {
    const int64_t t = first + i * stride;
    const int64_t lr0 = t * rows_per_tile;
    int64_t rows = avail_rows - lr0;
    if (rows > rows_per_tile) rows = rows_per_tile;
    const uint32_t bytes = uint32_t(rows * row_bytes);
    const int s = int(i % STAGES);
    mbar_arrive_expect_tx(&bars[s], bytes);
    bulk_g2s(bufs + size_t(s) * stage_bytes, reinterpret_cast<const unsigned char*>(vals) + lr0 * row_bytes, bytes,
             &bars[s]);
  };

  if (tid == 0)
    for (int64_t i = 0; i < STAGES && i < my_tiles; ++i) issue(i);

  for (int64_t i = 0; i < my_tiles; ++i) {
    const int s = int(i % STAGES);
    mbar_wait(&bars[s], uint32_t((i / STAGES) & 1));
    const int64_t t = first + i * stride;
    const int64_t lr0 = t * rows_per_tile;
    const T* tile = reinterpret_cast<const T*>(bufs + size_t(s) * stage_bytes);
    int64_t rows = nrows - lr0;
    if (rows > rows_per_tile) rows = rows_per_tile;
    for (int lr = tid; lr < rows; lr += blockDim.x)
      y[lr0 + lr] = dia_row<T, ND>(tile + size_t(lr) * nd, s_off, nd, row_base + lr0 + lr, ncols, xb);
    __syncthreads();  // every thread is done with stage s
    if (tid == 0 && i + STAGES < my_tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + STAGES);
    }
  }
}

// Fallback for blocks the bulk engine cannot address (misaligned base or a
// row count that does not give 16-byte multiples): thread per row, values
// read straight from global memory.
template <typename T>
__global__ void __launch_bounds__(kDiaThreads)
dia_direct_kernel(const T* __restrict__ vals, const int32_t* __restrict__ offsets, int nd, const T* __restrict__ x,
                  T* __restrict__ y, int64_t nrows, int64_t ncols, int64_t row_base, int64_t col_base) {
  const T* xb = x - col_base;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nrows; i += int64_t(gridDim.x) * blockDim.x) {
    T acc = T(0);
    const T* v = vals + size_t(i) * nd;
    for (int d = 0; d < nd; ++d) {
      const int64_t col = row_base + i + __ldg(offsets + d);
      if (col >= 0 && col < ncols) acc = add_rn(acc, mul_rn(__ldg(v + d), ldx(xb + col)));
    }
    y[i] = acc;
  }
}

template <typename T>
static int dia_launch(int64_t nrows, int64_t ncols, int64_t nd, int64_t avail_rows, const int32_t* offsets,
                      const T* vals, const T* x, int64_t row_base, int64_t col_base, T* y, cudaStream_t st) {
  if (nrows == 0) return SPMV_OK;
  const int sms = sm_count();
  const size_t row_bytes = size_t(nd) * sizeof(T);
  // Tile size: one row per thread (R = 256) when a stage fits ~56 KB, else
  // fewer rows (a multiple of 8).  Measured: 256-row tiles beat 512-row
  // tiles by 43% on 11 diagonals (more CTAs per SM, one row per thread).
  int64_t R = int64_t(57344 / (row_bytes ? row_bytes : 1)) / 8 * 8;
  if (R > kDiaThreads) R = kDiaThreads;
  if (dia_rows_per_tile() >= 8) R = dia_rows_per_tile() / 8 * 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(vals) % 16 == 0) && ((R * row_bytes) % 16 == 0) &&
                       ((avail_rows * row_bytes) % 16 == 0);
  const bool use_bulk = nd > 0 && nd <= kMaxSmemOffsets && R >= 8 && aligned;
  if (!use_bulk) {
    int64_t grid = (nrows + kDiaThreads - 1) / kDiaThreads;
    if (grid > int64_t(sms) * 32) grid = int64_t(sms) * 32;
    dia_direct_kernel<T><<<unsigned(grid), kDiaThreads, 0, st>>>(vals, offsets, int(nd), x, y, nrows, ncols,
                                                                   row_base, col_base);
    SPMV_LAUNCH_CHECK();
    return SPMV_OK;
  }
  const int64_t ntiles = (nrows + R - 1) / R;
  const uint32_t stage_bytes = uint32_t(((R * row_bytes) + 127) & ~size_t(127));
  int stages = stage_bytes > 40960 ? 2 : 3;
  if (dia_stages() == 2 || dia_stages() == 3) stages = dia_stages();
  const size_t off_bytes = (size_t(nd) * 4 + 127) & ~size_t(127);
  const size_t smem = 128 + off_bytes + size_t(stages) * stage_bytes;
  int ctas_per_sm = int((227 * 1024) / (smem + 1024));
  if (ctas_per_sm < 1) ctas_per_sm = 1;
  if (ctas_per_sm > 4) ctas_per_sm = 4;
  int64_t grid = int64_t(sms) * ctas_per_sm;
  if (grid > ntiles) grid = ntiles;
  auto launch = [&](auto kernel) -> int {
    SPMV_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kernel<<<unsigned(grid), kDiaThreads, smem, st>>>(vals, offsets, int(nd), x, y, nrows, avail_rows, ncols,
                                                       row_base, col_base, int(R), ntiles, stage_bytes);
    return SPMV_OK;
  };
  int rc;
  if (stages == 2) {
    switch (nd) {
      case 27: rc = launch(dia_bulk_kernel<T, 2, 27>); break;
      case 11: rc = launch(dia_bulk_kernel<T, 2, 11>); break;
      case 7: rc = launch(dia_bulk_kernel<T, 2, 7>); break;
      case 5: rc = launch(dia_bulk_kernel<T, 2, 5>); break;
      case 3: rc = launch(dia_bulk_kernel<T, 2, 3>); break;
      default: rc = launch(dia_bulk_kernel<T, 2, 0>); break;
    }
  } else {
    switch (nd) {
      case 27: rc = launch(dia_bulk_kernel<T, 3, 27>); break;
      case 11: rc = launch(dia_bulk_kernel<T, 3, 11>); break;
      case 7: rc = launch(dia_bulk_kernel<T, 3, 7>); break;
      case 5: rc = launch(dia_bulk_kernel<T, 3, 5>); break;
      case 3: rc = launch(dia_bulk_kernel<T, 3, 3>); break;
      default: rc = launch(dia_bulk_kernel<T, 3, 0>); break;
    }
  }
  if (rc) return rc;
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

}  // namespace spmv

using namespace spmv;

extern "C" int spmv_dia(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags, int64_t avail_rows,
                        const int32_t* offsets, const void* values, const void* x, int64_t row_base,
                        int64_t col_base, int64_t x_len, void* y, void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows < 0 || ncols < 0 || ndiags < 0 || avail_rows < nrows || row_base < 0 || col_base < 0 || x_len < 0)
    return fail(SPMV_INVALID_ARG, "bad DIA sizes");
  if (nrows == 0) return SPMV_OK;
  if (!y) return fail(SPMV_INVALID_ARG, "y is NULL");
  cudaStream_t st = as_stream(stream);
  if (ndiags == 0) {
    SPMV_CUDA_TRY(cudaMemsetAsync(y, 0, size_t(nrows) * value_size(dtype), st));
    return SPMV_OK;
  }
  if (!offsets || !values || !x) return fail(SPMV_INVALID_ARG, "NULL pointer");
  if (dtype == SPMV_F64)
    return dia_launch<double>(nrows, ncols, ndiags, avail_rows, offsets, static_cast<const double*>(values),
                              static_cast<const double*>(x), row_base, col_base, static_cast<double*>(y), st);
  return dia_launch<float>(nrows, ncols, ndiags, avail_rows, offsets, static_cast<const float*>(values),
                           static_cast<const float*>(x), row_base, col_base, static_cast<float*>(y), st);
}
