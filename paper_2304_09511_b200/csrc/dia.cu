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
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "hostpipe.cuh"
#include "tma.cuh"

namespace spmv {


template <int G_, int S_, int NT_>
struct DiaCfg {
  static constexpr int G = G_, S = S_, NT = NT_;
};

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
// [t*R, t*R + R) (the last tile is clipped to avail_rows).  G consumer
// groups of NT threads share an S-stage ring: tile i of the CTA goes to
// group i % G and stage i % S, so G tiles compute while S - G load (more
// rows in flight per byte of shared memory than one group with a
// double buffer).
//
// GAPPED (spmv_dia_gapped): launch rows v >= split are slab rows v + gap, so
// a rank's two boundary blocks run as one launch; split is a multiple of
// rows_per_tile, so no tile straddles the gap.
template <typename T, int G, int S, int NT, int ND, bool GAPPED = false>
__global__ void __launch_bounds__(G * NT)
dia_bulk_kernel(const T* __restrict__ vals, const int32_t* __restrict__ offsets, int nd, const T* __restrict__ x,
                T* __restrict__ y, int64_t nrows, int64_t avail_rows, int64_t ncols, int64_t row_base,
                int64_t col_base, int rows_per_tile, int64_t ntiles, uint32_t stage_bytes, int64_t split = 0,
                int64_t gap = 0) {
  static_assert(S > G && S <= 8, "stages");
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                 // [0, 64)
  volatile int* tickets = reinterpret_cast<volatile int*>(smem + 64);  // [64, 96): CTA-local tile of each stage
  int32_t* s_off = reinterpret_cast<int32_t*>(smem + 128);
  const size_t off_bytes = (size_t(nd) * 4 + 127) & ~size_t(127);
  unsigned char* bufs = smem + 128 + off_bytes;
  const int g = int(threadIdx.x) / NT, tid = int(threadIdx.x) % NT;
  const T* xb = x - col_base;

  for (int d = threadIdx.x; d < nd; d += blockDim.x) s_off[d] = offsets[d];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&bars[s], 1);
      tickets[s] = -1;
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t first = blockIdx.x;
  const int64_t stride = gridDim.x;
  const int64_t my_tiles = first < ntiles ? (ntiles - 1 - first) / stride + 1 : 0;
  const size_t row_bytes = size_t(nd) * sizeof(T);

  // launch row -> slab row (GAPPED: rows past split jump the gap)
  auto slab_row = [&](int64_t lr) { return GAPPED && lr >= split ? lr + gap : lr; };
  auto issue = [&](int64_t i) {
    const int64_t t = first + i * stride;
    const int64_t lr0 = t * rows_per_tile;
    int64_t rows = (GAPPED && lr0 < split ? split : avail_rows) - lr0;
    if (rows > rows_per_tile) rows = rows_per_tile;
    const uint32_t bytes = uint32_t(rows * row_bytes);
    const int s = int(i % S);
    if (G > 1) tickets[s] = int(i);
    mbar_arrive_expect_tx(&bars[s], bytes);
    bulk_g2s(bufs + size_t(s) * stage_bytes,
             reinterpret_cast<const unsigned char*>(vals) + slab_row(lr0) * int64_t(row_bytes), bytes, &bars[s]);
  };
  auto group_sync = [&]() {
    if (G == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(NT) : "memory");
  };

  if (threadIdx.x == 0)
    for (int64_t i = 0; i < S && i < my_tiles; ++i) issue(i);

  for (int64_t i = g; i < my_tiles; i += G) {
    const int s = int(i % S);
    // parity waits only tell the current phase from the previous one: with
    // G > 1 wait until tile i is the one issued into the stage
    if (G > 1)
      while (tickets[s] != int(i)) __nanosleep(32);
    mbar_wait(&bars[s], uint32_t((i / S) & 1));
    const int64_t t = first + i * stride;
    const int64_t lr0 = t * rows_per_tile;
    const int64_t sr0 = slab_row(lr0);
    const T* tile = reinterpret_cast<const T*>(bufs + size_t(s) * stage_bytes);
#ifdef SPMV_DEBUG_CHECKS
    {  // the staged rows are exactly the global block (no ring race)
      int64_t rr = (GAPPED && lr0 < split ? split : avail_rows) - lr0;
      if (rr > rows_per_tile) rr = rows_per_tile;
      for (int64_t k = tid; k < rr * nd; k += NT) SPMV_DCHECK(same_bits(tile[k], vals[sr0 * nd + k]), 0);
    }
#endif
    int64_t rows = (GAPPED && lr0 < split ? split : nrows) - lr0;
    if (rows > rows_per_tile) rows = rows_per_tile;
    for (int lr = tid; lr < rows; lr += NT)
      y[sr0 + lr] = dia_row<T, ND>(tile + size_t(lr) * nd, s_off, nd, row_base + sr0 + lr, ncols, xb);
    group_sync();  // every thread of the group is done with stage s
    if (tid == 0 && i + S < my_tiles) {
      fence_proxy_async();
      issue(i + S);
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
                      const T* vals, const T* x, int64_t row_base, int64_t col_base, T* y, cudaStream_t st,
                      int64_t split = -1, int64_t gap = 0, const spmv_plan_config* pc = nullptr) {
  if (nrows == 0) return SPMV_OK;
  const bool gapped = split >= 0;
  const int sms = sm_count();
  const size_t row_bytes = size_t(nd) * sizeof(T);
  // Tile size: one row per thread (R = 256) when a stage fits ~56 KB, else
  // fewer rows (a multiple of 8).  Measured: 256-row tiles beat 512-row
  // tiles by 43% on 11 diagonals (more CTAs per SM, one row per thread).
  // Kernel configuration (groups G, stages S, threads per group NT; one row
  // per thread): spmv_plan_config.dia_kernel, else 3 groups over 4 stages — 256-row
  // stages when a stage holds more than 40 KB (e.g. 27 diagonals: one CTA
  // per SM, 768 rows computing), else 128-row stages (several CTAs per SM).
  // Measured on B200: 27-pt stencil 1287 -> 1610 GFLOP/s, 11-diagonal
  // banded 1225 -> 1398 against one group with a double buffer.
  static constexpr int kCfgStages[5] = {2, 3, 4, 4, 8};
  static constexpr int kCfgThreads[5] = {256, 256, 128, 256, 128};
  const spmv_plan_config C = config_or_default(pc);
  int cfg = C.dia_kernel;
  if (cfg < 0 || cfg > 4) cfg = row_bytes * 256 > 40960 ? 3 : 2;
  const int nt = kCfgThreads[cfg], nstage = kCfgStages[cfg];
  // rows per stage: NT, or fewer (a multiple of 8) so that S stages fit
  const size_t budget = (size_t(227) * 1024 - 1024 - 128 - ((size_t(nd) * 4 + 127) & ~size_t(127))) / nstage;
  int64_t R = int64_t(budget / (row_bytes ? row_bytes : 1)) / 8 * 8;
  if (R > nt) R = nt;
  if (C.dia_rows >= 8 && C.dia_rows / 8 * 8 <= R) R = C.dia_rows / 8 * 8;
  const bool aligned = (reinterpret_cast<uintptr_t>(vals) % 16 == 0) && ((R * row_bytes) % 16 == 0) &&
                       ((avail_rows * row_bytes) % 16 == 0);
  const bool use_bulk = nd > 0 && nd <= kMaxSmemOffsets && R >= 8 && aligned;
  if (gapped && (!use_bulk || split % R != 0 || (gap * int64_t(row_bytes)) % 16 != 0)) {
    // the split is not on this block's row-tile boundary (R depends on the
    // diagonal count and dtype): the two blocks as two plain launches
    int rc = dia_launch<T>(split, ncols, nd, avail_rows + gap, offsets, vals, x, row_base, col_base, y, st, -1, 0, pc);
    if (rc || nrows == split) return rc;
    const int64_t s1 = split + gap;  // slab row of launch row `split`
    return dia_launch<T>(nrows - split, ncols, nd, avail_rows - split, offsets, vals + s1 * nd, x, row_base + s1,
                         col_base, y + s1, st, -1, 0, pc);
  }
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
  const size_t off_bytes = (size_t(nd) * 4 + 127) & ~size_t(127);
  auto launch = [&](auto kernel, int threads, int stages) -> int {
    const size_t smem = 128 + off_bytes + size_t(stages) * stage_bytes;
    // the attribute and occupancy of a (device, kernel, shared-memory size)
    // are queried once; these host calls used to run on every product
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> attr;      // largest smem allowed so far
    static std::map<std::tuple<int, const void*, size_t>, int> occ;  // CTAs per SM at a smem size
    int per_sm = 0;
    {
      int dev = 0;
      SPMV_CUDA_TRY(cudaGetDevice(&dev));
      const void* kp = reinterpret_cast<const void*>(kernel);
      std::lock_guard<std::mutex> lock(mu);
      size_t& allowed = attr[{dev, kp}];
      if (smem > allowed) {  // the attribute only ever grows
        SPMV_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        allowed = smem;
      }
      const auto key = std::make_tuple(dev, kp, smem);
      auto it = occ.find(key);
      if (it != occ.end()) {
        per_sm = it->second;
      } else {
        SPMV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
        occ[key] = per_sm;
      }
    }
    if (per_sm < 1) return fail(SPMV_UNSUPPORTED, "DIA tile of %u bytes x %d stages does not fit", stage_bytes, stages);
    per_sm = cap_ctas(per_sm, C.ctas_per_sm);
    int64_t grid = int64_t(sms) * per_sm;
    if (grid > ntiles) grid = ntiles;
    kernel<<<unsigned(grid), threads, smem, st>>>(vals, offsets, int(nd), x, y, nrows, avail_rows, ncols, row_base,
                                                 col_base, int(R), ntiles, stage_bytes, split, gap);
    return SPMV_OK;
  };
  auto by_nd = [&](auto cfg) -> int {
    using C = decltype(cfg);
    constexpr int G = C::G, S = C::S, NT = C::NT;
    if (gapped) {  // the stencil and the banded matrix; other widths run generic
      switch (nd) {
        case 27: return launch(dia_bulk_kernel<T, G, S, NT, 27, true>, G * NT, S);
        case 11: return launch(dia_bulk_kernel<T, G, S, NT, 11, true>, G * NT, S);
        default: return launch(dia_bulk_kernel<T, G, S, NT, 0, true>, G * NT, S);
      }
    }
    switch (nd) {
      case 27: return launch(dia_bulk_kernel<T, G, S, NT, 27>, G * NT, S);
      case 11: return launch(dia_bulk_kernel<T, G, S, NT, 11>, G * NT, S);
      case 7: return launch(dia_bulk_kernel<T, G, S, NT, 7>, G * NT, S);
      case 5: return launch(dia_bulk_kernel<T, G, S, NT, 5>, G * NT, S);
      case 3: return launch(dia_bulk_kernel<T, G, S, NT, 3>, G * NT, S);
      default: return launch(dia_bulk_kernel<T, G, S, NT, 0>, G * NT, S);
    }
  };
  int rc;
  switch (cfg) {
    case 1: rc = by_nd(DiaCfg<1, 3, 256>{}); break;
    case 2: rc = by_nd(DiaCfg<3, 4, 128>{}); break;
    case 3: rc = by_nd(DiaCfg<3, 4, 256>{}); break;
    case 4: rc = by_nd(DiaCfg<7, 8, 128>{}); break;
    default: rc = by_nd(DiaCfg<1, 2, 256>{}); break;
  }
  if (rc) return rc;
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

}  // namespace spmv

using namespace spmv;

namespace spmv {
int debug_counts_dia(unsigned long long* out4) { return debug_read_tu(out4); }
}  // namespace spmv

extern "C" int spmv_dia_gapped(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags, int64_t avail_rows,
                               const int32_t* offsets, const void* values, const void* x, int64_t row_base,
                               int64_t col_base, int64_t x_len, void* y, int64_t y_split, int64_t y_gap,
                               void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows <= 0 || ncols < 0 || ndiags <= 0 || avail_rows < nrows || row_base < 0 || col_base < 0 || x_len < 0 ||
      y_split < 0 || y_split > nrows || y_gap < 0)
    return fail(SPMV_INVALID_ARG, "bad gapped DIA sizes");
  if (!offsets || !values || !x || !y) return fail(SPMV_INVALID_ARG, "NULL pointer");
  cudaStream_t st = as_stream(stream);
  if (dtype == SPMV_F64)
    return dia_launch<double>(nrows, ncols, ndiags, avail_rows, offsets, static_cast<const double*>(values),
                              static_cast<const double*>(x), row_base, col_base, static_cast<double*>(y), st, y_split,
                              y_gap);
  return dia_launch<float>(nrows, ncols, ndiags, avail_rows, offsets, static_cast<const float*>(values),
                           static_cast<const float*>(x), row_base, col_base, static_cast<float*>(y), st, y_split,
                           y_gap);
}

extern "C" int spmv_dia(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags, int64_t avail_rows,
                        const int32_t* offsets, const void* values, const void* x, int64_t row_base,
                        int64_t col_base, int64_t x_len, void* y, void* stream) {
  return spmv_dia_ex(dtype, nrows, ncols, ndiags, avail_rows, offsets, values, x, row_base, col_base, x_len, y,
                     nullptr, stream);
}

extern "C" int spmv_dia_ex(int dtype, int64_t nrows, int64_t ncols, int64_t ndiags, int64_t avail_rows,
                           const int32_t* offsets, const void* values, const void* x, int64_t row_base,
                           int64_t col_base, int64_t x_len, void* y, const spmv_plan_config* cfg, void* stream) {
  if (cfg && cfg->version != SPMV_PLAN_CONFIG_VERSION)
    return fail(SPMV_INVALID_ARG, "spmv_plan_config version %d, expected %d", cfg->version, SPMV_PLAN_CONFIG_VERSION);
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
                              static_cast<const double*>(x), row_base, col_base, static_cast<double*>(y), st, -1, 0,
                              cfg);
  return dia_launch<float>(nrows, ncols, ndiags, avail_rows, offsets, static_cast<const float*>(values),
                           static_cast<const float*>(x), row_base, col_base, static_cast<float*>(y), st, -1, 0, cfg);
}

// ---- host-buffer products (hostpipe.cuh) -----------------------------------
struct spmv_host_pipe {
  HostPipe hp;
};

extern "C" int spmv_host_pipe_create(spmv_host_pipe** out) {
  if (!out) return fail(SPMV_INVALID_ARG, "out is NULL");
  *out = new spmv_host_pipe();
  return SPMV_OK;
}

extern "C" int spmv_host_pipe_destroy(spmv_host_pipe* p) {
  delete p;
  return SPMV_OK;
}

// Row blocks: block [done, r) runs once x holds every column its rows reach
// (row + max_offset < the uploaded prefix); its rows of y then go down.
template <typename T>
static int dia_host_run(HostPipe& hp, int64_t nrows, int64_t ncols, int64_t nd, int64_t padded_rows,
                        const int32_t* offsets, int64_t max_offset, const T* vals, const T* xh, T* yh, int chunks,
                        const spmv_plan_config* cfg, cudaStream_t st) {
  const std::vector<int64_t> xb = host_x_chunks(ncols, chunks);
  const int nx = int(xb.size()) - 1;
  int64_t done = 0;
  auto compute = [&](int j, char* xd, char* yd, cudaStream_t s) -> int64_t {
    int64_t r = j == nx - 1 ? nrows : std::min<int64_t>(nrows, xb[j + 1] - std::max<int64_t>(max_offset, 0));
    if (r < nrows) r = r / 8 * 8;  // row blocks start on 8-row (TMA-aligned) boundaries
    if (r > done) {
      const int rc = dia_launch<T>(r - done, ncols, nd, padded_rows - done, offsets, vals + done * nd,
                                   reinterpret_cast<const T*>(xd), done, 0, reinterpret_cast<T*>(yd) + done, s, -1, 0,
                                   cfg);
      if (rc) return -rc;
      done = r;
    }
    return done;
  };
  return run_host_pipeline(hp, xh, yh, sizeof(T), ncols, nrows, xb, compute, false, st);
}

extern "C" int spmv_dia_host(spmv_host_pipe* pipe, int dtype, int64_t nrows, int64_t ncols, int64_t ndiags,
                             int64_t padded_rows, const int32_t* offsets, int64_t max_offset, const void* values,
                             const void* x_host, void* y_host, int chunks, const spmv_plan_config* cfg,
                             void* stream) {
  if (!pipe) return fail(SPMV_INVALID_ARG, "pipe is NULL");
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (nrows <= 0 || ncols <= 0 || ndiags <= 0 || padded_rows < nrows || !offsets || !values || !x_host || !y_host)
    return fail(SPMV_INVALID_ARG, "host pipeline needs a non-empty DIA block and host buffers");
  if (cfg && cfg->version != SPMV_PLAN_CONFIG_VERSION)
    return fail(SPMV_INVALID_ARG, "spmv_plan_config version %d, expected %d", cfg->version, SPMV_PLAN_CONFIG_VERSION);
  if (chunks <= 0) chunks = 16;
  if (chunks > 1024) chunks = 1024;
  cudaStream_t st = as_stream(stream);
  if (dtype == SPMV_F64)
    return dia_host_run<double>(pipe->hp, nrows, ncols, ndiags, padded_rows, offsets, max_offset,
                                static_cast<const double*>(values), static_cast<const double*>(x_host),
                                static_cast<double*>(y_host), chunks, cfg, st);
  return dia_host_run<float>(pipe->hp, nrows, ncols, ndiags, padded_rows, offsets, max_offset,
                             static_cast<const float*>(values), static_cast<const float*>(x_host),
                             static_cast<float*>(y_host), chunks, cfg, st);
}
