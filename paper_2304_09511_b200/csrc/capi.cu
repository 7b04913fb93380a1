// Library-level C ABI: error reporting, device queries, partition helpers.
#include <cub/cub.cuh>

#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace spmv {

static thread_local std::string g_last_error;

void set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  (void)code;
  g_last_error = buf;
}

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int sm_count() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

}  // namespace spmv

using namespace spmv;

extern "C" {

int spmv_abi_version(void) { return SPMV_B200_ABI_VERSION; }

const char* spmv_last_error(void) { return g_last_error.c_str(); }

int spmv_device_sm_count(int* out) {
  if (!out) return fail(SPMV_INVALID_ARG, "out is NULL");
  *out = sm_count();
  return SPMV_OK;
}

int spmv_csr_col_bounds(int64_t nrows, const uint32_t* irp, const uint32_t* aj, void* stream, uint32_t* min_out,
                        uint32_t* max_out) {
  if (!min_out || !max_out) return fail(SPMV_INVALID_ARG, "NULL output");
  *min_out = UINT32_MAX;
  *max_out = 0;
  if (nrows <= 0) return SPMV_OK;
  cudaStream_t st = as_stream(stream);
  uint32_t b[2] = {0, 0};
  SPMV_CUDA_TRY(cudaMemcpyAsync(&b[0], irp, 4, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaMemcpyAsync(&b[1], irp + nrows, 4, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t n = int64_t(b[1]) - int64_t(b[0]);
  if (n <= 0) return SPMV_OK;
  DevBuf out, tmp;
  int rc = out.alloc(8);
  if (rc) return rc;
  size_t t1 = 0, t2 = 0;
  SPMV_CUDA_TRY(cub::DeviceReduce::Min(nullptr, t1, aj + b[0], out.as<uint32_t>(), n, st));
  SPMV_CUDA_TRY(cub::DeviceReduce::Max(nullptr, t2, aj + b[0], out.as<uint32_t>() + 1, n, st));
  if ((rc = tmp.alloc(t1 > t2 ? t1 : t2))) return rc;
  SPMV_CUDA_TRY(cub::DeviceReduce::Min(tmp.ptr, t1, aj + b[0], out.as<uint32_t>(), n, st));
  SPMV_CUDA_TRY(cub::DeviceReduce::Max(tmp.ptr, t2, aj + b[0], out.as<uint32_t>() + 1, n, st));
  uint32_t h[2];
  SPMV_CUDA_TRY(cudaMemcpyAsync(h, out.ptr, 8, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  *min_out = h[0];
  *max_out = h[1];
  return SPMV_OK;
}

}  // extern "C"

// ---- interior / boundary split of a row slab (hpcg.py:95-154 semantics) ----
namespace spmv {
__global__ void halo_split_kernel(const uint32_t* __restrict__ irp, const uint32_t* __restrict__ aj, int64_t nrows,
                                  int64_t col_lo, int64_t col_hi, unsigned long long* __restrict__ out) {
  // out[0] = max row + 1 touching a column < col_lo; out[1] = min row touching a column >= col_hi
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows; r += int64_t(gridDim.x) * blockDim.x) {
    bool lo = false, hi = false;
    for (uint32_t j = irp[r]; j < irp[r + 1]; ++j) {
      const int64_t c = aj[j];
      lo |= c < col_lo;
      hi |= c >= col_hi;
    }
    if (lo) atomicMax(out, (unsigned long long)(r + 1));
    if (hi) atomicMin(out + 1, (unsigned long long)r);
  }
}
}  // namespace spmv

extern "C" int spmv_csr_halo_split(int64_t nrows, const uint32_t* irp, const uint32_t* aj, int64_t col_lo,
                                   int64_t col_hi, void* stream, int64_t* i_lo, int64_t* i_hi) {
  if (!i_lo || !i_hi) return fail(SPMV_INVALID_ARG, "NULL output");
  *i_lo = 0;
  *i_hi = nrows;
  if (nrows <= 0) return SPMV_OK;
  cudaStream_t st = as_stream(stream);
  DevBuf out;
  int rc = out.alloc(16);
  if (rc) return rc;
  unsigned long long init[2] = {0ull, (unsigned long long)nrows};
  SPMV_CUDA_TRY(cudaMemcpyAsync(out.ptr, init, 16, cudaMemcpyHostToDevice, st));
  int64_t grid = (nrows + 255) / 256;
  if (grid > int64_t(sm_count()) * 16) grid = int64_t(sm_count()) * 16;
  halo_split_kernel<<<unsigned(grid), 256, 0, st>>>(irp, aj, nrows, col_lo, col_hi, out.as<unsigned long long>());
  SPMV_LAUNCH_CHECK();
  unsigned long long h[2];
  SPMV_CUDA_TRY(cudaMemcpyAsync(h, out.ptr, 16, cudaMemcpyDeviceToHost, st));
  SPMV_CUDA_TRY(cudaStreamSynchronize(st));
  *i_lo = int64_t(h[0]);
  *i_hi = int64_t(h[1]);
  return SPMV_OK;
}

namespace spmv {
int pool_keep_memory() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(SPMV_CUDA_ERROR, "cudaGetDevice: %s", cudaGetErrorString(e));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && done[dev]) return SPMV_OK;
  cudaMemPool_t pool;
  e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e != cudaSuccess) return fail(SPMV_CUDA_ERROR, "cudaDeviceGetDefaultMemPool: %s", cudaGetErrorString(e));
  uint64_t keep = kPoolKeepBytes;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e != cudaSuccess) return fail(SPMV_CUDA_ERROR, "cudaMemPoolSetAttribute: %s", cudaGetErrorString(e));
  if (dev < 64) done[dev] = true;
  return SPMV_OK;
}
}  // namespace spmv

namespace spmv {
int debug_counts_csr(unsigned long long* out4);
int debug_counts_coo(unsigned long long* out4);
int debug_counts_dia(unsigned long long* out4);
}  // namespace spmv

// Debug builds: read and reset the device-side check counters of every
// kernel translation unit (common.cuh SPMV_DCHECK).  SPMV_UNSUPPORTED in
// normal builds.
extern "C" int spmv_debug_check_counts(unsigned long long* out4) {
  if (!out4) return fail(SPMV_INVALID_ARG, "out is NULL");
  for (int i = 0; i < 4; ++i) out4[i] = 0;
  int rc = debug_counts_csr(out4);
  if (rc == SPMV_UNSUPPORTED) return fail(SPMV_UNSUPPORTED, "library built without SPMV_DEBUG_CHECKS");
  if (rc || (rc = debug_counts_coo(out4)) || (rc = debug_counts_dia(out4)))
    return fail(rc, "reading the debug counters failed");
  return SPMV_OK;
}

extern "C" int spmv_plan_config_init(spmv_plan_config* cfg) {
  if (!cfg) return fail(SPMV_INVALID_ARG, "cfg is NULL");
  *cfg = config_or_default(nullptr);
  return SPMV_OK;
}
