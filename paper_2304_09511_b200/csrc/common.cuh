// Shared helpers for the sm_100a SpMV kernels and their C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/spmv_b200.h"

// Internal entry points shared between translation units (not part of
// include/spmv_b200.h).
extern "C" int spmvi_csr_vla_tiles(spmv_csr_plan* plan, const uint32_t* irp, const uint32_t* aj, const void* av,
                                  const void* x, int64_t col_base, void* y, int lanes, void* stream, int* done);

namespace spmv {

// ---------------------------------------------------------------- errors --
void set_error(int code, const char* fmt, ...);
int fail(int code, const char* fmt, ...);

#define SPMV_CUDA_TRY(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess)                                                    \
      return ::spmv::fail(SPMV_CUDA_ERROR, "%s failed: %s (%s:%d)", #expr,    \
                          cudaGetErrorString(_e), __FILE__, __LINE__);        \
  } while (0)

#define SPMV_LAUNCH_CHECK()                                                   \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess)                                                    \
      return ::spmv::fail(SPMV_CUDA_ERROR, "kernel launch failed: %s (%s:%d)",\
                          cudaGetErrorString(_e), __FILE__, __LINE__);        \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Device scratch owned by plans and builders.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int alloc(size_t n) {
    release();
    if (n == 0) return SPMV_OK;
    cudaError_t e = cudaMalloc(&ptr, n);
    if (e != cudaSuccess) {
      ptr = nullptr;
      return fail(SPMV_CUDA_ERROR, "cudaMalloc(%zu) failed: %s", n, cudaGetErrorString(e));
    }
    bytes = n;
    return SPMV_OK;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(ptr); }
  ~DevBuf() { release(); }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Stream-ordered scratch from the device's default memory pool (conversions
// allocate GB-sized temporaries per call; cudaMalloc/cudaFree would map and
// unmap them and synchronise the device every time).  The pool keeps up to
// kPoolKeepBytes cached between calls.
constexpr uint64_t kPoolKeepBytes = uint64_t(32) << 30;
int pool_keep_memory();  // once per device; capi.cu
struct ScratchBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
  int alloc(size_t n, cudaStream_t s) {
    release();
    if (n == 0) return SPMV_OK;
    int rc = pool_keep_memory();
    if (rc) return rc;
    cudaError_t e = cudaMallocAsync(&ptr, n, s);
    if (e != cudaSuccess) {
      ptr = nullptr;
      return fail(SPMV_CUDA_ERROR, "cudaMallocAsync(%zu) failed: %s", n, cudaGetErrorString(e));
    }
    bytes = n;
    st = s;
    return SPMV_OK;
  }
  void release() {
    if (ptr) cudaFreeAsync(ptr, st);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(ptr); }
  ~ScratchBuf() { release(); }
  ScratchBuf() = default;
  ScratchBuf(const ScratchBuf&) = delete;
  ScratchBuf& operator=(const ScratchBuf&) = delete;
};

// Per-stream launch scratch of a plan (partial-sum slots, range counters).
// Two launches on different streams get different slots, so one plan can
// serve concurrent products; launches on one stream are
// ordered, so they share theirs.  A slot is allocated and zero-filled on its
// stream the first time that stream launches, then reused.
struct StreamSlots {
  struct Slot {
    cudaStream_t st;
    void* ptr;
  };
  std::mutex mu;
  std::vector<Slot> slots;
  size_t bytes = 0;  // per slot
  int get(cudaStream_t st, void** out) {
    *out = nullptr;
    if (bytes == 0) return SPMV_OK;
    std::lock_guard<std::mutex> lock(mu);
    for (const Slot& s : slots)
      if (s.st == st) {
        *out = s.ptr;
        return SPMV_OK;
      }
    // A stream's first product may be inside a CUDA graph capture (global
    // capture mode forbids cudaMalloc): allocate under relaxed mode; the
    // zero fill below is then captured as the graph's first node on this
    // stream and re-zeroes the slot at every replay.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) {
      cudaGetLastError();
      cap = cudaStreamCaptureStatusNone;
    }
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    if (cap == cudaStreamCaptureStatusActive) cudaThreadExchangeStreamCaptureMode(&mode);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (cap == cudaStreamCaptureStatusActive) cudaThreadExchangeStreamCaptureMode(&mode);
    if (e != cudaSuccess) return fail(SPMV_CUDA_ERROR, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    e = cudaMemsetAsync(p, 0, bytes, st);
    if (e != cudaSuccess) {
      cudaFree(p);
      return fail(SPMV_CUDA_ERROR, "cudaMemsetAsync failed: %s", cudaGetErrorString(e));
    }
    slots.push_back({st, p});
    *out = p;
    return SPMV_OK;
  }
  void release() {
    std::lock_guard<std::mutex> lock(mu);
    for (const Slot& s : slots) cudaFree(s.ptr);  // cudaFree waits for the device
    slots.clear();
  }
  ~StreamSlots() { release(); }
};

// Byte layout of one scratch slot: add(n) reserves n bytes (256-aligned).
struct SlotLayout {
  size_t total = 0;
  size_t add(size_t n) {
    const size_t off = total;
    total += (n + 255) & ~size_t(255);
    return off;
  }
};

// Plan configuration with auto values resolved (include/spmv_b200.h).
inline spmv_plan_config config_or_default(const spmv_plan_config* c) {
  spmv_plan_config d;
  d.version = SPMV_PLAN_CONFIG_VERSION;
  d.tile = 0;
  d.groups = 0;
  d.exact_len = 0;
  d.warp_stream = -1;
  d.ranges_per_warp = 0;
  d.tma_hint = -1;
  d.ctas_per_sm = 0;
  d.dia_kernel = -1;
  d.dia_rows = 0;
  d.flags = 0;
  d.panels = -1;
  for (int i = 0; i < 4; ++i) d.reserved[i] = 0;
  return c ? *c : d;
}
inline int cap_ctas(int per_sm, int cap) {
  if (cap > 0 && per_sm > cap) per_sm = cap;
  return per_sm < 1 ? 1 : per_sm;
}

inline size_t value_size(int dtype) { return dtype == SPMV_F64 ? 8 : 4; }

// ---- debug builds (-DSPMV_DEBUG_CHECKS; _build.build(debug=True)) -----------
// Device-side consistency checks in place of compute-sanitizer (closed on
// this pool): every TMA-staged tile / step / x panel is compared with global
// memory after its barrier completes (a stale or half-written stage, i.e. a
// ring race, shows up as a mismatch), and the panel path's indices are
// bounds-checked.  Counters per translation unit: [0] stage mismatch,
// [1] index out of range, [2] x panel mismatch, [3] other.
#ifdef SPMV_DEBUG_CHECKS
static __device__ unsigned long long spmv_dbg_counts[4];
#define SPMV_DCHECK(cond, k)                                      \
  do {                                                            \
    if (!(cond)) atomicAdd(&spmv_dbg_counts[k], 1ull);             \
  } while (0)
static inline int debug_read_tu(unsigned long long* out4) {
  unsigned long long h[4] = {0, 0, 0, 0};
  if (cudaDeviceSynchronize() != cudaSuccess) return SPMV_CUDA_ERROR;
  if (cudaMemcpyFromSymbol(h, spmv_dbg_counts, sizeof(h)) != cudaSuccess) return SPMV_CUDA_ERROR;
  const unsigned long long z[4] = {0, 0, 0, 0};
  if (cudaMemcpyToSymbol(spmv_dbg_counts, z, sizeof(z)) != cudaSuccess) return SPMV_CUDA_ERROR;
  for (int i = 0; i < 4; ++i) out4[i] += h[i];
  return SPMV_OK;
}
#else
#define SPMV_DCHECK(cond, k) \
  do {                       \
  } while (0)
static inline int debug_read_tu(unsigned long long*) { return SPMV_UNSUPPORTED; }
#endif
template <typename T> __device__ __forceinline__ bool same_bits(T a, T b);
template <> __device__ __forceinline__ bool same_bits<double>(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}
template <> __device__ __forceinline__ bool same_bits<float>(float a, float b) {
  return __float_as_uint(a) == __float_as_uint(b);
}
inline bool valid_dtype(int dtype) { return dtype == SPMV_F32 || dtype == SPMV_F64; }

// ------------------------------------------------------------ arithmetic --
// The reference never fuses multiply-add (kernels.py:65,75,81,100 and
// lanes.py:104 round the product, then add).  Explicit _rn intrinsics keep
// nvcc from contracting to FMA, so every product/sum rounds like numpy.
template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }

// Streaming (read-once) loads: bypass L1 allocation so the x window keeps L1.
template <typename T> __device__ __forceinline__ T ld_stream(const T* p);
template <> __device__ __forceinline__ double ld_stream<double>(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ float ld_stream<float>(const float* p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ uint32_t ld_stream<uint32_t>(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// x gathers go through the read-only path.  (An L2 evict_last policy on
// them cost DIA a third of its throughput; see profiles/r1_notes.md.)
template <typename T> __device__ __forceinline__ T ldx(const T* p) {
#ifdef SPMV_NO_X  // experiment: gathers replaced by a constant (results wrong)
  (void)p;
  return T(1);
#else
  return __ldg(p);
#endif
}

// Warp tree of lanes.py:107-128: vals[:w] + vals[w:2w] for w = W/2 .. 1.
// shfl_down by w hands lane i the value of lane i+w, i.e. the same pairs in
// the same operand order.
template <typename T>
__device__ __forceinline__ T tree_reduce_warp(T v, int width) {
  for (int w = width >> 1; w >= 1; w >>= 1)
    v = add_rn(v, __shfl_down_sync(0xffffffffu, v, w, width));
  return v;
}

// Long-row work item shared by the CSR and COO plans: entries [begin, end)
// of one row; rows with nchunks > 1 combine partials[first .. first+nchunks)
// in chunk order.
struct LongItem {
  uint32_t row;
  uint32_t begin;
  uint32_t end;
  uint32_t first;
  uint32_t nchunks;
  uint32_t pad0, pad1, pad2;
};

constexpr int kExactLen = 32;        // rows up to this length are summed by one thread
constexpr int kChunk = 2048;         // entries per long-row warp item

}  // namespace spmv
