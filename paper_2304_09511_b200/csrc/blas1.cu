// Vector kernels for the device CG (hpcg.py:211-258).
//
// The reference's CG uses np.dot partial sums reduced in rank order
// (hpcg.py:192-197) and numpy elementwise updates (round the product, then
// add: hpcg.py:243-250).  Here:
//   * dot: fixed grid of kDotBlocks x 256 threads, each thread sums a fixed
//     strided subset left to right, block tree, then one block adds the
//     partials in a fixed tree — deterministic run to run and independent of
//     the SM count (not bit-equal to BLAS ddot, whose order is unpinned);
//   * updates with explicit _rn products and sums, no FMA, like numpy.
#include "common.cuh"

namespace spmv {

constexpr int kDotBlocks = 1024;
constexpr int kDotThreads = 256;

template <typename T>
__device__ __forceinline__ T block_tree_sum(T v, T* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int w = kDotThreads / 2; w >= 32; w >>= 1) {
    if (t < w) red[t] = add_rn(red[t], red[t + w]);
    __syncthreads();
  }
  if (t < 32) {
    v = tree_reduce_warp(red[t], 32);
  }
  __syncthreads();
  return v;
}

template <typename T>
__global__ void __launch_bounds__(kDotThreads) dot_partial_kernel(int64_t n, const T* __restrict__ a,
                                                                  const T* __restrict__ b, T* __restrict__ part) {
  __shared__ T red[kDotThreads];
  T acc = T(0);
  for (int64_t i = int64_t(blockIdx.x) * kDotThreads + threadIdx.x; i < n; i += int64_t(kDotBlocks) * kDotThreads)
    acc = add_rn(acc, mul_rn(a[i], b[i]));
  acc = block_tree_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

template <typename T>
__global__ void __launch_bounds__(kDotThreads) dot_final_kernel(const T* __restrict__ part, T* __restrict__ out) {
  __shared__ T red[kDotThreads];
  T acc = T(0);
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) acc = add_rn(acc, part[i]);
  acc = block_tree_sum(acc, red);
  if (threadIdx.x == 0) *out = acc;
}

// x += alpha p ; r -= alpha Ap ; part = partial sums of r.r (new r)
template <typename T>
__global__ void __launch_bounds__(kDotThreads) cg_update_kernel(int64_t n, T alpha, const T* __restrict__ p,
                                                                const T* __restrict__ ap, T* __restrict__ x,
                                                                T* __restrict__ r, T* __restrict__ part) {
  __shared__ T red[kDotThreads];
  T acc = T(0);
  for (int64_t i = int64_t(blockIdx.x) * kDotThreads + threadIdx.x; i < n; i += int64_t(kDotBlocks) * kDotThreads) {
    x[i] = add_rn(x[i], mul_rn(alpha, p[i]));
    const T ri = add_rn(r[i], -mul_rn(alpha, ap[i]));
    r[i] = ri;
    acc = add_rn(acc, mul_rn(ri, ri));
  }
  acc = block_tree_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// p = r + beta p
template <typename T>
__global__ void cg_direction_kernel(int64_t n, T beta, const T* __restrict__ r, T* __restrict__ p) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = add_rn(r[i], mul_rn(beta, p[i]));
}

}  // namespace spmv

using namespace spmv;

extern "C" {

int spmv_dot_workspace_entries(void) { return kDotBlocks + 1; }

int spmv_dot(int dtype, int64_t n, const void* a, const void* b, void* ws, void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (n < 0 || !ws) return fail(SPMV_INVALID_ARG, "bad dot arguments");
  cudaStream_t st = as_stream(stream);
  if (dtype == SPMV_F64) {
    double* w = static_cast<double*>(ws);
    dot_partial_kernel<double><<<kDotBlocks, kDotThreads, 0, st>>>(n, static_cast<const double*>(a),
                                                                  static_cast<const double*>(b), w);
    dot_final_kernel<double><<<1, kDotThreads, 0, st>>>(w, w + kDotBlocks);
  } else {
    float* w = static_cast<float*>(ws);
    dot_partial_kernel<float><<<kDotBlocks, kDotThreads, 0, st>>>(n, static_cast<const float*>(a),
                                                                 static_cast<const float*>(b), w);
    dot_final_kernel<float><<<1, kDotThreads, 0, st>>>(w, w + kDotBlocks);
  }
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

int spmv_cg_update(int dtype, int64_t n, double alpha, const void* p, const void* ap, void* x, void* r, void* ws,
                   void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (n < 0 || !ws) return fail(SPMV_INVALID_ARG, "bad cg_update arguments");
  cudaStream_t st = as_stream(stream);
  if (dtype == SPMV_F64) {
    double* w = static_cast<double*>(ws);
    cg_update_kernel<double><<<kDotBlocks, kDotThreads, 0, st>>>(n, alpha, static_cast<const double*>(p),
                                                                static_cast<const double*>(ap),
                                                                static_cast<double*>(x), static_cast<double*>(r), w);
    dot_final_kernel<double><<<1, kDotThreads, 0, st>>>(w, w + kDotBlocks);
  } else {
    float* w = static_cast<float*>(ws);
    cg_update_kernel<float><<<kDotBlocks, kDotThreads, 0, st>>>(n, float(alpha), static_cast<const float*>(p),
                                                               static_cast<const float*>(ap), static_cast<float*>(x),
                                                               static_cast<float*>(r), w);
    dot_final_kernel<float><<<1, kDotThreads, 0, st>>>(w, w + kDotBlocks);
  }
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

int spmv_cg_direction(int dtype, int64_t n, double beta, const void* r, void* p, void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  if (n <= 0) return SPMV_OK;
  cudaStream_t st = as_stream(stream);
  int64_t grid = (n + 255) / 256;
  if (grid > int64_t(sm_count()) * 8) grid = int64_t(sm_count()) * 8;
  if (dtype == SPMV_F64)
    cg_direction_kernel<double><<<unsigned(grid), 256, 0, st>>>(n, beta, static_cast<const double*>(r),
                                                                static_cast<double*>(p));
  else
    cg_direction_kernel<float><<<unsigned(grid), 256, 0, st>>>(n, float(beta), static_cast<const float*>(r),
                                                               static_cast<float*>(p));
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

}  // extern "C"
