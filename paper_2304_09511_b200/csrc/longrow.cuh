// Long-row path shared by the CSR and COO plans.
//
// Rows longer than kExactLen entries are cut into kChunk-entry work items.
// One warp reduces one item the way spmv_csr_vla(lanes=32) reduces a row
// (kernels.py:143-171): lane l accumulates entries begin+l, begin+l+32, ...
// then the pairwise-halving tree of lanes.py:107-128.  A row of one chunk
// is therefore bit-exact with the reference's 32-lane vla kernel; a row of
// several chunks stores one partial per chunk and the last warp to finish
// (atomic ticket, no spin) adds the partials in chunk order, so the result
// is deterministic run to run and within 1e-12 of spmv_csr_plain.
#pragma once

#include <cub/cub.cuh>

#include "common.cuh"

namespace spmv {

template <typename T>
__global__ void __launch_bounds__(256)
long_rows_kernel(const LongItem* __restrict__ items, int64_t n_items,
                 const uint32_t* __restrict__ aj, const T* __restrict__ av,
                 const T* __restrict__ x, int64_t col_base, T* __restrict__ y,
                 T* __restrict__ partial, uint32_t* __restrict__ counter) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const T* xb = x - col_base;
  for (int64_t w = warp; w < n_items; w += nwarps) {
    const LongItem it = items[w];
    T acc = T(0);
    uint32_t j = it.begin + lane;
    // Four strided entries per lane in flight; the adds stay in lane order.
    for (; j + 96 < it.end; j += 128) {
      const uint32_t c0 = ld_stream(aj + j), c1 = ld_stream(aj + j + 32);
      const uint32_t c2 = ld_stream(aj + j + 64), c3 = ld_stream(aj + j + 96);
      const T v0 = ld_stream(av + j), v1 = ld_stream(av + j + 32);
      const T v2 = ld_stream(av + j + 64), v3 = ld_stream(av + j + 96);
      const T p0 = mul_rn(v0, __ldg(xb + c0)), p1 = mul_rn(v1, __ldg(xb + c1));
      const T p2 = mul_rn(v2, __ldg(xb + c2)), p3 = mul_rn(v3, __ldg(xb + c3));
      acc = add_rn(acc, p0);
      acc = add_rn(acc, p1);
      acc = add_rn(acc, p2);
      acc = add_rn(acc, p3);
    }
    for (; j < it.end; j += 32) acc = add_rn(acc, mul_rn(ld_stream(av + j), __ldg(xb + ld_stream(aj + j))));
    acc = tree_reduce_warp(acc, 32);
    if (lane == 0) {
      if (it.nchunks == 1) {
        y[it.row] = acc;
      } else {
        partial[w] = acc;
        __threadfence();
        const uint32_t ticket = atomicAdd(counter + it.first, 1u);
        if (ticket == it.nchunks - 1) {
          __threadfence();
          T s = __ldcg(partial + it.first);
          for (uint32_t c = 1; c < it.nchunks; ++c) s = add_rn(s, __ldcg(partial + it.first + c));
          y[it.row] = s;
          counter[it.first] = 0;  // ready for the next product
        }
      }
    }
  }
}

// chunks[i] = ceil(len_i / kChunk) for runs longer than exact_len, else 0.
static __global__ void count_long_chunks_kernel(const uint32_t* __restrict__ run_start, int64_t n_runs,
                                         int exact_len, uint32_t* __restrict__ chunks,
                                         unsigned long long* __restrict__ n_long) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t c = 0;
  if (i < n_runs) {
    const uint32_t len = run_start[i + 1] - run_start[i];
    if (len > uint32_t(exact_len)) c = (len + kChunk - 1) / kChunk;
    chunks[i] = c;
  }
  const unsigned long long any = __ballot_sync(0xffffffffu, c != 0);
  if ((threadIdx.x & 31) == 0 && any) atomicAdd(n_long, (unsigned long long)__popc(unsigned(any)));
}

static __global__ void fill_long_items_kernel(const uint32_t* __restrict__ run_start,
                                       const uint32_t* __restrict__ run_row, int64_t n_runs,
                                       const uint32_t* __restrict__ chunks,
                                       const uint32_t* __restrict__ base, LongItem* __restrict__ items) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_runs) return;
  const uint32_t c = chunks[i];
  if (c == 0) return;
  const uint32_t s = run_start[i], e = run_start[i + 1], b = base[i];
  const uint32_t row = run_row ? run_row[i] : uint32_t(i);
  for (uint32_t k = 0; k < c; ++k) {
    LongItem it;
    it.row = row;
    it.begin = s + k * uint32_t(kChunk);
    it.end = min(e, it.begin + uint32_t(kChunk));
    it.first = b;
    it.nchunks = c;
    it.pad0 = it.pad1 = it.pad2 = 0;
    items[b + k] = it;
  }
}

// Work list for the long runs of a run table (run_start has n_runs + 1
// entries; run_row NULL means run i is row i, as for a CSR IRP).
struct LongRows {
  DevBuf items, partial, counter;
  int64_t n_items = 0;
  int64_t n_long = 0;

  int build(const uint32_t* run_start, const uint32_t* run_row, int64_t n_runs, int exact_len,
            size_t vsize, cudaStream_t st) {
    n_items = n_long = 0;
    if (n_runs <= 0) return SPMV_OK;
    DevBuf chunks, base, tmp, cnt;
    int rc;
    if ((rc = chunks.alloc(sizeof(uint32_t) * n_runs)) || (rc = base.alloc(sizeof(uint32_t) * n_runs)) ||
        (rc = cnt.alloc(sizeof(unsigned long long) * 2)))
      return rc;
    SPMV_CUDA_TRY(cudaMemsetAsync(cnt.ptr, 0, sizeof(unsigned long long) * 2, st));
    const int tb = 256;
    const int64_t grid = (n_runs + tb - 1) / tb;
    count_long_chunks_kernel<<<unsigned(grid), tb, 0, st>>>(run_start, n_runs, exact_len,
                                                            chunks.as<uint32_t>(),
                                                            cnt.as<unsigned long long>());
    SPMV_LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    SPMV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, chunks.as<uint32_t>(),
                                                base.as<uint32_t>(), n_runs, st));
    if ((rc = tmp.alloc(tmp_bytes))) return rc;
    SPMV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, chunks.as<uint32_t>(),
                                                base.as<uint32_t>(), n_runs, st));
    uint32_t last_base = 0, last_chunks = 0;
    unsigned long long nl = 0;
    SPMV_CUDA_TRY(cudaMemcpyAsync(&last_base, base.as<uint32_t>() + n_runs - 1, 4, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaMemcpyAsync(&last_chunks, chunks.as<uint32_t>() + n_runs - 1, 4, cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaMemcpyAsync(&nl, cnt.ptr, sizeof(nl), cudaMemcpyDeviceToHost, st));
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    n_items = int64_t(last_base) + last_chunks;
    n_long = int64_t(nl);
    if (n_items == 0) return SPMV_OK;
    if ((rc = items.alloc(sizeof(LongItem) * n_items)) || (rc = partial.alloc(vsize * n_items)) ||
        (rc = counter.alloc(sizeof(uint32_t) * n_items)))
      return rc;
    SPMV_CUDA_TRY(cudaMemsetAsync(counter.ptr, 0, sizeof(uint32_t) * n_items, st));
    fill_long_items_kernel<<<unsigned(grid), tb, 0, st>>>(run_start, run_row, n_runs, chunks.as<uint32_t>(),
                                                          base.as<uint32_t>(), items.as<LongItem>());
    SPMV_LAUNCH_CHECK();
    SPMV_CUDA_TRY(cudaStreamSynchronize(st));
    return SPMV_OK;
  }

  template <typename T>
  int launch(const uint32_t* aj, const T* av, const T* x, int64_t col_base, T* y, cudaStream_t st) const {
    if (n_items == 0) return SPMV_OK;
    const int tb = 256;
    int64_t grid = (n_items + (tb / 32) - 1) / (tb / 32);
    const int64_t cap = int64_t(sm_count()) * 8;
    if (grid > cap) grid = cap;
    long_rows_kernel<T><<<unsigned(grid), tb, 0, st>>>(items.as<LongItem>(), n_items, aj, av, x, col_base, y,
                                                      partial.as<T>(), counter.as<uint32_t>());
    SPMV_LAUNCH_CHECK();
    return SPMV_OK;
  }
};

}  // namespace spmv
