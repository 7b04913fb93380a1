// Host-buffer products: x in host memory, y to host memory, PCIe-bound.
//
// The reference contract is fn(matrix, numpy x, config) -> fresh numpy y
// (kernels.py:46-53, :59, :72, :94).  A product whose x and y live on the
// host moves 2 x n x 8 bytes over PCIe (134 MB each way at 256^3) against
// ~0.8 ms of kernel time, so the pipeline overlaps three things: x goes up
// in column chunks on one copy stream, each part of the product runs on the
// caller's stream as soon as the x prefix it reads has arrived, and
// finished rows of y come down on a second copy stream (PCIe is full
// duplex).  The format decides what "the part that needs x[0, c)" is
// (CSR: tile ranges by their largest column; DIA: row blocks by the largest
// offset; COO: the whole product after the last chunk).
//
// Pinned x is copied directly.  Pageable x (a plain numpy array) is staged
// through a pinned ring owned by the pipe: host threads copy chunk j into a
// free slot while the DMA of chunk j - 1 runs.  y should be pinned (the
// Python layer returns a fresh numpy array over pinned memory); a pageable
// y is still correct, its copies are just not overlapped.
//
// One pipe serves one call at a time (its device staging and copy streams
// are shared): calls are serialised by a mutex on the host and, on the
// device, each call waits for the previous call's end.
#pragma once

#include <condition_variable>
#include <cstring>
#include <functional>
#include <thread>

#include "common.cuh"

namespace spmv {

// Small persistent pool for parallel host copies into the pinned ring.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  // dst[0, n) = src[0, n), split over the pool's threads
  void copy(void* dst, const void* src, size_t n) {
    const int parts = n < (size_t(1) << 20) ? 1 : nthreads_ + 1;
    if (parts == 1) {
      std::memcpy(dst, src, n);
      return;
    }
    std::unique_lock<std::mutex> lock(mu_);
    job_dst_ = static_cast<char*>(dst);
    job_src_ = static_cast<const char*>(src);
    job_n_ = n;
    job_parts_ = parts;
    pending_ = nthreads_;
    ++gen_;
    cv_.notify_all();
    lock.unlock();
    do_part(0);  // the caller takes part 0
    lock.lock();
    done_cv_.wait(lock, [&] { return pending_ == 0; });
  }

 private:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = int(std::max(1u, std::min(7u, hw > 2 ? hw / 2 - 1 : 1u)));
    for (int i = 0; i < nthreads_; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void do_part(int k) {
    const size_t lo = job_n_ * size_t(k) / size_t(job_parts_), hi = job_n_ * size_t(k + 1) / size_t(job_parts_);
    if (hi > lo) std::memcpy(job_dst_ + lo, job_src_ + lo, hi - lo);
  }
  void loop(int k) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lock(mu_);
    while (true) {
      cv_.wait(lock, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      lock.unlock();
      do_part(k);
      lock.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> workers_;
  int nthreads_ = 1, job_parts_ = 1, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  char* job_dst_ = nullptr;
  const char* job_src_ = nullptr;
  size_t job_n_ = 0;
};

inline bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

struct HostPipe {
  std::mutex mu;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t done = nullptr;  // end of the previous call
  std::vector<cudaEvent_t> ev;
  DevBuf xd, yd;
  char* ring = nullptr;  // pinned staging for pageable x
  static constexpr size_t kSlotBytes = size_t(8) << 20;
  static constexpr int kSlots = 4;
  cudaEvent_t slot_ev[kSlots] = {};
  bool slot_used[kSlots] = {};

  ~HostPipe() {
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (done) cudaEventDestroy(done);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : slot_ev)
      if (e) cudaEventDestroy(e);
    if (ring) cudaFreeHost(ring);
  }

  int prepare(size_t xbytes, size_t ybytes, int nev, bool staged) {
    if (!h2d) {
      SPMV_CUDA_TRY(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
      SPMV_CUDA_TRY(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
      SPMV_CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    }
    int rc;
    if (xd.bytes < xbytes && (rc = xd.alloc(xbytes))) return rc;
    if (yd.bytes < ybytes && (rc = yd.alloc(ybytes))) return rc;
    while (int(ev.size()) < nev) {
      cudaEvent_t e;
      SPMV_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    if (staged && !ring) {
      SPMV_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ring), kSlotBytes * kSlots, cudaHostAllocDefault));
      for (auto& e : slot_ev) SPMV_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return SPMV_OK;
  }
};

// Column chunks of x: ramp up from 1/16 of a full chunk (so the first rows
// of y can leave early), full chunks of max(ncols / chunks, 1M) in the
// middle, ramp down at the end (copies under ~8 MB lose PCIe bandwidth when
// both directions run).
inline std::vector<int64_t> host_x_chunks(int64_t n, int chunks) {
  std::vector<int64_t> xb{0};
  const int64_t big = std::max<int64_t>(std::max<int64_t>(1, n / std::max(chunks, 1)),
                                        std::min<int64_t>(n, int64_t(1) << 20));
  std::vector<int64_t> ramp;
  for (int sh = 4; sh >= 1; --sh)
    if ((big >> sh) >= 4096) ramp.push_back(big >> sh);
  int64_t ramp_total = 0;
  for (int64_t r : ramp) ramp_total += 2 * r;
  if (2 * ramp_total > n) ramp.clear(), ramp_total = 0;
  for (int64_t r : ramp) xb.push_back(xb.back() + r);
  const int64_t mid = n - ramp_total, nmid = std::max<int64_t>(1, (mid + big / 2) / big);
  const int64_t m0 = xb.back();
  for (int64_t j = 1; j <= nmid; ++j) xb.push_back(m0 + mid * j / nmid);
  for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) xb.push_back(xb.back() + *it);
  xb.back() = n;
  return xb;
}

// One host-buffer product.  compute(j, xd, yd, st) enqueues on `st` the
// work that needs only x[0, xb[j+1]) and returns how many leading rows of y
// are then final (non-decreasing over j; the last call must finish the
// product).  yfinal_at_end: y rows only become final with the last call
// (e.g. a fix-up kernel adds long rows at the end).
template <typename Compute>
int run_host_pipeline(HostPipe& hp, const void* xh, void* yh, size_t esz, int64_t ncols, int64_t nrows,
                      const std::vector<int64_t>& xb, Compute&& compute, bool yfinal_at_end, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(hp.mu);
  const bool pinned = host_pinned(xh);
  const int nx = int(xb.size()) - 1;
  int rc = hp.prepare(esz * std::max<int64_t>(ncols, 1), esz * std::max<int64_t>(nrows, 1), 2 * nx + 2, !pinned);
  if (rc) return rc;
  char* xd = static_cast<char*>(hp.xd.ptr);
  char* yd = static_cast<char*>(hp.yd.ptr);
  const char* xs = static_cast<const char*>(xh);
  char* ys = static_cast<char*>(yh);
  cudaEvent_t* ev = hp.ev.data();  // [0, nx): x chunks, [nx, 2nx): compute, 2nx: start, 2nx+1: end
  SPMV_CUDA_TRY(cudaStreamWaitEvent(st, hp.done, 0));  // the previous call's staging is free
  SPMV_CUDA_TRY(cudaEventRecord(ev[2 * nx], st));
  SPMV_CUDA_TRY(cudaStreamWaitEvent(hp.h2d, ev[2 * nx], 0));
  SPMV_CUDA_TRY(cudaStreamWaitEvent(hp.d2h, ev[2 * nx], 0));
  int64_t done = 0;
  int slot = 0;
  for (int j = 0; j < nx; ++j) {
    const size_t b0 = esz * size_t(xb[j]), b1 = esz * size_t(xb[j + 1]);
    if (pinned) {
      if (b1 > b0) SPMV_CUDA_TRY(cudaMemcpyAsync(xd + b0, xs + b0, b1 - b0, cudaMemcpyHostToDevice, hp.h2d));
    } else {
      for (size_t o = b0; o < b1; o += HostPipe::kSlotBytes, slot = (slot + 1) % HostPipe::kSlots) {
        const size_t n = std::min(HostPipe::kSlotBytes, b1 - o);
        if (hp.slot_used[slot]) SPMV_CUDA_TRY(cudaEventSynchronize(hp.slot_ev[slot]));  // its DMA is done
        char* sp = hp.ring + size_t(slot) * HostPipe::kSlotBytes;
        CopyPool::get().copy(sp, xs + o, n);
        SPMV_CUDA_TRY(cudaMemcpyAsync(xd + o, sp, n, cudaMemcpyHostToDevice, hp.h2d));
        SPMV_CUDA_TRY(cudaEventRecord(hp.slot_ev[slot], hp.h2d));
        hp.slot_used[slot] = true;
      }
    }
    SPMV_CUDA_TRY(cudaEventRecord(ev[j], hp.h2d));
    SPMV_CUDA_TRY(cudaStreamWaitEvent(st, ev[j], 0));
    const int64_t rows = compute(j, xd, yd, st);
    if (rows < 0) return -int(rows);  // an error status from compute
    if (!yfinal_at_end && rows > done) {
      SPMV_CUDA_TRY(cudaEventRecord(ev[nx + j], st));
      SPMV_CUDA_TRY(cudaStreamWaitEvent(hp.d2h, ev[nx + j], 0));
      SPMV_CUDA_TRY(cudaMemcpyAsync(ys + esz * size_t(done), yd + esz * size_t(done), esz * size_t(rows - done),
                                    cudaMemcpyDeviceToHost, hp.d2h));
      done = rows;
    }
  }
  if (done < nrows) {
    SPMV_CUDA_TRY(cudaEventRecord(ev[2 * nx - 1], st));
    SPMV_CUDA_TRY(cudaStreamWaitEvent(hp.d2h, ev[2 * nx - 1], 0));
    SPMV_CUDA_TRY(cudaMemcpyAsync(ys + esz * size_t(done), yd + esz * size_t(done), esz * size_t(nrows - done),
                                  cudaMemcpyDeviceToHost, hp.d2h));
  }
  SPMV_CUDA_TRY(cudaEventRecord(ev[2 * nx + 1], hp.d2h));
  SPMV_CUDA_TRY(cudaStreamWaitEvent(st, ev[2 * nx + 1], 0));
  SPMV_CUDA_TRY(cudaEventRecord(hp.done, st));
  return SPMV_OK;
}

}  // namespace spmv
