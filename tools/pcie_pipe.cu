// PCIe pipeline probe: what does the H2D -> compute -> D2H dependency pattern
// of the host-buffer products cost against free-running copies?
//   nvcc -O2 -arch=sm_100a -o /tmp/pcie_pipe tools/pcie_pipe.cu && /tmp/pcie_pipe
// Cases (134 MB each way, pinned): whole-buffer copies alone / together;
// chunked copies without events; the gated chain (H2D chunk -> stand-in kernel
// -> D2H chunk) per chunk size; copy kernels on a few SMs over mapped host
// memory instead of the copy engines, for either direction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t err_ = (x);                                                       \
    if (err_ != cudaSuccess) {                                                  \
      std::printf("%s: %s\n", #x, cudaGetErrorString(err_));                    \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void touch_kernel(const double* x, double* y, size_t lo, size_t hi) {
  for (size_t i = lo + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < hi; i += size_t(gridDim.x) * blockDim.x)
    y[i] = x[i] + 1.0;
}

// dst[0, n) = src[0, n) with 16-byte accesses
__global__ void copy_kernel(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(src + i));
    dst[i] = v;
  }
}

int main() {
  const size_t n = size_t(256) * 256 * 256, bytes = n * 8;
  double *xh, *yh, *xd, *yd;
  CK(cudaHostAlloc(&xh, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&yh, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&xd, bytes));
  CK(cudaMalloc(&yd, bytes));
  for (size_t i = 0; i < n; ++i) xh[i] = double(i & 1023);
  CK(cudaMemset(yd, 0, bytes));
  cudaStream_t sa, sb, sc;
  CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  cudaEvent_t t0, t1, t2;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventCreate(&t2));
  std::vector<cudaEvent_t> ev(1024);
  for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  auto median = [](std::vector<float> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  const int reps = 7;

  // 1. whole copies alone and together
  {
    std::vector<float> a, b, c;
    for (int r = 0; r < reps; ++r) {
      float ms;
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(t0, sa));
      CK(cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice, sa));
      CK(cudaEventRecord(t1, sa));
      CK(cudaDeviceSynchronize());
      CK(cudaEventElapsedTime(&ms, t0, t1));
      a.push_back(ms);
      CK(cudaEventRecord(t0, sc));
      CK(cudaMemcpyAsync(yh, yd, bytes, cudaMemcpyDeviceToHost, sc));
      CK(cudaEventRecord(t1, sc));
      CK(cudaDeviceSynchronize());
      CK(cudaEventElapsedTime(&ms, t0, t1));
      b.push_back(ms);
      CK(cudaEventRecord(t0, sb));
      CK(cudaStreamWaitEvent(sa, t0, 0));
      CK(cudaStreamWaitEvent(sc, t0, 0));
      CK(cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice, sa));
      CK(cudaMemcpyAsync(yh, yd, bytes, cudaMemcpyDeviceToHost, sc));
      CK(cudaEventRecord(ev[0], sa));
      CK(cudaEventRecord(ev[1], sc));
      CK(cudaStreamWaitEvent(sb, ev[0], 0));
      CK(cudaStreamWaitEvent(sb, ev[1], 0));
      CK(cudaEventRecord(t1, sb));
      CK(cudaDeviceSynchronize());
      CK(cudaEventElapsedTime(&ms, t0, t1));
      c.push_back(ms);
    }
    std::printf("whole: H2D alone %.3f ms (%.1f GB/s)  D2H alone %.3f ms (%.1f GB/s)  both %.3f ms (%.1f GB/s each)\n",
                median(a), bytes / median(a) / 1e6, median(b), bytes / median(b) / 1e6, median(c),
                bytes / median(c) / 1e6);
  }

  // 2. chunked, no events / gated chain, per chunk size
  for (int gated = 0; gated <= 2; ++gated)
    for (size_t mb : {2, 4, 8, 16, 32}) {
      const size_t step = mb << 17;  // doubles per chunk
      const int nc = int((n + step - 1) / step);
      std::vector<float> c;
      for (int r = 0; r < reps; ++r) {
        float ms;
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(t0, sb));
        CK(cudaStreamWaitEvent(sa, t0, 0));
        CK(cudaStreamWaitEvent(sc, t0, 0));
        for (int j = 0; j < nc; ++j) {
          const size_t lo = j * step, hi = std::min(n, lo + step);
          CK(cudaMemcpyAsync(xd + lo, xh + lo, (hi - lo) * 8, cudaMemcpyHostToDevice, sa));
          if (gated) {
            CK(cudaEventRecord(ev[2 * j], sa));
            CK(cudaStreamWaitEvent(sb, ev[2 * j], 0));
            if (gated == 2) touch_kernel<<<148, 256, 0, sb>>>(xd, yd, lo, hi);
            CK(cudaEventRecord(ev[2 * j + 1], sb));
            CK(cudaStreamWaitEvent(sc, ev[2 * j + 1], 0));
          }
          CK(cudaMemcpyAsync(yh + lo, yd + lo, (hi - lo) * 8, cudaMemcpyDeviceToHost, sc));
        }
        CK(cudaEventRecord(ev[1000], sa));
        CK(cudaEventRecord(ev[1001], sc));
        CK(cudaStreamWaitEvent(sb, ev[1000], 0));
        CK(cudaStreamWaitEvent(sb, ev[1001], 0));
        CK(cudaEventRecord(t1, sb));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms, t0, t1));
        c.push_back(ms);
      }
      std::printf("%s chunks of %2zu MB (%3d): %.3f ms\n",
                  gated == 0 ? "free " : gated == 1 ? "gated (events only)" : "gated (+ kernel)   ", mb, nc, median(c));
    }

  // 3. copy kernels over mapped host memory
  double *xm, *ym;
  CK(cudaHostGetDevicePointer(&xm, xh, 0));
  CK(cudaHostGetDevicePointer(&ym, yh, 0));
  for (int ctas : {4, 8, 16, 32, 64}) {
    std::vector<float> a, b, c, d;
    for (int r = 0; r < 5; ++r) {
      float ms;
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(t0, sa));
      copy_kernel<<<ctas, 512, 0, sa>>>(reinterpret_cast<const double2*>(xm), reinterpret_cast<double2*>(xd), n / 2);
      CK(cudaEventRecord(t1, sa));
      CK(cudaDeviceSynchronize());
      CK(cudaEventElapsedTime(&ms, t0, t1));
      a.push_back(ms);
      CK(cudaEventRecord(t0, sc));
      copy_kernel<<<ctas, 512, 0, sc>>>(reinterpret_cast<const double2*>(yd), reinterpret_cast<double2*>(ym), n / 2);
      CK(cudaEventRecord(t1, sc));
      CK(cudaDeviceSynchronize());
      CK(cudaEventElapsedTime(&ms, t0, t1));
      b.push_back(ms);
      // both directions by kernels
      CK(cudaEventRecord(t0, sb));
      CK(cudaStreamWaitEvent(sa, t0, 0));
      CK(cudaStreamWaitEvent(sc, t0, 0));
      copy_kernel<<<ctas, 512, 0, sa>>>(reinterpret_cast<const double2*>(xm), reinterpret_cast<double2*>(xd), n / 2);
      copy_kernel<<<ctas, 512, 0, sc>>>(reinterpret_cast<const double2*>(yd), reinterpret_cast<double2*>(ym), n / 2);
      CK(cudaEventRecord(ev[0], sa));
      CK(cudaEventRecord(ev[1], sc));
      CK(cudaStreamWaitEvent(sb, ev[0], 0));
      CK(cudaStreamWaitEvent(sb, ev[1], 0));
      CK(cudaEventRecord(t1, sb));
      CK(cudaDeviceSynchronize());
      CK(cudaEventElapsedTime(&ms, t0, t1));
      c.push_back(ms);
      // H2D by the copy engine, D2H by a kernel
      CK(cudaEventRecord(t0, sb));
      CK(cudaStreamWaitEvent(sa, t0, 0));
      CK(cudaStreamWaitEvent(sc, t0, 0));
      CK(cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice, sa));
      copy_kernel<<<ctas, 512, 0, sc>>>(reinterpret_cast<const double2*>(yd), reinterpret_cast<double2*>(ym), n / 2);
      CK(cudaEventRecord(ev[0], sa));
      CK(cudaEventRecord(ev[1], sc));
      CK(cudaStreamWaitEvent(sb, ev[0], 0));
      CK(cudaStreamWaitEvent(sb, ev[1], 0));
      CK(cudaEventRecord(t1, sb));
      CK(cudaDeviceSynchronize());
      CK(cudaEventElapsedTime(&ms, t0, t1));
      d.push_back(ms);
    }
    std::printf("copy kernels, %2d CTAs: H2D %.3f ms  D2H %.3f ms  both %.3f ms  CE H2D + kernel D2H %.3f ms\n", ctas,
                median(a), median(b), median(c), median(d));
  }
  return 0;
}
