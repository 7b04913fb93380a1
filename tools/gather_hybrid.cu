// Does a TMA tile::gather4 stream add to the LSU random-gather ceiling?
// Warps 0..NL-1 of each CTA gather entries [0, split) through the LSU (8
// deep, __ldg); the other warps gather [split, n) with TMA gather4 (32-byte
// rows of x, one mbarrier stage pair per warp).  Same per-entry work as
// tools/gather_ceiling.cu.  Prints G gathers/s per TMA share.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_hybrid tools/gather_hybrid.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void fill(uint32_t* idx, double* av, double* x, size_t n, uint32_t ncols) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = 42 + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    idx[i] = (uint32_t)((z >> 32) % ncols);
    av[i] = (double)(z & 0xffff) * 1e-5;
    if (i < ncols) x[i] = 1.0 + i * 1e-9;
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int S = 2;  // TMA stages per TMA warp
template <int NL>
__global__ void __launch_bounds__(256) hybrid(const __grid_constant__ CUtensorMap tmap, const uint32_t* __restrict__ idx,
                                              const double* __restrict__ av, const double* __restrict__ x,
                                              double* __restrict__ out, size_t split, size_t n) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc = 0.0;
  if (wid < NL) {
    const size_t w = blockIdx.x * (size_t)NL + wid, nw = (size_t)gridDim.x * NL;
    for (size_t base = w * 256; base < split; base += nw * 256) {
      uint32_t c[8];
      double a[8], g[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        size_t e = base + k * 32 + lane;
        bool ok = e < split;
        c[k] = ok ? __ldg(idx + e) : 0u;
        a[k] = ok ? __ldg(av + e) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) g[k] = __ldg(x + c[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, __dmul_rn(a[k], g[k]));
    }
  } else {
    constexpr int NT = 8 - NL;
    const int tw = wid - NL;
    double4* stage = reinterpret_cast<double4*>(smem) + (size_t)tw * S * 128;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)NT * S * 128 * 32) + tw * S;
    if (lane == 0) for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const size_t gw = blockIdx.x * (size_t)NT + tw, ngw = (size_t)gridDim.x * NT;
    const size_t s0 = split / 128, nsteps = n / 128;
    auto do_issue = [&](int s, size_t step) {
      uint4 c = *reinterpret_cast<const uint4*>(idx + step * 128 + lane * 4);
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bars + s)), "r"(128 * 32) : "memory");
      __syncwarp();
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                   " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                   :: "r"(su32(stage + s * 128 + lane * 4)), "l"(&tmap), "r"(su32(bars + s)),
                      "r"(0), "r"(c.x >> 2), "r"(c.y >> 2), "r"(c.z >> 2), "r"(c.w >> 2) : "memory");
    };
    size_t issue = s0 + gw;
    for (int s = 0; s < S && issue < nsteps; ++s, issue += ngw) do_issue(s, issue);
    int sc = 0;
    size_t it = 0;
    for (size_t cons = s0 + gw; cons < nsteps; cons += ngw, ++it) {
      asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                   :: "r"(su32(bars + sc)), "r"((uint32_t)((it / S) & 1)) : "memory");
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        size_t e = cons * 128 + k * 32 + lane;
        uint32_t c = __ldg(idx + e);
        double v = reinterpret_cast<const double*>(stage + sc * 128 + k * 32 + lane)[c & 3];
        acc = __dadd_rn(acc, __dmul_rn(__ldg(av + e), v));
      }
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (issue < nsteps) { do_issue(sc, issue); issue += ngw; }
      sc = (sc + 1) % S;
    }
  }
  out[blockIdx.x * (size_t)blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int NL>
void run(const CUtensorMap& tm, const uint32_t* idx, const double* av, const double* x, double* out, size_t n,
         double frac_tma, int ctas, int sms) {
  size_t split = (size_t)((1.0 - frac_tma) * n) / 128 * 128;
  if (NL == 8) split = n;
  size_t n128 = n / 128 * 128;
  size_t smem = (size_t)(8 - NL) * S * (128 * 32 + 8);
  auto k = hybrid<NL>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = sms * ctas;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) k<<<grid, 256, smem>>>(tm, idx, av, x, out, split, n128);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < 30; ++i) k<<<grid, 256, smem>>>(tm, idx, av, x, out, split, n128);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  double t = ms * 1e-3 / 30;
  printf("{\"lsu_warps\": %d, \"tma_frac\": %.3f, \"ctas_per_sm\": %d, \"us\": %.1f, \"ggathers_per_s\": %.1f}\n", NL,
         NL == 8 ? 0.0 : 1.0 - (double)split / n128, ctas, t * 1e6, n128 / t * 1e-9);
}

int main() {
  size_t n = 41849856;
  uint32_t ncols = 2000000;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t* idx;
  double *av, *x, *out;
  CK(cudaMalloc(&idx, n * 4));
  CK(cudaMalloc(&av, n * 8));
  CK(cudaMalloc(&x, (size_t)ncols * 8 + 64));
  CK(cudaMalloc(&out, (size_t)sms * 8 * 256 * 8));
  fill<<<sms * 8, 256>>>(idx, av, x, n, ncols);
  CK(cudaDeviceSynchronize());
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[2] = {4, (cuuint64_t)(ncols + 3) / 4};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  run<8>(tm, idx, av, x, out, n, 0.0, 4, sms);
  for (double f : {0.2, 0.3, 0.4}) {
    run<6>(tm, idx, av, x, out, n, f, 4, sms);
    run<5>(tm, idx, av, x, out, n, f, 4, sms);
    run<4>(tm, idx, av, x, out, n, f, 4, sms);
  }
  return 0;
}
