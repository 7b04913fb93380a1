// Random-gather ceiling probe for the Zipf config (C3).
//
// C3's columns are uniform over 2M, so every x read is one random 32-byte L2
// sector for 8 useful bytes. This probe measures how many such gathers per
// second the B200 memory system serves when nothing else limits the kernel:
// a coalesced index stream (4 B/entry, like CSR's col_indices) plus a value
// stream (8 B/entry) and one random x gather per entry, summed per thread.
// The best variant is the practical ceiling for any C3 SpMV kernel; it is
// reported beside the HBM roofline (profiles/).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_ceiling tools/gather_ceiling.cu
//   ./gather_ceiling [n_entries=41849860] [ncols=2000000]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void fill_idx(uint32_t* idx, double* av, size_t n, uint32_t ncols, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    idx[i] = (uint32_t)((z >> 32) % ncols);
    av[i] = (double)(z & 0xffff) * 1e-5;
  }
}

__global__ void fill_x(double* x, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = 1.0 + i * 1e-9;
}

enum Mode { NC = 0, NC_NOALLOC = 1, CG = 2, NO_VALS = 3 };

template <int MODE>
__device__ __forceinline__ double gather(const double* p) {
  double v;
  if (MODE == NC || MODE == NO_VALS) {
    v = __ldg(p);
  } else if (MODE == NC_NOALLOC) {
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  } else {
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  }
  return v;
}

// Each warp takes chunks of 32*DEPTH consecutive entries: lane l reads
// entries chunk + k*32 + l (coalesced), issues all DEPTH gathers, then sums.
template <int MODE, int DEPTH>
__global__ void gather_kernel(const uint32_t* __restrict__ idx, const double* __restrict__ av,
                              const double* __restrict__ x, double* __restrict__ out, size_t n) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t chunk = 32 * DEPTH;
  double acc = 0.0;
  for (size_t base = warp * chunk; base < n; base += nwarps * chunk) {
    uint32_t c[DEPTH];
    double a[DEPTH];
#pragma unroll
    for (int k = 0; k < DEPTH; ++k) {
      size_t e = base + k * 32 + lane;
      bool ok = e < n;
      c[k] = ok ? __ldg(idx + e) : 0u;
      a[k] = (MODE == NO_VALS) ? 1.0 : (ok ? __ldg(av + e) : 0.0);
    }
    double g[DEPTH];
#pragma unroll
    for (int k = 0; k < DEPTH; ++k) g[k] = gather<MODE>(x + c[k]);
#pragma unroll
    for (int k = 0; k < DEPTH; ++k) acc = __dadd_rn(acc, __dmul_rn(a[k], g[k]));
  }
  out[blockIdx.x * (size_t)blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int DEPTH>
static void run(const char* name, const uint32_t* idx, const double* av, const double* x, double* out,
                size_t n, int threads, int ctas_per_sm, int sms) {
  auto k = gather_kernel<MODE, DEPTH>;
  int grid = sms * ctas_per_sm;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) k<<<grid, threads>>>(idx, av, x, out, n);
  if (cudaGetLastError() != cudaSuccess) { printf("{\"variant\": \"%s\", \"depth\": %d, \"threads\": %d, \"error\": \"launch\"}\n", name, DEPTH, threads); return; }
  const int reps = 50;
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) k<<<grid, threads>>>(idx, av, x, out, n);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  double t = ms * 1e-3 / reps;
  printf("{\"variant\": \"%s\", \"depth\": %d, \"threads\": %d, \"ctas_per_sm\": %d, \"us\": %.2f, "
         "\"ggathers_per_s\": %.1f, \"spmv_equiv_gflops\": %.1f}\n",
         name, DEPTH, threads, ctas_per_sm, t * 1e6, n / t * 1e-9, 2.0 * n / t * 1e-9);
}

// ---- TMA gather4 variant: x viewed as [ncols/4][4] f64 rows (32 B = one L2
// sector; 128 B per gather4, the smem alignment it needs); one cp.async.bulk.tensor ... tile::gather4 fetches 4
// rows. Each warp owns S stages of 128 entries (32 lanes x one gather4).
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void __launch_bounds__(256) gather4_kernel(const __grid_constant__ CUtensorMap tmap,
    const uint32_t* __restrict__ idx, const double* __restrict__ av, double* __restrict__ out, size_t n) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double4* stage = reinterpret_cast<double4*>(smem) + (size_t)wid * S * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nw * S * 128 * 32) + wid * S;
  if (lane == 0) for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bars + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const size_t gw = blockIdx.x * (size_t)nw + wid, ngw = (size_t)gridDim.x * nw;
  const size_t nsteps = n / 128;
  double acc = 0.0;
  size_t issue = gw, consume = gw;
  auto do_issue = [&](int s, size_t step) {
    uint4 c = *reinterpret_cast<const uint4*>(idx + step * 128 + lane * 4);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bars + s)), "r"(128 * 32) : "memory");
    __syncwarp();
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                 :: "r"(su32(stage + s * 128 + lane * 4)), "l"(&tmap), "r"(su32(bars + s)),
                    "r"(0), "r"(c.x >> 2), "r"(c.y >> 2), "r"(c.z >> 2), "r"(c.w >> 2) : "memory");
  };
  for (int s = 0; s < S && issue < nsteps; ++s, issue += ngw) do_issue(s, issue);
  int s_cons = 0;
  for (; consume < nsteps; consume += ngw) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                 :: "r"(su32(bars + s_cons)), "r"((uint32_t)(((consume - gw) / ngw / S) & 1)) : "memory");
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      size_t e = consume * 128 + k * 32 + lane;
      uint32_t c = __ldg(idx + e);
      double v = reinterpret_cast<const double*>(stage + s_cons * 128 + k * 32 + lane)[c & 3];
      acc = __dadd_rn(acc, __dmul_rn(__ldg(av + e), v));
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (issue < nsteps) { do_issue(s_cons, issue); issue += ngw; }
    s_cons = (s_cons + 1) % S;
  }
  out[blockIdx.x * (size_t)blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S>
static void run_g4(const uint32_t* idx, const double* av, const double* x, double* out, size_t n, uint32_t ncols,
                   int threads, int ctas_per_sm, int sms) {
  static EncodeFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {4, (cuuint64_t)(ncols + 3) / 4};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {4, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)x, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("{\"variant\": \"gather4\", \"error\": \"encode %d\"}\n", (int)r); return; }
  size_t smem = (size_t)(threads / 32) * S * (128 * 32 + 8);
  auto k = gather4_kernel<S>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = sms * ctas_per_sm;
  size_t n128 = n / 128 * 128;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) k<<<grid, threads, smem>>>(tm, idx, av, out, n128);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("{\"variant\": \"gather4\", \"S\": %d, \"error\": \"%s\"}\n", S, cudaGetErrorString(e)); exit(1); }
  const int reps = 50;
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) k<<<grid, threads, smem>>>(tm, idx, av, out, n128);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  double t = ms * 1e-3 / reps;
  printf("{\"variant\": \"tma_gather4\", \"stages\": %d, \"threads\": %d, \"ctas_per_sm\": %d, \"smem\": %zu, \"us\": %.2f, "
         "\"ggathers_per_s\": %.1f, \"spmv_equiv_gflops\": %.1f}\n",
         S, threads, ctas_per_sm, smem, t * 1e6, n128 / t * 1e-9, 2.0 * n128 / t * 1e-9);
}

int main(int argc, char** argv) {
  size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 41849860ull;
  uint32_t ncols = argc > 2 ? (uint32_t)strtoul(argv[2], 0, 10) : 2000000u;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t* idx;
  double *av, *x, *out;
  CK(cudaMalloc(&idx, n * 4));
  CK(cudaMalloc(&av, n * 8));
  CK(cudaMalloc(&x, (size_t)ncols * 8));
  CK(cudaMalloc(&out, (size_t)sms * 2048 * 8));
  fill_idx<<<sms * 8, 256>>>(idx, av, n, ncols, 42);
  fill_x<<<sms * 8, 256>>>(x, ncols);
  CK(cudaDeviceSynchronize());
  printf("{\"n\": %zu, \"ncols\": %u, \"sms\": %d}\n", n, ncols, sms);
  // warps per SM x gathers in flight per thread
  run<NC, 8>("nc", idx, av, x, out, n, 256, 8, sms);
  run<NC, 8>("nc", idx, av, x, out, n, 256, 6, sms);
  run<NC, 8>("nc", idx, av, x, out, n, 256, 4, sms);
  run<NC, 8>("nc", idx, av, x, out, n, 256, 3, sms);
  run<NC, 16>("nc", idx, av, x, out, n, 256, 3, sms);
  run<NC, 16>("nc", idx, av, x, out, n, 256, 2, sms);
  run<NC, 4>("nc", idx, av, x, out, n, 256, 8, sms);
  run<NC_NOALLOC, 8>("nc_no_allocate", idx, av, x, out, n, 256, 8, sms);
  run<CG, 8>("cg", idx, av, x, out, n, 256, 8, sms);
  run<NO_VALS, 16>("no_vals", idx, av, x, out, n, 256, 8, sms);
  run_g4<2>(idx, av, x, out, n, ncols, 256, 3, sms);
  run_g4<2>(idx, av, x, out, n, ncols, 128, 6, sms);
  run_g4<2>(idx, av, x, out, n, ncols, 64, 12, sms);
  run_g4<1>(idx, av, x, out, n, ncols, 64, 24, sms);
  run_g4<3>(idx, av, x, out, n, ncols, 64, 8, sms);
  return 0;
}
