// sort_coo's radix passes (CUB onesweep, 64-bit key + 64-bit value, 16 key
// bits = two 8-bit passes over 449M records at 256^3) under other onesweep
// tile shapes than CUB's sm_100 default for 8-byte keys (384 threads x 24
// items): is there a faster policy for these 16-byte records?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_bin/radix_tune tools/radix_tune.cu
#include <cub/cub.cuh>

#include <cstdio>
#include <vector>

#define CK(x)                                                     \
  do {                                                            \
    cudaError_t err_ = (x);                                       \
    if (err_ != cudaSuccess) {                                    \
      std::printf("%s: %s\n", #x, cudaGetErrorString(err_));      \
      std::exit(1);                                               \
    }                                                             \
  } while (0)

using KeyT = unsigned long long;
static bool kOverwrite = false;  // false: input kept, output in the second buffer (what sort_coo does)

template <typename ValT, typename OffT, int THREADS, int ITEMS>
struct Hub {
  using Base = cub::detail::radix::policy_hub<KeyT, ValT, OffT>;
  using B = typename Base::Policy1000;
  struct Policy : cub::ChainedPolicy<500, Policy, Policy> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = 8;
    using HistogramPolicy = typename B::HistogramPolicy;
    using ExclusiveSumPolicy = typename B::ExclusiveSumPolicy;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, KeyT, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, 8>;
    using ScanPolicy = typename B::ScanPolicy;
    using DownsweepPolicy = typename B::DownsweepPolicy;
    using AltDownsweepPolicy = typename B::AltDownsweepPolicy;
    using UpsweepPolicy = typename B::UpsweepPolicy;
    using AltUpsweepPolicy = typename B::AltUpsweepPolicy;
    using SingleTilePolicy = typename B::SingleTilePolicy;
    using SegmentedPolicy = typename B::SegmentedPolicy;
    using AltSegmentedPolicy = typename B::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy;
};

template <typename ValT>
__global__ void fill_kernel(KeyT* k, ValT* v, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    unsigned long long h = i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    k[i] = ((h % 16777216ull) << 32) | (h >> 40);  // row << 32 | column, rows shuffled
    v[i] = ValT(i);
  }
}

static KeyT *k0, *k1;
static void *v0, *v1;
static void* tmp;
static size_t tmp_bytes = size_t(9) << 30;  // non-overwriting sorts keep their intermediate pass here
static size_t n = 449455096;

template <typename ValT, typename OffT, typename HubT>
float run(const char* name) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cub::DoubleBuffer<KeyT> dk(k0, k1);
    cub::DoubleBuffer<ValT> dv(static_cast<ValT*>(v0), static_cast<ValT*>(v1));
    size_t tb = tmp_bytes;
    CK(cudaEventRecord(a));
    CK((cub::DispatchRadixSort<false, KeyT, ValT, OffT, HubT>::Dispatch(tmp, tb, dk, dv, OffT(n), 40, 56, kOverwrite, 0)));
    CK(cudaEventRecord(b));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (rep && ms < best) best = ms;
  }
  std::printf("%s off%d %-16s %7.3f ms (2 passes + histogram)\n", sizeof(ValT) == 8 ? "f64" : "f32", int(sizeof(OffT)) * 8, name, best);
  return best;
}

template <typename ValT, typename OffT>
void sweep() {
  fill_kernel<ValT><<<148 * 8, 256>>>(k0, static_cast<ValT*>(v0), n);
  CK(cudaDeviceSynchronize());
  run<ValT, OffT, cub::detail::radix::policy_hub<KeyT, ValT, OffT>>("CUB default");
  run<ValT, OffT, Hub<ValT, OffT, 384, 24>>("384 x 24");
  run<ValT, OffT, Hub<ValT, OffT, 384, 22>>("384 x 22");
  run<ValT, OffT, Hub<ValT, OffT, 384, 20>>("384 x 20");
  run<ValT, OffT, Hub<ValT, OffT, 256, 24>>("256 x 24");
  run<ValT, OffT, Hub<ValT, OffT, 256, 28>>("256 x 28");
  run<ValT, OffT, Hub<ValT, OffT, 256, 30>>("256 x 30");
  run<ValT, OffT, Hub<ValT, OffT, 256, 32>>("256 x 32");
  run<ValT, OffT, Hub<ValT, OffT, 512, 16>>("512 x 16");
  run<ValT, OffT, Hub<ValT, OffT, 512, 18>>("512 x 18");
}

int main() {
  CK(cudaMalloc(&k0, n * 8));
  CK(cudaMalloc(&k1, n * 8));
  CK(cudaMalloc(&v0, n * 8));
  CK(cudaMalloc(&v1, n * 8));
  CK(cudaMalloc(&tmp, tmp_bytes));
  kOverwrite = false;
  sweep<double, unsigned int>();
  sweep<double, unsigned long long>();
  sweep<float, unsigned int>();
  sweep<float, unsigned long long>();
  return 0;
}
