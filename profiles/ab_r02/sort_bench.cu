// sort_bench.cu — CUB onesweep radix sort of (57-bit uint64 key, uint32 position) pairs, the
// CSF builder's full sort at c5 size (150M nonzeros): the stock sm_100 policy (8-bit digits,
// 8 passes) against policy hubs with wider digits (fewer passes).  Also 32-bit keys of 14/16/18
// bits (the derived trees' root re-sorts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 sort_bench.cu -o sort_bench
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <typename KeyT, typename ValueT, typename OffsetT, int BITS, int THREADS, int ITEMS>
struct Hub {
  using Base = typename cub::detail::radix::policy_hub<KeyT, ValueT, OffsetT>::Policy1000;
  using DominantT = ::cuda::std::_If<(sizeof(ValueT) > sizeof(KeyT)), ValueT, KeyT>;
  struct Policy : cub::ChainedPolicy<1000, Policy, Policy> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = BITS;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, KeyT, BITS>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, BITS>;
    using OnesweepPolicy = cub::AgentRadixSortOnesweepPolicy<
        THREADS, ITEMS, DominantT, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
        cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, BITS>;
    using ScanPolicy = typename Base::ScanPolicy;
    using DownsweepPolicy = typename Base::DownsweepPolicy;
    using AltDownsweepPolicy = typename Base::AltDownsweepPolicy;
    using UpsweepPolicy = typename Base::UpsweepPolicy;
    using AltUpsweepPolicy = typename Base::AltUpsweepPolicy;
    using SingleTilePolicy = typename Base::SingleTilePolicy;
    using SegmentedPolicy = typename Base::SegmentedPolicy;
    using AltSegmentedPolicy = typename Base::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy;
};

template <typename KeyT, typename Hub>
float run(const KeyT* kin, KeyT* kout, const unsigned* vin, unsigned* vout, int n, int bits,
          cudaStream_t s) {
  using Dispatch = cub::DispatchRadixSort<false, KeyT, unsigned, int, Hub>;
  cub::DoubleBuffer<KeyT> dk(const_cast<KeyT*>(kin), kout);
  cub::DoubleBuffer<unsigned> dv(const_cast<unsigned*>(vin), vout);
  size_t tb = 0;
  CK(Dispatch::Dispatch(nullptr, tb, dk, dv, n, 0, bits, false, s));
  void* tmp;
  CK(cudaMalloc(&tmp, tb));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cub::DoubleBuffer<KeyT> k2(const_cast<KeyT*>(kin), kout);
    cub::DoubleBuffer<unsigned> v2(const_cast<unsigned*>(vin), vout);
    cudaEventRecord(a, s);
    CK(Dispatch::Dispatch(tmp, tb, k2, v2, n, 0, bits, false, s));
    cudaEventRecord(b, s);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r) best = std::min(best, ms);
  }
  cudaFree(tmp);
  return best;
}

__global__ void fill(unsigned long long* k, unsigned* v, int n, int bits, unsigned long long seed) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long z = seed + (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    k[i] = bits >= 64 ? z : (z & ((1ull << bits) - 1));
    v[i] = i;
  }
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int n = argc > 1 ? atoi(argv[1]) : 150000000;
  cudaStream_t s;
  cudaStreamCreate(&s);
  unsigned long long *k, *k2;
  unsigned *v, *v2;
  CK(cudaMalloc(&k, (size_t)n * 8));
  CK(cudaMalloc(&k2, (size_t)n * 8));
  CK(cudaMalloc(&v, (size_t)n * 4));
  CK(cudaMalloc(&v2, (size_t)n * 4));
  using U64 = unsigned long long;
  for (int bits : {57, 45}) {
    fill<<<2048, 256, 0, s>>>(k, v, n, bits, 5);
    CK(cudaStreamSynchronize(s));
    printf("u64 keys, %d bits, n=%d\n", bits, n);
    printf("  stock (8-bit digits)      %8.3f ms\n",
           run<U64, cub::detail::radix::policy_hub<U64, unsigned, int>>(k, k2, v, v2, n, bits, s));
    printf("  8b 384x30                 %8.3f ms\n", run<U64, Hub<U64, unsigned, int, 8, 384, 30>>(k, k2, v, v2, n, bits, s));
    printf("  9b 384x24                 %8.3f ms\n", run<U64, Hub<U64, unsigned, int, 9, 384, 24>>(k, k2, v, v2, n, bits, s));
    printf("  10b 256x24                %8.3f ms\n", run<U64, Hub<U64, unsigned, int, 10, 256, 24>>(k, k2, v, v2, n, bits, s));
    printf("  10b 192x30                %8.3f ms\n", run<U64, Hub<U64, unsigned, int, 10, 192, 30>>(k, k2, v, v2, n, bits, s));
  }
  unsigned *k3, *k4;
  CK(cudaMalloc(&k3, (size_t)n * 4));
  CK(cudaMalloc(&k4, (size_t)n * 4));
  for (int bits : {18, 16, 14}) {
    fill<<<2048, 256, 0, s>>>(k, v, n, bits, 7);
    // narrow to 32-bit keys
    CK(cudaMemcpy2DAsync(k3, 4, k, 8, 4, n, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    printf("u32 keys, %d bits\n", bits);
    printf("  stock (8-bit digits)      %8.3f ms\n",
           run<unsigned, cub::detail::radix::policy_hub<unsigned, unsigned, int>>(k3, k4, v, v2, n, bits, s));
    printf("  9b 384x24                 %8.3f ms\n", run<unsigned, Hub<unsigned, unsigned, int, 9, 384, 24>>(k3, k4, v, v2, n, bits, s));
    printf("  10b 256x24                %8.3f ms\n", run<unsigned, Hub<unsigned, unsigned, int, 10, 256, 24>>(k3, k4, v, v2, n, bits, s));
  }
  return 0;
}
