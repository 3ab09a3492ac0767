// onesweep_bench.cu — the library's hand-written onesweep radix sort (csrc/radix_sort.cuh)
// against CUB's DeviceRadixSort::SortPairs on the CSF builder's sorts at c5 size: 150M
// (57-bit packed key, uint32 position) pairs (uniform and Zipf-like coordinates) and 150M
// (18/16-bit uint32 key, position) pairs (the derived trees' root re-sorts).  Checks that both
// produce identical output (both are stable sorts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 onesweep_bench.cu -o osb
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_1812_05961_b200/csrc/radix_sort.cuh"

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

using namespace sb::rs;

template <typename K, int BITS, int T, int IPT, typename V = uint32_t>
struct Sorter {
  using P = Pass<K, V, BITS, T, IPT>;
  static constexpr int B = P::B;
  uint32_t* counts = nullptr;
  int npass = 0, nranges = 0;
  uint32_t tpr = 0;
  int shift[8];
  uint32_t mask[8];
  void setup(uint32_t n, int begin, int end) {
    npass = (end - begin + BITS - 1) / BITS;
    for (int p = 0; p < npass; ++p) {
      shift[p] = begin + p * BITS;
      const int b = std::min(BITS, end - shift[p]);
      mask[p] = (1u << b) - 1u;
    }
    CK(cudaFuncSetAttribute(downsweep_kernel<K, V, BITS, T, IPT>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::kSmem));
    const uint32_t ntiles = (n + P::kTile - 1) / P::kTile;
    const uint32_t C = 148u * (uint32_t)downsweep_ctas_per_sm<K, V, BITS, T, IPT>();
    tpr = (ntiles + C - 1) / C;
    nranges = (int)((ntiles + tpr - 1) / tpr);
    CK(cudaMalloc(&counts, (size_t)nranges * B * 4));
  }
  // returns true when the result is in (k1, v1)
  bool run(K* k0, K* k1, V* v0, V* v1, uint32_t n, cudaStream_t s) {
    K* ki = k0; K* ko = k1; V* vi = v0; V* vo = v1;
    for (int p = 0; p < npass; ++p) {
      upsweep_kernel<K, BITS><<<nranges, 512, 0, s>>>(ki, n, shift[p], mask[p], tpr * P::kTile, counts);
      scan_kernel<BITS><<<1, 1024, 0, s>>>(counts, nranges);
      downsweep_kernel<K, V, BITS, T, IPT><<<nranges, T, P::kSmem, s>>>(ki, ko, vi, vo, n, shift[p],
                                                                      mask[p], tpr, counts);
      std::swap(ki, ko);
      std::swap(vi, vo);
    }
    CK(cudaGetLastError());
    return npass & 1;
  }
};

__device__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// power-law coordinate in [0, I): floor((I+1)^u) - 1, scattered by an odd multiplier
__device__ uint32_t zipfish(uint64_t r, uint32_t I) {
  const double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);
  uint64_t x = (uint64_t)floor(pow((double)I + 1.0, u)) - 1;
  if (x >= I) x = I - 1;
  return (uint32_t)((x * 2654435761ull) % I);
}

__global__ void fill_c5(unsigned long long* k, uint32_t* v, uint32_t n, int zipf, uint64_t seed) {
  const uint32_t dims[4] = {500, 10000, 50000, 200000};  // Q order (ascending)
  const int bits[4] = {9, 14, 16, 18};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long key = 0;
    int sh = 57;
    for (int l = 0; l < 4; ++l) {
      const uint64_t r = mix(seed + (uint64_t)i * 4 + l + 1);
      const uint32_t c = zipf ? zipfish(r, dims[l]) : (uint32_t)(r % dims[l]);
      sh -= bits[l];
      key |= (unsigned long long)c << sh;
    }
    k[i] = key;
    v[i] = i;
  }
}
__global__ void fill_u32(uint32_t* k, uint32_t* v, uint32_t n, uint32_t I, uint64_t seed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    k[i] = zipfish(mix(seed + i), I);
    v[i] = i;
  }
}

template <typename K>
float cub_sort(K* k0, K* k1, uint32_t* v0, uint32_t* v1, uint32_t n, int bits, cudaStream_t s,
               K** outk, uint32_t** outv) {
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, (int)n, 0, bits, s));
  void* tmp;
  CK(cudaMalloc(&tmp, tb));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a, s);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)n, 0, bits, s));
    cudaEventRecord(b, s);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r) best = std::min(best, ms);
  }
  cudaFree(tmp);
  *outk = k1;
  *outv = v1;
  return best;
}

template <typename K, int BITS, int T, int IPT>
void trial(const char* name, K* src_k, uint32_t* src_v, K* k0, K* k1, uint32_t* v0, uint32_t* v1,
           uint32_t n, int bits, const K* ref_k, const uint32_t* ref_v, cudaStream_t s) {
  Sorter<K, BITS, T, IPT> so;
  so.setup(n, 0, bits);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  bool in1 = false;
  for (int r = 0; r < 4; ++r) {
    CK(cudaMemcpyAsync(k0, src_k, (size_t)n * sizeof(K), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(v0, src_v, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
    cudaEventRecord(a, s);
    in1 = so.run(k0, k1, v0, v1, n, s);
    cudaEventRecord(b, s);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r) best = std::min(best, ms);
  }
  K* ok = in1 ? k1 : k0;
  uint32_t* ov = in1 ? v1 : v0;
  std::vector<K> hk(n), rk(n);
  std::vector<uint32_t> hv(n), rv(n);
  CK(cudaMemcpy(hk.data(), ok, (size_t)n * sizeof(K), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(rk.data(), ref_k, (size_t)n * sizeof(K), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hv.data(), ov, (size_t)n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(rv.data(), ref_v, (size_t)n * 4, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (uint32_t i = 0; i < n; ++i) bad += (hk[i] != rk[i]) || (hv[i] != rv[i]);
  printf("  %-28s %8.3f ms  (%d passes, tile %d, smem %zu, %d ranges)  mismatches %zu\n", name, best,
         so.npass, Pass<K, uint32_t, BITS, T, IPT>::kTile, Pass<K, uint32_t, BITS, T, IPT>::kSmem, so.nranges, bad);
  cudaFree(so.counts);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const uint32_t n = argc > 1 ? (uint32_t)atol(argv[1]) : 150000000u;
  cudaStream_t s;
  cudaStreamCreate(&s);
  using U64 = unsigned long long;
  U64 *k, *ka, *kb, *kc;
  uint32_t *v, *va, *vb, *vc;
  CK(cudaMalloc(&k, (size_t)n * 8));
  CK(cudaMalloc(&ka, (size_t)n * 8));
  CK(cudaMalloc(&kb, (size_t)n * 8));
  CK(cudaMalloc(&kc, (size_t)n * 8));
  CK(cudaMalloc(&v, (size_t)n * 4));
  CK(cudaMalloc(&va, (size_t)n * 4));
  CK(cudaMalloc(&vb, (size_t)n * 4));
  CK(cudaMalloc(&vc, (size_t)n * 4));
  for (int zipf : {1}) {
    fill_c5<<<2048, 256, 0, s>>>(k, v, n, zipf, 5);
    CK(cudaStreamSynchronize(s));
    printf("u64 c5-packed keys (57 bits), %s coordinates, n=%u\n", zipf ? "zipf-like" : "uniform", n);
    CK(cudaMemcpy(ka, k, (size_t)n * 8, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(va, v, (size_t)n * 4, cudaMemcpyDeviceToDevice));
    U64* rk;
    uint32_t* rv;
    printf("  %-28s %8.3f ms\n", "cub SortPairs", cub_sort<U64>(ka, kc, va, vc, n, 57, s, &rk, &rv));
    trial<U64, 8, 256, 12>("sort 8b 256x12", k, v, ka, kb, va, vb, n, 57, rk, rv, s);
    trial<U64, 8, 256, 8>("sort 8b 256x8", k, v, ka, kb, va, vb, n, 57, rk, rv, s);
    trial<U64, 8, 256, 10>("sort 8b 256x10", k, v, ka, kb, va, vb, n, 57, rk, rv, s);
    trial<U64, 8, 256, 16>("sort 8b 256x16", k, v, ka, kb, va, vb, n, 57, rk, rv, s);
    {
      // (key, 64-bit value): timing only
      U64 *w0, *w1;
      CK(cudaMalloc(&w0, (size_t)n * 8));
      CK(cudaMalloc(&w1, (size_t)n * 8));
      for (int ipt : {12, 16}) {
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
          CK(cudaMemcpyAsync(ka, k, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          cudaEventRecord(a, s);
          if (ipt == 12) { Sorter<U64, 8, 256, 12, U64> so; so.setup(n, 0, 57); so.run(ka, kb, w0, w1, n, s); }
          else { Sorter<U64, 8, 256, 16, U64> so; so.setup(n, 0, 57); so.run(ka, kb, w0, w1, n, s); }
          cudaEventRecord(b, s);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (r) best = std::min(best, ms);
        }
        printf("  sort 8b 256x%d u64 values     %8.3f ms\n", ipt, best);
      }
      cudaFree(w0);
      cudaFree(w1);
    }
  }
  uint32_t* k32 = reinterpret_cast<uint32_t*>(k);
  uint32_t* k32a = reinterpret_cast<uint32_t*>(ka);
  uint32_t* k32b = reinterpret_cast<uint32_t*>(kb);
  uint32_t* k32c = reinterpret_cast<uint32_t*>(kc);
  for (uint32_t I : {200000u, 50000u}) {
    const int bits = I == 200000u ? 18 : 16;
    fill_u32<<<2048, 256, 0, s>>>(k32, v, n, I, 7);
    CK(cudaStreamSynchronize(s));
    printf("u32 keys, %d bits (zipf-like over %u), n=%u\n", bits, I, n);
    CK(cudaMemcpy(k32a, k32, (size_t)n * 4, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(va, v, (size_t)n * 4, cudaMemcpyDeviceToDevice));
    uint32_t *rk, *rv;
    printf("  %-28s %8.3f ms\n", "cub SortPairs",
           cub_sort<uint32_t>(k32a, k32c, va, vc, n, bits, s, &rk, &rv));
    trial<uint32_t, 8, 512, 16>("sort 8b 512x16", k32, v, k32a, k32b, va, vb, n, bits, rk, rv, s);
    trial<uint32_t, 8, 256, 8>("sort 8b 256x8", k32, v, k32a, k32b, va, vb, n, bits, rk, rv, s);
    trial<uint32_t, 8, 256, 12>("sort 8b 256x12", k32, v, k32a, k32b, va, vb, n, bits, rk, rv, s);
    trial<uint32_t, 8, 256, 16>("sort 8b 256x16", k32, v, k32a, k32b, va, vb, n, bits, rk, rv, s);
    trial<uint32_t, 8, 256, 24>("sort 8b 256x24", k32, v, k32a, k32b, va, vb, n, bits, rk, rv, s);
  }
  return 0;
}
