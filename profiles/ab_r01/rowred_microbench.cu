// Microbenchmark: scatter-add of fp64 rows (R = 36) into an output matrix.
//  A: per-lane scalar fp64 atomics (RED.E.ADD.F64), 9 lanes x 4 columns per row
//  B: row staged in shared memory, one lane issues cp.reduce.async.bulk .add.f64 (UBLKRED)
// ids: uniform over I rows, or Zipf-like (heavy rows).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

constexpr int LD = 36;
constexpr int G = 16;

__global__ void scatter_atomic(const uint32_t* ids, int K, double* out) {
  const int lane = threadIdx.x & 31, q = lane & (G - 1);
  const int group = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int ngroups = gridDim.x * blockDim.x / G;
  if (4 * q >= LD) return;
  for (int k = group; k < K; k += ngroups) {
    double* p = out + (size_t)ids[k] * LD + 4 * q;
    double v = 1.0 + k * 1e-9;
    atomicAdd(p + 0, v); atomicAdd(p + 1, v); atomicAdd(p + 2, v); atomicAdd(p + 3, v);
  }
}

constexpr int NBUF = 4;
__global__ void scatter_bulk(const uint32_t* ids, int K, double* out) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, q = lane & (G - 1);
  const int gib = threadIdx.x / G;
  const int group = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int ngroups = gridDim.x * blockDim.x / G;
  double* buf = sm + (size_t)gib * NBUF * LD;
  const unsigned gmask = 0xffffu << (lane & 16);
  int slot = 0, it = 0;
  for (int k = group; k < K; k += ngroups, ++it) {
    if (q == 0 && it >= NBUF) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
    __syncwarp(gmask);
    double* b = buf + slot * LD;
    if (4 * q < LD) {
      double v = 1.0 + k * 1e-9;
      b[4 * q] = v; b[4 * q + 1] = v; b[4 * q + 2] = v; b[4 * q + 3] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp(gmask);
    if (q == 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(b);
      double* p = out + (size_t)ids[k] * LD;
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                   :: "l"(p), "r"(sa), "r"(LD * 8) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    slot = (slot + 1) % NBUF;
  }
  if (q == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int I = 75000, K = 8000000;
  std::mt19937_64 rng(1);
  std::vector<uint32_t> uni(K), zipf(K);
  for (auto& x : uni) x = rng() % I;
  std::vector<double> cdf(I);
  double s = 0;
  for (int i = 0; i < I; ++i) { s += std::pow(i + 1.0, -1.1); cdf[i] = s; }
  std::vector<uint32_t> perm(I);
  for (int i = 0; i < I; ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), rng);
  std::uniform_real_distribution<double> U(0, s);
  for (auto& x : zipf) x = perm[std::upper_bound(cdf.begin(), cdf.end(), U(rng)) - cdf.begin()];
  uint32_t* d_ids;
  double* d_out;
  cudaMalloc(&d_ids, K * 4);
  cudaMalloc(&d_out, (size_t)I * LD * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(scatter_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int dist = 0; dist < 2; ++dist) {
    cudaMemcpy(d_ids, dist ? zipf.data() : uni.data(), K * 4, cudaMemcpyHostToDevice);
    for (int var = 0; var < 2; ++var) {
      for (int bps : {4, 8, 16}) {
        const int threads = 256;
        const int grid = sms * bps;
        const size_t smem = (threads / G) * NBUF * LD * 8;
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemset(d_out, 0, (size_t)I * LD * 8);
          cudaEventRecord(a);
          if (var == 0) scatter_atomic<<<grid, threads>>>(d_ids, K, d_out);
          else scatter_bulk<<<grid, threads, smem>>>(d_ids, K, d_out);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best = std::min(best, ms);
        }
        cudaError_t e = cudaGetLastError();
        std::vector<double> h((size_t)I * LD);
        cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost);
        double tot = 0;
        for (double x : h) tot += x;
        printf("%s %s blocks/SM %2d: %.3f ms  (%.1f G rows/s)  checksum %.6e  %s\n",
               dist ? "zipf" : "unif", var ? "bulk  " : "atomic", bps, best, K / best / 1e6,
               tot, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
