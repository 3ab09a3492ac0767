// Microbenchmark: leaf-row gather of the ROOT MTTKRP, LDG lane groups vs TMA tile::gather4.
// out[c,:] = sum_{j<32} v[32c+j] * F[idx[32c+j], :], F: I x ld fp64 (ld = 36, R = 35).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o g4 gather4_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int LD = 36;
constexpr int ROWB = LD * 8;  // 288 B

// ---------------------------------------------------------------- A: LDG lane groups
// 9 lanes x 4 doubles per row, 3 groups per warp; each group one chunk of 32 leaves.
template <int U, int LDX = LD, int POL = 0>
__global__ void __launch_bounds__(256, 3) gather_ldg(const double* __restrict__ F,
                                                     const uint32_t* __restrict__ idx,
                                                     const double* __restrict__ val,
                                                     uint64_t nchunks, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane / 9, gl = lane % 9;
  const bool live = lane < 27;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t c0 = warp * 3; c0 < nchunks; c0 += nwarps * 3) {
    const uint64_t c = c0 + g;
    const bool ok = live && c < nchunks;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 1
    for (int j0 = 0; j0 < 32; j0 += U) {
      double4 r[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u;
        const uint32_t id = ok ? __ldg(idx + c * 32 + j) : 0u;
        const double vv = ok ? __ldg(val + c * 32 + j) : 0.0;
        v[u] = vv;
        const double* p = F + (size_t)id * LDX + gl * 4;
        if (ok && POL == 0)
          asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(r[u].x), "=d"(r[u].y), "=d"(r[u].z), "=d"(r[u].w) : "l"(p));
        else if (ok && POL == 1)
          asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(r[u].x), "=d"(r[u].y), "=d"(r[u].z), "=d"(r[u].w) : "l"(p));
        else if (ok && POL == 2)
          asm volatile("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(r[u].x), "=d"(r[u].y), "=d"(r[u].z), "=d"(r[u].w) : "l"(p));
        else
          r[u] = make_double4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a0 += v[u] * r[u].x; a1 += v[u] * r[u].y; a2 += v[u] * r[u].z; a3 += v[u] * r[u].w;
      }
    }
    if (ok) *reinterpret_cast<double4*>(out + c * LD + gl * 4) = make_double4(a0, a1, a2, a3);
  }
}


// ---------------------------------------------------------------- C: flat (position-major)
// A warp gathers B rows at once as one contiguous run of B*36 doubles: element e = 32*VW*k +
// VW*lane (+0..VW-1) belongs to row e/36, column e%36 of the batch.  Every lane owns the fixed
// columns (VW*lane + 32*VW*k) % 36; chunk of 32 leaves = 32/B batches.
template <int VW, int POL>
__global__ void __launch_bounds__(256, 2) gather_flat(const double* __restrict__ F,
                                                      const uint32_t* __restrict__ idx,
                                                      const double* __restrict__ val,
                                                      uint64_t nchunks, double* __restrict__ out) {
  constexpr int B = 8 * VW;            // rows per batch (8 for LDG.64, 16 for LDG.128)
  constexpr int K = B * LD / (32 * VW); // loads per lane per batch = 9
  static_assert(K == 9, "K");
  __shared__ double red[8][LD * 8 + 8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  int rowk[K], colk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int e = 32 * VW * k + VW * lane;
    rowk[k] = e / LD;
    colk[k] = e % LD;
  }
  for (uint64_t c = warp; c < nchunks; c += nwarps) {
    const uint32_t myid = __ldg(idx + c * 32 + lane);
    const double myv = __ldg(val + c * 32 + lane);
    double acc[K][VW];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int q = 0; q < VW; ++q) acc[k][q] = 0.0;
#pragma unroll
    for (int b = 0; b < 32 / B; ++b) {
      double x[K][VW];
      double vv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t id = __shfl_sync(0xffffffffu, myid, b * B + rowk[k]);
        vv[k] = __shfl_sync(0xffffffffu, myv, b * B + rowk[k]);
        const double* p = F + (size_t)id * LD + colk[k];
        if (VW == 1) {
          if (POL == 0)
            asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(x[k][0]) : "l"(p));
          else
            asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(x[k][0]) : "l"(p));
        } else {
          if (POL == 0)
            asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                         : "=d"(x[k][0]), "=d"(x[k][VW - 1]) : "l"(p));
          else
            asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];"
                         : "=d"(x[k][0]), "=d"(x[k][VW - 1]) : "l"(p));
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[k][q] += vv[k] * x[k][q];
    }
    // reduce: position (k, lane) -> column colk[k] (+q); 8*36 slots = B/VW... each column has
    // B*LD/(32*VW*... ) contributors; go through shared memory by (row-in-batch, column)
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int q = 0; q < VW; ++q) red[w][rowk[k] * LD + colk[k] + q] = acc[k][q];
    __syncwarp();
    for (int col = lane; col < LD; col += 32) {
      double s = 0;
#pragma unroll
      for (int r = 0; r < B; ++r) s += red[w][r * LD + col];
      out[c * LD + col] = s;
    }
    __syncwarp();
  }
}


// ---------------------------------------------------------------- A': LDG lane groups, any ld
// lanes per row L = ld / 4 (256-bit per lane), 32 / L groups per warp; L1-allocating loads.
template <int LDX, int U>
__global__ void __launch_bounds__(256, 3) gather_ldg_w(const double* __restrict__ F,
                                                       const uint32_t* __restrict__ idx,
                                                       const double* __restrict__ val,
                                                       uint64_t nchunks, double* __restrict__ out) {
  constexpr int L = LDX / 4, GPW = 32 / L;
  const int lane = threadIdx.x & 31, g = lane / L, gl = lane % L;
  const bool live = g < GPW;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t c0 = warp * GPW; c0 < nchunks; c0 += nwarps * GPW) {
    const uint64_t c = c0 + g;
    const bool ok = live && c < nchunks;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 1
    for (int j0 = 0; j0 < 32; j0 += U) {
      double4 r[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u;
        const uint32_t id = ok ? __ldg(idx + c * 32 + j) : 0u;
        v[u] = ok ? __ldg(val + c * 32 + j) : 0.0;
        const double* p = F + (size_t)id * LDX + gl * 4;
        if (ok)
          asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(r[u].x), "=d"(r[u].y), "=d"(r[u].z), "=d"(r[u].w) : "l"(p));
        else
          r[u] = make_double4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a0 += v[u] * r[u].x; a1 += v[u] * r[u].y; a2 += v[u] * r[u].z; a3 += v[u] * r[u].w;
      }
    }
    if (ok) *reinterpret_cast<double4*>(out + c * LDX + gl * 4) = make_double4(a0, a1, a2, a3);
  }
}


// ---------------------------------------------------------------- A'': leaf records via smem or SHFL
// 9-lane groups, 3 per warp, one 32-leaf chunk per group.  MODE 0: per-leaf id/value read
// back from a per-group shared table (LDS.32 + LDS.64 broadcast); MODE 1: the group's lanes
// hold ids/values in registers (lane gl holds leaves gl + 9 e) and each leaf's pair is
// shuffled from its owner (warp-uniform register choice).
template <int MODE>
__global__ void __launch_bounds__(256, 3) gather_rec(const double* __restrict__ F,
                                                     const uint32_t* __restrict__ idx,
                                                     const double* __restrict__ val,
                                                     uint64_t nchunks, double* __restrict__ out) {
  __shared__ uint32_t sid[8][3][36];
  __shared__ double sv[8][3][36];
  const int lane = threadIdx.x & 31, g = lane / 9, gl = lane % 9, w = threadIdx.x >> 5;
  const bool live = lane < 27;
  const int gs = live ? g : 0;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t c0 = warp * 3; c0 < nchunks; c0 += nwarps * 3) {
    const uint64_t c = c0 + gs;
    const bool ok = live && c < nchunks;
    uint32_t rid[4];
    double rv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = gl + 9 * e;
      const bool in = ok && j < 32;
      rid[e] = in ? __ldg(idx + c * 32 + j) : 0u;
      rv[e] = in ? __ldg(val + c * 32 + j) : 0.0;
      if (MODE == 0 && in) { sid[w][gs][j] = rid[e]; sv[w][gs][j] = rv[e]; }
    }
    __syncwarp();
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 1
    for (int j0 = 0; j0 < 32; j0 += 2) {
      double4 r[2];
      double v[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = j0 + u;
        uint32_t id;
        if (MODE == 0) {
          id = sid[w][gs][j];
          v[u] = sv[w][gs][j];
        } else {
          const int src = gs * 9 + (j % 9), e = j / 9;  // e warp-uniform
          uint32_t x = e == 0 ? rid[0] : e == 1 ? rid[1] : e == 2 ? rid[2] : rid[3];
          double y = e == 0 ? rv[0] : e == 1 ? rv[1] : e == 2 ? rv[2] : rv[3];
          id = __shfl_sync(0xffffffffu, x, src);
          v[u] = __shfl_sync(0xffffffffu, y, src);
        }
        const double* p = F + (size_t)id * LD + gl * 4;
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(r[u].x), "=d"(r[u].y), "=d"(r[u].z), "=d"(r[u].w) : "l"(p));
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        a0 += v[u] * r[u].x; a1 += v[u] * r[u].y; a2 += v[u] * r[u].z; a3 += v[u] * r[u].w;
      }
    }
    if (ok) *reinterpret_cast<double4*>(out + c * LD + gl * 4) = make_double4(a0, a1, a2, a3);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- B: TMA gather4
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                            int col, uint32_t r0, uint32_t r1, uint32_t r2,
                                            uint32_t r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)), "l"(tm), "r"(col),
      "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}

// Each warp: a ring of S stages of 4 rows (1152 B); one chunk = 8 quads.  Lane 0 issues.
template <int S, int WPB>
__global__ void __launch_bounds__(WPB * 32) gather_tma(const __grid_constant__ CUtensorMap tm,
                                                     const uint32_t* __restrict__ idx,
                                                     const double* __restrict__ val,
                                                     uint64_t nchunks, double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* ring = reinterpret_cast<double*>(smem + (size_t)w * (S * 4 * ROWB + 160 * 8));
  double* red = ring + S * 4 * LD;  // 144 doubles (+pad) for the chunk-end reduction
  __shared__ __align__(8) uint64_t bars[WPB][S];
  const uint64_t warp = blockIdx.x * (uint64_t)WPB + w;
  const uint64_t nwarps = (uint64_t)gridDim.x * WPB;
  if (lane < S) mbar_init(&bars[w][lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (warp >= nchunks) return;
  // quad q of the warp's stream (chunk k = q / 8 of this warp) -> stage q % S
  uint64_t cur = warp;                     // chunk being consumed
  uint32_t cid = __ldg(idx + cur * 32 + lane);
  double cv = __ldg(val + cur * 32 + lane);
  uint64_t nxt = cur + nwarps;
  uint32_t nid = nxt < nchunks ? __ldg(idx + nxt * 32 + lane) : 0u;
  // prologue: the first S quads (S <= 8: all from the current chunk; S = 16: two chunks)
  static_assert(S == 8 || S == 16, "S");
  auto issue = [&](int stage, uint32_t idreg, int quad) {
    const uint32_t r0 = __shfl_sync(0xffffffffu, idreg, quad * 4 + 0);
    const uint32_t r1 = __shfl_sync(0xffffffffu, idreg, quad * 4 + 1);
    const uint32_t r2 = __shfl_sync(0xffffffffu, idreg, quad * 4 + 2);
    const uint32_t r3 = __shfl_sync(0xffffffffu, idreg, quad * 4 + 3);
    if (lane == 0) {
      mbar_expect(&bars[w][stage], 4 * ROWB);
      tma_gather4(ring + stage * 4 * LD, &tm, &bars[w][stage], 0, r0, r1, r2, r3);
    }
  };
  for (int q = 0; q < 8; ++q) issue(q, cid, q);
  if (S == 16 && nxt < nchunks)
    for (int q = 0; q < 8; ++q) issue(8 + q, nid, q);
  uint32_t phase = 0;  // parity bits per stage packed: stage s parity = (phase >> s) & 1
  int sbase = 0;       // stage of quad 0 of the current chunk
  while (true) {
    double acc[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int st = sbase + q;
      mbar_wait(&bars[w][st], (phase >> st) & 1);
      phase ^= 1u << st;
      const double* s = ring + st * 4 * LD;
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        const int p = lane + 32 * t;
        const double vv = __shfl_sync(0xffffffffu, cv, q * 4 + (p / 36 < 4 ? p / 36 : 3));
        if (t < 4 || p < 144) acc[t] += vv * s[p];
      }
      __syncwarp();
      // refill this stage with the quad S quads ahead
      if (S == 8) {
        if (nxt < nchunks) issue(st, nid, q);
      } else {
        const uint64_t nn = nxt + nwarps;
        // stage st gets quad q of chunk nn (two chunks ahead)
        if (nn < nchunks) {
          const uint32_t nnid = __ldg(idx + nn * 32 + lane);
          issue(st, nnid, q);
        }
      }
    }
    // reduce the 144 positions to 36 columns: column c = p % 36
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const int p = lane + 32 * t;
      if (p < 144) red[p] = acc[t];
    }
    __syncwarp();
    for (int c = lane; c < LD; c += 32)
      out[cur * LD + c] = red[c] + red[c + 36] + red[c + 72] + red[c + 108];
    __syncwarp();
    // advance
    cur = nxt;
    if (cur >= nchunks) break;
    cid = nid;
    cv = __ldg(val + cur * 32 + lane);
    nxt = cur + nwarps;
    nid = nxt < nchunks ? __ldg(idx + nxt * 32 + lane) : 0u;
    if (S == 16) sbase ^= 8;
  }
}

int main(int argc, char** argv) {
  const uint64_t I = argc > 1 ? strtoull(argv[1], 0, 10) : 75000;
  const uint64_t nnz = argc > 2 ? strtoull(argv[2], 0, 10) : 8000000;
  const double zipf = argc > 3 ? atof(argv[3]) : 0.0;
  const uint64_t nch = nnz / 32;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 rng(1);
  std::vector<double> hF(I * LD);
  for (auto& x : hF) x = (double)(rng() % 1000) / 64.0;
  std::vector<uint32_t> hi(nch * 32);
  std::vector<double> hv(nch * 32);
  std::vector<double> cdf;
  if (zipf > 0) {
    cdf.resize(I);
    double s = 0;
    for (uint64_t i = 0; i < I; ++i) { s += 1.0 / pow((double)(i + 1), zipf); cdf[i] = s; }
    for (auto& x : cdf) x /= s;
  }
  std::uniform_real_distribution<double> U01(0, 1);
  for (uint64_t j = 0; j < nch * 32; ++j) {
    if (zipf > 0) {
      const double u = U01(rng);
      hi[j] = (uint32_t)(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      if (hi[j] >= I) hi[j] = I - 1;
    } else {
      hi[j] = (uint32_t)(rng() % I);
    }
    hv[j] = (double)(rng() % 17) / 16.0;
  }
  double *F, *v, *o1, *o2;
  uint32_t* ix;
  CK(cudaMalloc(&F, I * LD * 8));
  CK(cudaMalloc(&v, nch * 32 * 8));
  CK(cudaMalloc(&ix, nch * 32 * 4));
  CK(cudaMalloc(&o1, nch * LD * 8));
  CK(cudaMalloc(&o2, nch * LD * 8));
  CK(cudaMemcpy(F, hF.data(), I * LD * 8, cudaMemcpyHostToDevice));
  double *F40, *F48;
  CK(cudaMalloc(&F40, I * 40 * 8));
  CK(cudaMalloc(&F48, I * 48 * 8));
  CK(cudaMemcpy2D(F40, 320, F, 288, 288, I, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy2D(F48, 384, F, 288, 288, I, cudaMemcpyDeviceToDevice));
  CK(cudaMemcpy(v, hv.data(), nch * 32 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ix, hi.data(), nch * 32 * 4, cudaMemcpyHostToDevice));

  PFN_cuTensorMapEncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {LD, I};
  cuuint64_t gstr[1] = {ROWB};
  cuuint32_t box[2] = {LD, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, F, gdim, gstr, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }

  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto timeit = [&](auto launch, const char* name, double* o) {
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= reps;
    // check vs host on sampled chunks
    std::vector<double> ho(nch * LD);
    CK(cudaMemcpy(ho.data(), o, nch * LD * 8, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (uint64_t c = 0; c < nch; c += 997) {
      for (int k = 0; k < LD; ++k) {
        double s = 0;
        for (int j = 0; j < 32; ++j) s += hv[c * 32 + j] * hF[(size_t)hi[c * 32 + j] * LD + k];
        maxerr = std::max(maxerr, fabs(s - ho[c * LD + k]));
      }
    }
    printf("%-28s I=%8lu nnz=%lu zipf=%.2f  %.4f ms  %.3e rows/s  %.2f TB/s(row bytes)  err %.2e\n",
           name, (unsigned long)I, (unsigned long)(nch * 32), zipf, ms, nch * 32 / (ms * 1e-3),
           nch * 32 * (double)ROWB / (ms * 1e-3) / 1e12, maxerr);
  };
  if (getenv("RECS")) {
    const int blocks = 3;
    timeit([&] { gather_ldg<2, 36, 1><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "ldg U=2 global ids", o1);
    timeit([&] { gather_rec<0><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "records in smem", o1);
    timeit([&] { gather_rec<1><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "records via shfl", o1);
    return 0;
  }
  if (getenv("WIDTHS")) {
    // row-gather ceiling by row width (ld = 16 / 36 / 64 doubles), L1-allocating, U = 4
    for (int w : {16, 36, 64}) {
      double* Fw;
      CK(cudaMalloc(&Fw, I * w * 8));
      CK(cudaMemset(Fw, 0, I * w * 8));
      double* ow;
      CK(cudaMalloc(&ow, nch * w * 8));
      cudaEvent_t x, y;
      CK(cudaEventCreate(&x));
      CK(cudaEventCreate(&y));
      auto run = [&] {
        if (w == 16) gather_ldg_w<16, 4><<<nsm * 3, 256>>>(Fw, ix, v, nch, ow);
        if (w == 36) gather_ldg_w<36, 4><<<nsm * 3, 256>>>(Fw, ix, v, nch, ow);
        if (w == 64) gather_ldg_w<64, 4><<<nsm * 3, 256>>>(Fw, ix, v, nch, ow);
      };
      run();
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(x));
      for (int i = 0; i < 20; ++i) run();
      CK(cudaEventRecord(y));
      CK(cudaEventSynchronize(y));
      float ms;
      CK(cudaEventElapsedTime(&ms, x, y));
      ms /= 20;
      printf("width ld=%d row_bytes=%d I=%lu zipf=%.2f  %.4f ms  %.3e rows/s\n", w, w * 8,
             (unsigned long)I, zipf, ms, nch * 32 / (ms * 1e-3));
      CK(cudaFree(Fw));
      CK(cudaFree(ow));
    }
    return 0;
  }
  const bool only_ldg = getenv("ONLY_LDG") != nullptr;
  {
    const int blocks = 3;
    timeit([&] { gather_ldg<4><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "ldg U=4 ld36 noalloc", o1);
    timeit([&] { gather_ldg<4, 40><<<nsm * blocks, 256>>>(F40, ix, v, nch, o1); }, "ldg U=4 ld40 noalloc", o1);
    timeit([&] { gather_ldg<4, 48><<<nsm * blocks, 256>>>(F48, ix, v, nch, o1); }, "ldg U=4 ld48 noalloc", o1);
    timeit([&] { gather_ldg<4, 36, 1><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "ldg U=4 ld36 L1alloc", o1);
    timeit([&] { gather_ldg<4, 36, 2><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "ldg U=4 ld36 L1evlast", o1);
    timeit([&] { gather_flat<1, 0><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "flat LDG.64 noalloc", o1);
    timeit([&] { gather_flat<1, 1><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "flat LDG.64 L1alloc", o1);
    timeit([&] { gather_flat<2, 0><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "flat LDG.128 noalloc", o1);
    timeit([&] { gather_flat<2, 1><<<nsm * blocks, 256>>>(F, ix, v, nch, o1); }, "flat LDG.128 L1alloc", o1);
  }
  if (only_ldg) return 0;
  {
    constexpr int S = 8, W = 8;
    const size_t sm = (size_t)W * (S * 4 * ROWB + 160 * 8);
    CK(cudaFuncSetAttribute(gather_tma<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (int bps : {1, 2}) {
      char nm[64];
      snprintf(nm, sizeof nm, "tma S=8 W=8 x%d/SM", bps);
      timeit([&] { gather_tma<S, W><<<nsm * bps, W * 32, sm>>>(tm, ix, v, nch, o2); }, nm, o2);
    }
  }
  {
    constexpr int S = 16, W = 8;
    const size_t sm = (size_t)W * (S * 4 * ROWB + 160 * 8);
    CK(cudaFuncSetAttribute(gather_tma<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    timeit([&] { gather_tma<S, W><<<nsm, W * 32, sm>>>(tm, ix, v, nch, o2); }, "tma S=16 W=8 x1/SM", o2);
  }
  {
    constexpr int S = 8, W = 16;
    const size_t sm = (size_t)W * (S * 4 * ROWB + 160 * 8);
    CK(cudaFuncSetAttribute(gather_tma<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    timeit([&] { gather_tma<S, W><<<nsm, W * 32, sm>>>(tm, ix, v, nch, o2); }, "tma S=8 W=16 x1/SM", o2);
  }
  return 0;
}
