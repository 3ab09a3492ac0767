// radix_sort.cuh — stable LSD radix sort of (key, value) pairs for sm_100a, written
// for the CSF builder's sorts (the "Sort" of Table III).
//
// Each digit pass is three kernels over a persistent grid of C CTAs (as many as are resident),
// CTA c owning the contiguous range of tiles [c*tpr, (c+1)*tpr):
//   1. upsweep: CTA c counts the digits of its range (shared-memory counters in kParts copies);
//   2. scan: counts[c][d] becomes the global position of the first pair of digit d in range c
//      (digits in order, ranges in order within a digit);
//   3. downsweep: CTA c walks its tiles in order — the next tile lands in shared memory by the
//      TMA engine while the current one is ranked stably (per warp: rows of 32 consecutive
//      pairs, match.any peers, running per-warp digit counters), reordered by digit in shared
//      memory, and stored digit run by digit run (contiguous, coalesced) at the range's running
//      digit offsets.
// No inter-CTA communication inside a pass (a decoupled look-back, measured first, spent a third
// of the pass waiting on chains of tiles: profiles/ab_r02/README.md); the price is one extra
// read of the keys per pass.  Stable: ranges, tiles, warps, rows and lanes follow the input
// order.  Requires n < 2^31.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sb {
namespace rs {

constexpr int kParts = 8;  // shared-memory counter copies in the upsweep (lane % kParts)

template <typename K, typename V, int BITS, int T, int IPT>
struct Pass {
  static constexpr int B = 1 << BITS;
  static constexpr int W = T / 32;
  static constexpr int kTile = T * IPT;
  // two tile buffers (keys, then values): one being sorted, the next tile landing by TMA
  static constexpr size_t kBuf = (size_t)kTile * (sizeof(K) + sizeof(V));
  static constexpr size_t kSmem = 2 * kBuf + (size_t)W * B * 4 + 3 * (size_t)B * 4 + 16;
  static_assert(B <= T, "one thread per digit");
  static_assert(kTile % 16 == 0, "tiles start 16-byte aligned");
};

// counts[c * B + d] = pairs of digit d among pairs [c * range, (c + 1) * range).
template <typename K, int BITS>
__global__ void __launch_bounds__(512) upsweep_kernel(const K* __restrict__ kin, uint32_t n,
                                                      int shift, uint32_t mask, uint32_t range,
                                                      uint32_t* __restrict__ counts) {
  constexpr int B = 1 << BITS;
  __shared__ uint32_t h[kParts * B];
  for (int i = threadIdx.x; i < kParts * B; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  uint32_t* part = h + (threadIdx.x % kParts) * B;
  const uint32_t lo = blockIdx.x * range;
  const uint32_t hi = (uint32_t)min((uint64_t)n, (uint64_t)lo + range);
  constexpr int U = 4;
  uint32_t j = lo + threadIdx.x;
  for (; j + (U - 1) * blockDim.x < hi; j += U * blockDim.x) {
    K k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) k[u] = kin[j + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < U; ++u) atomicAdd(&part[(uint32_t)(k[u] >> shift) & mask], 1u);
  }
  for (; j < hi; j += blockDim.x) atomicAdd(&part[(uint32_t)(kin[j] >> shift) & mask], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < B; d += blockDim.x) {
    uint32_t c = 0u;
#pragma unroll
    for (int q = 0; q < kParts; ++q) c += h[q * B + d];
    counts[(size_t)blockIdx.x * B + d] = c;
  }
}

// In place: counts[c * B + d] -> sum over digits d' < d of all ranges' counts + sum over ranges
// c' < c of counts[c'][d].  One CTA of 1024 threads: B digits x (1024 / B) slices of ranges.
template <int BITS>
__global__ void __launch_bounds__(1024) scan_kernel(uint32_t* __restrict__ counts, int nranges) {
  constexpr int B = 1 << BITS;
  constexpr int S = 1024 / B;  // range slices per digit
  __shared__ uint32_t part[S][B];
  __shared__ uint32_t dstart[B];
  __shared__ uint32_t ws[32];
  const int d = threadIdx.x % B, s = threadIdx.x / B;
  const int per = (nranges + S - 1) / S;
  const int c0 = min(nranges, s * per), c1 = min(nranges, c0 + per);
  // (eight independent loads in flight per thread: the scan runs between two passes, so its
  // latency is on the sort's critical path)
  constexpr int U = 8;
  uint32_t sum = 0u;
  int c = c0;
  for (; c + U <= c1; c += U) {
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = counts[(size_t)(c + u) * B + d];
#pragma unroll
    for (int u = 0; u < U; ++u) sum += v[u];
  }
  for (; c < c1; ++c) sum += counts[(size_t)c * B + d];
  part[s][d] = sum;
  __syncthreads();
  uint32_t total = 0u, before_slice = 0u;
  for (int q = 0; q < S; ++q) {
    if (q < s) before_slice += part[q][d];
    total += part[q][d];
  }
  // exclusive scan of the digit totals (slice 0's threads are digits 0..B-1 in order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = (s == 0) ? total : 0u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = ws[lane];
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= o) vi += y;
    }
    ws[lane] = vi - v;
  }
  __syncthreads();
  if (s == 0) dstart[d] = incl - total + ws[warp];
  __syncthreads();
  uint32_t run = dstart[d] + before_slice;
  c = c0;
  for (; c + U <= c1; c += U) {
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = counts[(size_t)(c + u) * B + d];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      counts[(size_t)(c + u) * B + d] = run;
      run += v[u];
    }
  }
  for (; c < c1; ++c) {
    const uint32_t v = counts[(size_t)c * B + d];
    counts[(size_t)c * B + d] = run;
    run += v;
  }
}

__device__ __forceinline__ void rs_mbar_init(uint32_t mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
}
__device__ __forceinline__ void rs_mbar_wait(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "RSW%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra RSW%=;\n\t}" ::"r"(mb), "r"(parity) : "memory");
}
// SB_RS_EVICT (A/B, profiles/ab_r02/evict/): the once-read tiles with an L2 evict-first cache
// hint, leaving L2 to the scattered writes of the pass.
#ifndef SB_RS_EVICT
#define SB_RS_EVICT 0
#endif
__device__ __forceinline__ void rs_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
#if SB_RS_EVICT
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(mb), "l"(pol) : "memory");
#else
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(mb) : "memory");
#endif
}

// Issued by one thread: the first (count & ~3) pairs of tile `tile` into buffer `bk` (keys) /
// `bv` (values) by the TMA engine, completing on mbarrier `mb` (bulk copies move multiples of
// 16 bytes; the <= 3 pairs of a ragged end are loaded by the consumer).
template <typename K, typename V, int TILE>
__device__ __forceinline__ void rs_issue_tile(const K* kin, const V* vin, uint32_t n,
                                              uint32_t tile, uint32_t bk, uint32_t bv, uint32_t mb) {
  const uint32_t t0 = tile * (uint32_t)TILE;
  const uint32_t c4 = min((uint32_t)TILE, n - t0) & ~3u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic accesses
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
               "r"(c4 * (uint32_t)(sizeof(K) + sizeof(V))) : "memory");
  if (c4) {
    rs_bulk(bk, kin + t0, c4 * (uint32_t)sizeof(K), mb);
    rs_bulk(bv, vin + t0, c4 * (uint32_t)sizeof(V), mb);
  }
}

// One digit pass: (kin, vin) -> (kout, vout) stably by digit (k >> shift) & mask.  CTA c
// sorts tiles [c * tpr, (c + 1) * tpr) in order, starting from the digit offsets
// base[c * B + .] (scan_kernel).  kin / vin 16-byte aligned.
template <typename K, typename V, int BITS, int T, int IPT>
__global__ void __launch_bounds__(T) downsweep_kernel(const K* __restrict__ kin, K* __restrict__ kout,
                                                      const V* __restrict__ vin,
                                                      V* __restrict__ vout, uint32_t n,
                                                      int shift, uint32_t mask, uint32_t tpr,
                                                      const uint32_t* __restrict__ base) {
  using P = Pass<K, V, BITS, T, IPT>;
  constexpr int B = P::B, W = P::W, TILE = P::kTile;
  extern __shared__ __align__(128) unsigned char rs_smem[];
  uint32_t* whist = reinterpret_cast<uint32_t*>(rs_smem + 2 * P::kBuf);  // W x B
  uint32_t* lstart = whist + W * B;  // B: first position of each digit in the reordered tile
  uint32_t* goff = lstart + B;       // B: global position - tile position of each digit
  uint32_t* run = goff + B;          // B: the range's next global position of each digit
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(run + B);  // two mbarriers
  __shared__ uint32_t s_ws[32];
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const uint32_t first = blockIdx.x * tpr;
  const uint32_t last = min(ntiles, first + tpr);
  if (first >= last) return;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(rs_smem);
  auto issue = [&](uint32_t t, int b) {
    rs_issue_tile<K, V, TILE>(kin, vin, n, t, sbase + b * (uint32_t)P::kBuf,
                           sbase + b * (uint32_t)P::kBuf + (uint32_t)(TILE * sizeof(K)),
                           mbar + 8u * b);
  };
  const int d = threadIdx.x;
  if (threadIdx.x == 0) {
    rs_mbar_init(mbar);
    rs_mbar_init(mbar + 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    issue(first, 0);
  }
  if (d < B) run[d] = base[(size_t)blockIdx.x * B + d];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t parity = 0u;  // bit b: parity of buffer b's next completion
  for (uint32_t tile = first; tile < last; ++tile) {
    const int b = (int)((tile - first) & 1u);
    // the next tile into the other buffer (free: the previous iteration ended with a barrier)
    if (threadIdx.x == 0 && tile + 1 < last) issue(tile + 1, b ^ 1);
    for (int i = threadIdx.x; i < W * B; i += T) whist[i] = 0u;
    const uint32_t t0 = tile * (uint32_t)TILE;
    const uint32_t cnt = min((uint32_t)TILE, n - t0);
    K* sk = reinterpret_cast<K*>(rs_smem + b * P::kBuf);
    V* sv = reinterpret_cast<V*>(rs_smem + b * P::kBuf + (size_t)TILE * sizeof(K));
    rs_mbar_wait(mbar + 8u * b, (parity >> b) & 1u);
    parity ^= 1u << b;
    if (threadIdx.x < (cnt & 3u)) {  // ragged end: the last <= 3 pairs
      const uint32_t e = (cnt & ~3u) + threadIdx.x;
      sk[e] = kin[t0 + e];
      sv[e] = vin[t0 + e];
    }
    __syncthreads();
    // ---- this thread's pairs (rows of 32 consecutive pairs per warp), stable ranks
    const uint32_t wbase = (uint32_t)warp * 32u * IPT;
    K key[IPT];
    V val[IPT];
    uint32_t rank[IPT];
    uint32_t* wh = whist + warp * B;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t e = wbase + (uint32_t)i * 32u + lane;
      const bool valid = e < cnt;
      key[i] = valid ? sk[e] : K(0);
      val[i] = valid ? sv[e] : V(0);
      const uint32_t dg = valid ? ((uint32_t)(key[i] >> shift) & mask) : (uint32_t)B;
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      const uint32_t before = __popc(peers & lt);
      const uint32_t c = valid ? wh[dg] : 0u;
      __syncwarp();
      if (valid && before == 0u) wh[dg] = c + (uint32_t)__popc(peers);
      __syncwarp();
      rank[i] = c + before;
    }
    __syncthreads();
    // ---- per digit: offsets of the warps and the tile's count
    uint32_t total = 0u;
    if (d < B) {
#pragma unroll 4
      for (int w = 0; w < W; ++w) {
        const uint32_t c = whist[w * B + d];
        whist[w * B + d] = total;
        total += c;
      }
    }
    // ---- exclusive scan of the counts over digits: where each digit starts in the tile
    {
      uint32_t incl = total;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_ws[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const uint32_t s0 = lane < W ? s_ws[lane] : 0u;
        uint32_t si = s0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, si, o);
          if (lane >= o) si += y;
        }
        if (lane < W) s_ws[lane] = si - s0;
      }
      __syncthreads();
      if (d < B) {
        const uint32_t ls = incl - total + s_ws[warp];
        lstart[d] = ls;
        goff[d] = run[d] - ls;
        run[d] += total;
      }
    }
    __syncthreads();
    // ---- reorder the tile by digit in place (every pair is in registers)
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t e = wbase + (uint32_t)i * 32u + lane;
      if (e < cnt) {
        const uint32_t dg = (uint32_t)(key[i] >> shift) & mask;
        const uint32_t pos = lstart[dg] + whist[warp * B + dg] + rank[i];
        sk[pos] = key[i];
        sv[pos] = val[i];
      }
    }
    __syncthreads();
    // ---- the tile in digit order: each digit's run is one contiguous store
    for (uint32_t j = threadIdx.x; j < cnt; j += T) {
      const K k = sk[j];
      const uint32_t g = goff[(uint32_t)(k >> shift) & mask] + j;
      kout[g] = k;
      vout[g] = sv[j];
    }
    __syncthreads();  // buffer b, whist, lstart and goff free again
  }
}

// CTAs per SM the downsweep kernel runs with (its grid: that many per SM).
template <typename K, typename V, int BITS, int T, int IPT>
inline int downsweep_ctas_per_sm() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, downsweep_kernel<K, V, BITS, T, IPT>, T,
                                                Pass<K, V, BITS, T, IPT>::kSmem);
  return nb > 0 ? nb : 1;
}

}  // namespace rs
}  // namespace sb
