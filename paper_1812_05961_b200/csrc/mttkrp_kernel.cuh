// mttkrp_kernel.cuh — the CSF MTTKRP kernel template for sm_100a, any output level D
// (Alg. 1 lines 5/8/11).
// Included by mttkrp.cu (N = 3), mttkrp_n4.cu (N = 4) and mttkrp_nx.cu (N = 5..8), which
// instantiate it; nothing else includes it.
//
// For CSF levels l = 0..N-1 (mode perm[l] at level l) and output level D:
//
//   M[i, :] = sum over level-D nodes with id i of
//               ( prod_{l < D} A_l[ancestor_l, :] )  (*)  S_D(node)            (elementwise)
//   S_l(node) = sum_{children c} A_{l+1}[c] (*) S_{l+1}(c)   for l < N-2 ... (bottom-up),
//   S_{N-2}(fiber) = sum_{leaves k} v_k A_{N-1}[k, :]
//
// D = 0 is the root ("no-lock") traversal: rows are owned, written with plain stores.
// D = 1..N-2 is the INTERNAL kernel, D = N-1 the LEAF kernel:
// the same output row is reached from many parents, so rows are accumulated into the
// zero-filled output with asynchronous bulk fp64 reductions (one cp.reduce.async.bulk of
// the whole row, executed at L2) — the GPU's answer to the paper's mutex pool.
//
// Design:
//  * Work unit = a fixed chunk of CH consecutive leaves of the CSF, handled by a lane
//    group of G lanes (G = next pow2 of ld/4; each lane owns 4 consecutive columns
//    and moves them with one 256-bit load).  Fixed-size leaf chunks balance the
//    power-law slices (a 13.8M-nonzero slice is just many chunks) — SURVEY.md §8(a')1a.
//  * A group walks its chunk in batches of 32 leaves.  Per batch, lane-parallel: load
//    windows of leaf ids/values (streamed, L1 no-allocate) and of every internal
//    level's ptr, turn them into 32-bit "node closes here" masks (segment flags derived
//    from ptr, §8(a')2), and resolve for every leaf how many levels it closes and, per
//    closed level l, either the id of the closed node (l >= D: bottom-up factor rows and
//    the output row) or the id of the NEXT node (l < D: the top-down prefix product of
//    the ancestors' rows must be rebuilt for the following leaf).  One record per leaf
//    goes to a per-group shared-memory table.
//  * Then the group runs the batch's leaves in order with register accumulators per
//    level: a leaf row is FMA'd into the fiber accumulator; a closing node multiplies
//    its accumulator by its own factor row and pushes it one level up; a closing level-D
//    node emits (prefix (*) accumulator) to its output row.  The rows of U leaves (and of
//    the nodes they close/open) are issued before any is consumed (§8(a')4).
//  * D = 0: slices wholly inside a chunk are written with plain 256-bit stores; the <= 2
//    slices per chunk that cross a chunk seam go through a per-chunk seam row and fp64
//    atomics at the chunk end (no atomics in the leaf loop).
#pragma once
#include <algorithm>

#include "csf.hpp"

namespace sb {
namespace mk {

template <int N>
struct Args {
  const uint32_t* ids[N];
  const uint32_t* ptr[N];     // levels 0..N-2
  const double* fac[N];       // fac[l] = factor of mode perm[l]; fac[D] unused
  uint32_t nodes[N];
  const double* vals;
  double* out;
  const uint32_t* tab;
  double* seam;               // D = 0: nchunks x ld, the chunk's first slice if it began earlier
  uint32_t nnz, nchunks, chunk;
  uint32_t ld;
  int R;
  uint32_t hot[kHotRows];     // D > 0: the output level's most frequent ids (~0u = none)
  int accumulate;             // D = 0: owned rows are added to `out` (later leaf tiles)
  // D = 0, deterministic mode (splatt_ctx_set_deterministic): the chunk-seam rows are not
  // added with atomics but left per chunk (head row in `seam`, tail row in `tail`, their
  // output rows in headrow / tailrow, ~0u = none) for seam_combine_kernel's fixed-order sum.
  int det;
  double* tail;
  uint32_t* headrow;
  uint32_t* tailrow;
  const int* conv;            // ALS converged (splatt_ctx::d_conv): nothing to do
  // Chunk counter for dynamic assignment (zeroed before the launch; a persistent grid of
  // groups takes chunks in order as they finish), nullptr = static (one chunk per group for
  // D = 0, round-robin over a persistent grid for D > 0).
  unsigned* work;
  // Counter value at launch start: a launch takes exactly nchunks + ngroups values (every
  // group's last take overshoots once), so a sequence of launches can share one counter
  // zeroed once (DevCsf::work_seq) instead of a memset per launch.
  unsigned work_base;
};

struct d4 { double x, y, z, w; };

// Factor-row gathers.  Default: L1::no_allocate (+2% on c2/c4/c5 in a B200 A/B: the rows
// stream through L1 without evicting the group tables).  L1A (ROOT kernels whose leaf
// factor exceeds half the L2, e.g. c3's 138 MB mode-0 factor): L1-allocating, so the
// power-law hot rows are served from L1 instead of going back to L2 and DRAM (c3 +7.6%;
// profiles/ab_r01/sweep16.txt).
#ifndef SB_ROW_LOAD
#define SB_ROW_LOAD "ld.global.nc.L1::no_allocate.v4.f64"
#endif
template <bool L1A = false>
__device__ __forceinline__ d4 ldg_row(const double* p) {
  d4 r;
  if constexpr (L1A)
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  else
    asm(SB_ROW_LOAD " {%0,%1,%2,%3}, [%4];"
        : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
// Leaf ids and values: read once per launch.  SB_STREAM_EVICT: with an L2 evict-first cache
// hint, so the stream does not displace factor rows in L2 (A/B: profiles/ab_r02/evict/).
#ifndef SB_STREAM_EVICT
#define SB_STREAM_EVICT 0
#endif
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));  // pure: hoistable
  return pol;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
#if SB_STREAM_EVICT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(l2_evict_first_policy()));
#else
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
#endif
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
#if SB_STREAM_EVICT
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(l2_evict_first_policy()));
#else
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
#endif
  return v;
}
__device__ __forceinline__ void st_row(double* p, const d4& v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z),
               "d"(v.w) : "memory");
}
__device__ __forceinline__ void atomic_row(double* p, const d4& v) {
  atomicAdd(p + 0, v.x);
  atomicAdd(p + 1, v.y);
  atomicAdd(p + 2, v.z);
  atomicAdd(p + 3, v.w);
}
// Columns >= R of the output are written 0 whatever the factors' pad columns hold
// (every column is computed independently, so pads never touch real columns).
__device__ __forceinline__ d4 mask_pad(d4 v, int col, int R) {
  if (col + 0 >= R) v.x = 0.0;
  if (col + 1 >= R) v.y = 0.0;
  if (col + 2 >= R) v.z = 0.0;
  if (col + 3 >= R) v.w = 0.0;
  return v;
}
__device__ __forceinline__ uint32_t lowmask(uint32_t n) {
  return n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
}
template <int G>
__device__ __forceinline__ uint32_t group_or(uint32_t m, unsigned gmask) {
  if constexpr ((G & (G - 1)) == 0) {
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1) m |= __shfl_xor_sync(gmask, m, o, G);
    return m;
  } else {
    return __reduce_or_sync(gmask, m);  // packed groups of G lanes (G not a power of two)
  }
}

// Lane groups: G lanes per group (one 4-column slot of the row per lane), 32 / G groups per
// warp packed side by side.  G need not be a power of two: for R = 33..36 (ld = 36, 9 slots)
// G = 9 packs 3 groups in a warp (27 active lanes) where a power-of-two width would fit 2
// groups of 16 with 7 idle lanes each — 1.5x the rows in flight for the same registers.
template <int G>
struct Lanes {
  static constexpr int kPerWarp = 32 / G;
  static constexpr int kE = (32 + G - 1) / G;  // window entries per lane (32-leaf batches)
  static __host__ __device__ int groups_per_block(int threads) { return threads / 32 * kPerWarp; }
};
__device__ __forceinline__ void fma4(d4& acc, double v, const d4& r) {
  acc.x = fma(v, r.x, acc.x);
  acc.y = fma(v, r.y, acc.y);
  acc.z = fma(v, r.z, acc.z);
  acc.w = fma(v, r.w, acc.w);
}
__device__ __forceinline__ void fma4v(d4& acc, const d4& a, const d4& r) {
  acc.x = fma(a.x, r.x, acc.x);
  acc.y = fma(a.y, r.y, acc.y);
  acc.z = fma(a.z, r.z, acc.z);
  acc.w = fma(a.w, r.w, acc.w);
}
__device__ __forceinline__ d4 mul4(const d4& a, const d4& b) {
  return d4{a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w};
}
__device__ __forceinline__ d4 scale4(double v, const d4& a) {
  return d4{v * a.x, v * a.y, v * a.z, v * a.w};
}

// Per-leaf record written by the lane-parallel phase.  Word 0: leaf row id; word 1:
// closing depth d (levels d..N-2 close at this leaf; N-1 = none) | 0x100 if (D = 0) the
// closing slice is the chunk's first slice and began in an earlier chunk (its row goes
// to the chunk's seam row and is added to the output with atomics at the chunk end);
// word 2 + l (l = 0..N-2, only for closed levels l >= d): l >= D: the closed node's id
// (for D = 0, l = 0: the output row, or the chunk id for a seam slice); l < D: the id of
// the next node at level l (0 past the end).
template <int N>
struct MetaLayout {
  static constexpr int kWords = ((2 + (N - 1)) + 3) / 4 * 4;
  static constexpr int kVec = kWords / 4;
};

constexpr int kBatch = 32;
// Deterministic seams: a long-span entry needs > kLongSpanMin chunks, so at most
// nchunks / kLongSpanMin of them exist (mttkrp.cu's kLongSpan must not be smaller).
constexpr int kLongSpanMin = 64;
constexpr int kBlock = 256;

// Per-group table: records + values, plus 4 words of padding so that the tables of the
// groups sharing a warp start in different 16-byte bank windows (their same-index record
// and value reads are then conflict-free; without the pad, ncu showed half of the shared
// wavefronts to be bank conflicts).
template <int N>
__host__ __device__ constexpr int group_smem_words() {
  return MetaLayout<N>::kWords * kBatch + 2 * kBatch + 4;  // meta + values (doubles) + pad
}

// INTERNAL / LEAF kernels: output rows are added to global memory with bulk reductions
// (cp.reduce.async.bulk .add.f64, SASS UBLKRED): the group stages the row in shared memory
// and one lane hands the whole row (ld doubles) to the async-copy engine, instead of ld
// per-lane fp64 atomics — measured 2.5x the row-update rate on B200.
// Power-law output ids make a few rows receive most of the updates, and updates to one
// address serialise at L2: each group keeps private shared-memory accumulators for the
// kHot most frequent output ids (chosen at CSF build time) and adds them to global memory
// once, when the group finishes.
constexpr int kRedBufs = 4;  // staging rows per lane group (ring)
constexpr int kHot = kHotRows;  // privatised hot output rows per lane group
template <int D>
__host__ __device__ constexpr int group_red_doubles(int ld) {
  // + 2 doubles: the groups of a warp start in different 16-byte bank windows (as the tables)
  return D > 0 ? (kRedBufs + kHot) * ld + 2 : 0;
}

template <int N, int D, int G, int U, int MINB, bool L1A = false>
__global__ void __launch_bounds__(kBlock, MINB) mttkrp_csf_kernel(const Args<N> a) {
  constexpr int E = Lanes<G>::kE;           // window entries per lane
  constexpr int NB = (D < N - 1) ? (N - 2 - D) : 0;  // bottom-up factor levels D+1..N-2
  constexpr int NBA = NB > 0 ? NB : 1;
  constexpr int NP = D;                      // top-down prefix levels 0..D-1
  constexpr int NPA = NP > 0 ? NP : 1;
  constexpr int MV = MetaLayout<N>::kVec;
  constexpr int KW = MetaLayout<N>::kWords;
  extern __shared__ __align__(16) uint32_t smem[];
  if (a.conv && *a.conv) return;
  const int lane = threadIdx.x & 31;
  const int gw = lane / G;                    // group in warp
  if (gw >= Lanes<G>::kPerWarp) return;       // lanes beyond the packed groups: no work
  const int q = lane - gw * G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  const int gpb = Lanes<G>::groups_per_block(blockDim.x);
  const uint32_t gib = (threadIdx.x >> 5) * Lanes<G>::kPerWarp + gw;  // group in block
  uint32_t* gs = smem + gib * group_smem_words<N>();
  uint4* meta = reinterpret_cast<uint4*>(gs);
  double* sval = reinterpret_cast<double*>(gs + KW * kBatch);
  const uint32_t group = blockIdx.x * gpb + gib;
  const uint32_t ngroups = gridDim.x * gpb;
  const bool active = 4u * q < a.ld;
  const uint32_t col = 4u * q;
  // Idle lanes (4q >= ld) re-read column 0..3 so every load is unconditional and valid.
  const uint32_t colc = active ? col : 0u;
  const double* __restrict__ fleaf = a.fac[N - 1] + colc;
  // Row-reduction staging ring of this group (D > 0), after all groups' tables.
  double* rbuf = reinterpret_cast<double*>(smem + gpb * group_smem_words<N>()) +
                 (size_t)gib * group_red_doubles<D>(a.ld);
  uint32_t rslot = 0, rissued = 0;
  double* hacc = rbuf + kRedBufs * a.ld;  // kHot private rows (D > 0)
  if constexpr (D > 0) {
    if (active)
      for (int h = 0; h < kHot; ++h) {
        reinterpret_cast<double2*>(hacc + h * a.ld + col)[0] = make_double2(0.0, 0.0);
        reinterpret_cast<double2*>(hacc + h * a.ld + col)[1] = make_double2(0.0, 0.0);
      }
  }
  // Bulk-reduce one staged row (all lanes of the group call this together).
  auto bulk_row = [&](uint32_t row, const d4& v) {
    if (q == 0 && rissued >= (uint32_t)kRedBufs)
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kRedBufs - 1) : "memory");
    __syncwarp(gmask);
    double* b = rbuf + rslot * a.ld;
    if (active) {
      reinterpret_cast<double2*>(b + col)[0] = make_double2(v.x, v.y);
      reinterpret_cast<double2*>(b + col)[1] = make_double2(v.z, v.w);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp(gmask);
    if (q == 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(b);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                   ::"l"(a.out + (size_t)row * a.ld), "r"(sa), "r"(a.ld * 8) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    rslot = (rslot + 1 == (uint32_t)kRedBufs) ? 0 : rslot + 1;
    ++rissued;
  };
  // out[row, :] += v: privatised if `row` is a hot id (group-uniform branch), else bulk.
  auto emit_row = [&](uint32_t row, const d4& v) {
    int h = -1;
#pragma unroll
    for (int k = 0; k < kHot; ++k) h = (row == a.hot[k]) ? k : h;
    if (h >= 0) {
      if (active) {
        double2* p = reinterpret_cast<double2*>(hacc + h * a.ld + col);
        const double2 p0 = p[0], p1 = p[1];
        p[0] = make_double2(p0.x + v.x, p0.y + v.y);
        p[1] = make_double2(p1.x + v.z, p1.y + v.w);
      }
    } else {
      bulk_row(row, v);
    }
  };

  // Next chunk of this group: dynamic (with a counter: lane 0 of the group takes it, the
  // group shares it) or static round-robin.
  auto next_chunk = [&](uint32_t prev, bool first) -> uint32_t {
    if (a.work == nullptr) return first ? group : prev + ngroups;
    uint32_t v = 0;
    if (q == 0) v = atomicAdd(a.work, 1u) - a.work_base;
    return __shfl_sync(gmask, v, gw * G);
  };
  for (uint32_t c = next_chunk(0, true); c < a.nchunks; c = next_chunk(c, false)) {
    const uint32_t k0 = c * a.chunk;
    const uint32_t k1 = min(k0 + a.chunk, a.nnz);
    uint32_t base[N - 1];
#pragma unroll
    for (int l = 0; l < N - 1; ++l) base[l] = a.tab[(size_t)c * N + l];
    const bool first_partial = (D == 0) && (a.tab[(size_t)c * N + N - 1] & 1u);
    const uint32_t slice0 = base[0];
    d4 acc[N - 1];
#pragma unroll
    for (int l = 0; l < N - 1; ++l) acc[l] = d4{0, 0, 0, 0};
    // Q[l] = prod_{k <= l} A_k[ancestor_k] for the node containing the current leaf.
    d4 Q[NPA];
    if constexpr (NP > 0) {
#pragma unroll
      for (int l = 0; l < NP; ++l) {
        const d4 r = ldg_row<L1A>(a.fac[l] + colc + (size_t)a.ids[l][base[l]] * a.ld);
        Q[l] = (l == 0) ? r : mul4(Q[l > 0 ? l - 1 : 0], r);
      }
    }
    int last_dep = N - 1;

    for (uint32_t kb = k0; kb < k1; kb += kBatch) {
      const uint32_t nb = min((uint32_t)kBatch, k1 - kb);
      // ---- lane-parallel phase: masks, then one record per leaf into shared memory
      uint32_t msk[N - 1];
      {
        uint32_t m = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t idx = base[N - 2] + 1 + q + e * G;
          if (idx <= a.nodes[N - 2]) {
            const uint32_t pos = a.ptr[N - 2][idx] - 1u - kb;
            if (pos < nb) m |= 1u << pos;
          }
        }
        msk[N - 2] = group_or<G>(m, gmask);
      }
#pragma unroll
      for (int l = N - 3; l >= 0; --l) {
        uint32_t m = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t idx = base[l] + 1 + q + e * G;
          if (idx <= a.nodes[l]) {
            const uint32_t pos = a.ptr[l][idx] - 1u - base[l + 1];
            if (pos < 32u) m |= 1u << pos;
          }
        }
        msk[l] = group_or<G>(m, gmask);
      }
      uint32_t cnt[N - 1];
      cnt[N - 2] = __popc(msk[N - 2]);
#pragma unroll
      for (int l = N - 3; l >= 0; --l) cnt[l] = __popc(msk[l] & lowmask(cnt[l + 1]));

      // Record word of a closed level-l node (index `node`).
      auto level_word = [&](int l, uint32_t node) -> uint32_t {
        if (l >= D) return a.ids[l][node];
        return (node + 1u < a.nodes[l]) ? a.ids[l][node + 1u] : 0u;
      };
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t t = q + e * G;
        if (G * E > kBatch && t >= (uint32_t)kBatch) break;
        uint32_t w[KW];
#pragma unroll
        for (int z = 0; z < KW; ++z) w[z] = 0u;
        double v = 0.0;
        uint32_t dep = N - 1;
        if (t < nb) {
          w[0] = ld_stream_u32(a.ids[N - 1] + kb + t);
          v = ld_stream_f64(a.vals + kb + t);
          if ((msk[N - 2] >> t) & 1u) {
            uint32_t li = __popc(msk[N - 2] & lowmask(t));
            uint32_t node = base[N - 2] + li;
            dep = N - 2;
            w[2 + (N - 2)] = level_word(N - 2, node);
#pragma unroll
            for (int l = N - 3; l >= 0; --l) {
              if (dep == (uint32_t)(l + 1) && ((msk[l] >> li) & 1u)) {
                li = __popc(msk[l] & lowmask(li));
                node = base[l] + li;
                dep = l;
                if (D == 0 && l == 0) {
                  if (first_partial && node == slice0) { dep |= 0x100u; w[2] = c; }
                  else w[2] = a.ids[0][node];
                } else {
                  w[2 + l] = level_word(l, node);
                }
              }
            }
          }
        }
        w[1] = dep;
#pragma unroll
        for (int z = 0; z < MV; ++z)
          meta[t * MV + z] = make_uint4(w[4 * z], w[4 * z + 1], w[4 * z + 2], w[4 * z + 3]);
        sval[t] = v;
      }
      __syncwarp(gmask);

      // ---- sequential phase: U leaves at a time, all row loads issued first
      for (uint32_t t0 = 0; t0 < nb; t0 += U) {
        d4 row[U];
        d4 mid[U][NBA];
        d4 nxt[U][NPA];
        uint32_t dep[U], orow[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t t = min(t0 + u, nb - 1);  // clamped: a U not dividing the batch re-reads the last leaf (its FMA is skipped)
          uint32_t w[KW];
#pragma unroll
          for (int z = 0; z < MV; ++z) {
            const uint4 m4 = meta[t * MV + z];
            w[4 * z] = m4.x; w[4 * z + 1] = m4.y; w[4 * z + 2] = m4.z; w[4 * z + 3] = m4.w;
          }
          v[u] = sval[t];
          dep[u] = w[1];
          orow[u] = (D == N - 1) ? w[0] : w[2 + (D < N - 1 ? D : 0)];
          if constexpr (D < N - 1) row[u] = ldg_row<L1A>(fleaf + (size_t)w[0] * a.ld);
          const uint32_t d = w[1] & 0xffu;
#pragma unroll
          for (int l = D + 1; l <= N - 2; ++l)
            if (d <= (uint32_t)l)
              mid[u][l - D - 1] = ldg_row<L1A>(a.fac[l] + colc + (size_t)w[2 + l] * a.ld);
#pragma unroll
          for (int l = 0; l < NP; ++l)
            if (d <= (uint32_t)l) nxt[u][l] = ldg_row<L1A>(a.fac[l] + colc + (size_t)w[2 + l] * a.ld);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (t0 + u < nb) {
            const uint32_t d = dep[u] & 0xffu;
            if constexpr (D < N - 1) {
              fma4(acc[N - 2], v[u], row[u]);
#pragma unroll
              for (int l = N - 2; l >= D + 1; --l) {
                if (d <= (uint32_t)l) {
                  fma4v(acc[l - 1], acc[l], mid[u][l - D - 1]);
                  acc[l] = d4{0, 0, 0, 0};
                }
              }
              if (d <= (uint32_t)D) {
                if constexpr (D == 0) {
                  const bool seam = dep[u] & 0x100u;
                  double* dst = (seam ? a.seam : a.out) + (size_t)orow[u] * a.ld + col;
                  d4 r = mask_pad(acc[0], col, a.R);
                  if (a.accumulate && !seam && active) {  // a later leaf tile: add to the row
                    const d4 o = d4{dst[0], dst[1], dst[2], dst[3]};
                    r = d4{r.x + o.x, r.y + o.y, r.z + o.z, r.w + o.w};
                  }
                  if (active) st_row(dst, r);
                } else {
                  emit_row(orow[u], mask_pad(mul4(acc[D], Q[NP > 0 ? NP - 1 : 0]), col, a.R));
                }
                acc[D] = d4{0, 0, 0, 0};
              }
            } else {  // LEAF kernel: every leaf scatters v * prefix into its own row
              emit_row(orow[u], mask_pad(scale4(v[u], Q[NP > 0 ? NP - 1 : 0]), col, a.R));
            }
            if constexpr (NP > 0) {
              // Levels d..D-1 open new nodes at the next leaf: rebuild their prefixes.
#pragma unroll
              for (int l = 0; l < NP; ++l)
                if (d <= (uint32_t)l) Q[l] = (l == 0) ? nxt[u][0] : mul4(Q[l > 0 ? l - 1 : 0], nxt[u][l]);
            }
          }
        }
      }
      last_dep = (int)(meta[(nb - 1) * MV].y & 0xffu);
      __syncwarp(gmask);
#pragma unroll
      for (int l = 0; l < N - 1; ++l) base[l] += cnt[l];
    }
    if constexpr (D == 0) {
      // Chunk seams: the first slice (if it began earlier) and the still-open levels
      // (< last_dep) of the last slice go out through fp64 atomics.
      const bool head = first_partial && base[0] != slice0;  // the first slice closed here
      if (a.det) {
        if (q == 0) a.headrow[c] = head ? a.ids[0][slice0] : ~0u;
      } else if (head && active) {
        const double* sp = a.seam + (size_t)c * a.ld + col;  // written by this same lane
        const d4 r = d4{sp[0], sp[1], sp[2], sp[3]};
        atomic_row(a.out + (size_t)a.ids[0][slice0] * a.ld + col, r);
      }
      if (a.det && last_dep == 0 && q == 0) a.tailrow[c] = ~0u;
      if (last_dep > 0) {
#pragma unroll
        for (int l = N - 2; l >= 1; --l) {
          if (l < last_dep) {
            const uint32_t nid = a.ids[l][base[l]];
            const d4 r = ldg_row<L1A>(a.fac[l] + colc + (size_t)nid * a.ld);
            fma4v(acc[l - 1], acc[l], r);
          }
        }
        const uint32_t i = a.ids[0][base[0]];
        if (a.det) {
          if (active) st_row(a.tail + (size_t)c * a.ld + col, mask_pad(acc[0], col, a.R));
          if (q == 0) a.tailrow[c] = i;
        } else if (active) {
          atomic_row(a.out + (size_t)i * a.ld + col, mask_pad(acc[0], col, a.R));
        }
      }
    } else if constexpr (D < N - 1) {
      // The level-D node still open at the chunk end (and its open descendants).
      if (last_dep > D) {
#pragma unroll
        for (int l = N - 2; l >= D + 1; --l) {
          if (l < last_dep) {
            const uint32_t nid = a.ids[l][base[l]];
            const d4 r = ldg_row<L1A>(a.fac[l] + colc + (size_t)nid * a.ld);
            fma4v(acc[l - 1], acc[l], r);
          }
        }
        emit_row(a.ids[D][base[D]], mask_pad(mul4(acc[D], Q[NP > 0 ? NP - 1 : 0]), col, a.R));
      }
    }
  }
  if constexpr (D > 0) {
    // flush the privatised hot rows, then wait until every staged row has been read (and
    // reduced) before the shared memory goes away
    for (int h = 0; h < kHot; ++h) {
      if (a.hot[h] == ~0u) continue;
      d4 v{0, 0, 0, 0};
      if (active) {
        const double2* p = reinterpret_cast<const double2*>(hacc + h * a.ld + col);
        v = d4{p[0].x, p[0].y, p[1].x, p[1].y};
      }
      bulk_row(a.hot[h], v);
    }
    if (q == 0 && rissued > 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// acc: bit 0 = add into the output rows (a later leaf tile), bit 1 = L1-allocating gathers
// (D = 0 only).
template <int N, int D, int G, int U, int MINB, bool L1A = false>
void launch_t(splatt_ctx* ctx, DevCsf& c, const double* const* fac_by_mode, double* out,
              int ld, int R, int chunk, int acc) {
  Args<N> a{};
  for (int l = 0; l < N; ++l) {
    a.ids[l] = c.ids[l].p;
    a.ptr[l] = (l < N - 1) ? c.ptr[l].p : nullptr;
    a.fac[l] = (l == D) ? nullptr : fac_by_mode[c.perm[l]];
    a.nodes[l] = (uint32_t)c.nodes[l];
  }
  a.vals = c.vals.p;
  a.out = out;
  a.tab = c.tab.p;
  ArenaScope own(c.arena, false);  // per-tree scratch lives as long as the tree
  if (D == 0) {
    if (c.seam.n < c.nchunks * (size_t)ld) c.seam.alloc(c.nchunks * (size_t)ld, ctx->stream);
    a.seam = c.seam.p;
  }
  a.nnz = (uint32_t)c.nnz;
  a.nchunks = (uint32_t)c.nchunks;
  a.chunk = (uint32_t)chunk;
  a.ld = (uint32_t)ld;
  a.R = R;
  a.accumulate = acc & 1;
  a.conv = ctx->d_conv;
  // The tree's chunk counter for this launch (alloc'd from the tree's allocator): inside a
  // sequence (DevCsf::work_seq, set by cpd_als after zeroing it once) the launch starts at
  // the running base, else the counter is zeroed first.
  auto take_counter = [&](uint64_t ngroups) -> unsigned* {
    if (c.work.n < 1) {
      c.work.alloc(1, ctx->stream);
      SB_CUDA(cudaMemsetAsync(c.work.p, 0, sizeof(unsigned), ctx->stream));
      c.work_base = 0;
    }
    if (!c.work_seq) {
      SB_CUDA(cudaMemsetAsync(c.work.p, 0, sizeof(unsigned), ctx->stream));
      c.work_base = 0;
    }
    a.work_base = c.work_base;
    c.work_base += (unsigned)(c.nchunks + ngroups);
    return c.work.p;
  };
  if (D == 0 && ctx->deterministic) {
    if (c.tail.n < c.nchunks * (size_t)ld) c.tail.alloc(c.nchunks * (size_t)ld, ctx->stream);
    // head rows, tail rows, long-span count (+1 pad word), (c, c0) pairs for long spans
    const size_t words = 2 * c.nchunks + 2 + 4 * ((c.nchunks + kLongSpanMin - 1) / kLongSpanMin + 1);
    if (c.seamrows.n < words) c.seamrows.alloc(words, ctx->stream);
    a.det = 1;
    a.tail = c.tail.p;
    a.headrow = c.seamrows.p;
    a.tailrow = c.seamrows.p + c.nchunks;
  }
  // 256 threads per block unless the per-group tables would exceed 160 KB (many small
  // groups with many levels); the kernel indexes groups by blockDim, not kBlock.
  int threads = kBlock;
  auto smem_for = [&](int thr) {
    return (size_t)Lanes<G>::groups_per_block(thr) *
           (group_smem_words<N>() * 4 + group_red_doubles<D>(ld) * 8);
  };
  while (threads > 64 && smem_for(threads) > 160 * 1024) threads /= 2;
  const int groups_per_block = Lanes<G>::groups_per_block(threads);
  const size_t smem = smem_for(threads);
  set_max_dynamic_smem((const void*)mttkrp_csf_kernel<N, D, G, U, MINB, L1A>, 160 * 1024);
  uint64_t blocks = ceil_div(c.nchunks, groups_per_block);
  static const bool dyn_env = [] {
    const char* e = getenv("SPLATT_DYN");
    return !(e && *e == '0');
  }();
  if (D == 0 && dyn_env && blocks > (uint64_t)ctx->num_sms) {
    // dynamic chunk assignment over a persistent grid: no partial last wave, and a group
    // that drew cheap chunks takes more
    int occ = 0;
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, mttkrp_csf_kernel<N, D, G, U, MINB, L1A>, threads, smem));
    occ = std::max(occ, 1);
    if (blocks > (uint64_t)ctx->num_sms * occ) {
      blocks = (uint64_t)ctx->num_sms * occ;
      a.work = take_counter(blocks * groups_per_block);
    }
  }
  if (D > 0) {
    // persistent grid: each group walks many chunks, so the privatised hot rows are
    // flushed once per group rather than once per chunk
    int occ = 0;  // depends on ld through the staging rows' shared memory
    SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, mttkrp_csf_kernel<N, D, G, U, MINB, L1A>, threads, smem));
    occ = std::max(occ, 1);
    blocks = std::min<uint64_t>(blocks, (uint64_t)ctx->num_sms * occ);
    for (int h = 0; h < kHotRows; ++h) a.hot[h] = c.hot[D][h];
    if (dyn_env)  // chunks taken dynamically here too (the grid is persistent anyway)
      a.work = take_counter(blocks * groups_per_block);
  }
  mttkrp_csf_kernel<N, D, G, U, MINB, L1A>
      <<<(unsigned)std::max<uint64_t>(1, blocks), threads, smem, ctx->stream>>>(a);
  SB_CHECK_LAUNCH(ctx);
}

// Lane-group width by ld (G = next pow2 of ld/4); GSET restricts the instantiated widths
// for the rarely used N >= 5 (a wider group only idles more lanes).
template <int N, int D, int U, int MB, bool ALLG>
void launch_g(splatt_ctx* ctx, DevCsf& c, const double* const* f, double* out, int ld, int R,
              int chunk, int acc) {
  const int slots = ld / 4;
  if constexpr (ALLG) {
    if (slots <= 2) return launch_t<N, D, 2, U, MB>(ctx, c, f, out, ld, R, chunk, acc);
    if (slots <= 4) return launch_t<N, D, 4, U, MB>(ctx, c, f, out, ld, R, chunk, acc);
#ifndef SB_MTTKRP_NO_PACK
    if (D == 0 && (slots == 9 || slots == 10)) {  // ROOT, R = 33..40: 3 packed groups per warp
      if (acc & 2) return launch_t<N, D, 10, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
      return launch_t<N, D, 10, U, MB>(ctx, c, f, out, ld, R, chunk, acc);
    }
#endif
    if (D == 0 && (acc & 2)) {
      if (slots <= 8) return launch_t<N, D, 8, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
      if (slots <= 16) return launch_t<N, D, 16, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
      return launch_t<N, D, 32, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    }
    if (slots <= 16 && slots > 8) return launch_t<N, D, 16, U, MB>(ctx, c, f, out, ld, R, chunk, acc);
  }
  if (slots <= 8) return launch_t<N, D, 8, U, MB>(ctx, c, f, out, ld, R, chunk, acc);
  return launch_t<N, D, 32, U, MB>(ctx, c, f, out, ld, R, chunk, acc);
}

}  // namespace mk

// Per-N entry points (mttkrp.cu / mttkrp_n4.cu / mttkrp_nx.cu): launch the level-D kernel.
void mttkrp_launch_n3(splatt_ctx*, DevCsf&, int D, const double* const*, double*, int, int, int,
                      int acc);
void mttkrp_launch_n4(splatt_ctx*, DevCsf&, int D, const double* const*, double*, int, int, int,
                      int acc);
void mttkrp_launch_nx(splatt_ctx*, DevCsf&, int D, const double* const*, double*, int, int, int,
                      int acc);

}  // namespace sb
