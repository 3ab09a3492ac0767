// root2.cuh — ROOT ("no-lock") CSF MTTKRP, second generation (
// PAPER.md:182-185, Alg. 1 lines 5/8/11).  Included by root2.cu only.
//
//   M[i, :] = sum over the leaves k below root node i of
//             v_k * A_{N-1}[leaf_k, :] (*) A_{N-2}[fiber_k, :] (*) ... (*) A_1[node1_k, :]
//
// evaluated bottom-up per CSF node exactly as the first-generation kernel
// (mttkrp_kernel.cuh, D = 0), with two changes measured to matter on B200:
//
//  * The per-leaf closing structure is precomputed once per tree (RootPlan, root2.cu):
//    one 16-byte record per leaf {leaf code | d << 29, code of the fiber closing here, v_k},
//    where d is the shallowest level whose node ends at this leaf.  A lane group stages
//    its chunk's records through shared memory with cp.async (double-buffered batches of
//    kB leaves) instead of deriving them from ptr windows, which cost ~2.3 L1TEX
//    wavefronts per leaf in the first kernel (as much as the row gathers themselves on
//    R = 16).
//  * The K most gathered factor rows of the tree (over every non-root level, chosen from a
//    sampled histogram) live in shared memory for the whole launch: a code with bit 28 set
//    is a slot of that table, else a row id.  Power-law tensors send most gathers to a few
//    rows (c5: the top ~1000 of 50k leaf rows take ~70% of the leaf gathers), and L2, not
//    HBM, is what the gathers saturate (~12 TB/s row rate measured by the gather
//    microbenchmark).
//
// Work unit, lane groups, chunk seams and the dynamic chunk counter are those of the first
// kernel: a chunk of consecutive leaves per G-lane group (lane q owns columns 4q..4q+3 and
// moves them with 256-bit loads), slices wholly inside a chunk are written with plain
// stores, the first slice (if it began earlier) and the still-open last slice go out with
// fp64 atomics.  Levels 1..N-3 (N >= 4) keep the factor row of their open node in registers,
// loaded when the previous node closed (its id one node ahead), so no dependent load sits
// on the path of a close.
#pragma once
#include "csf.hpp"

namespace sb {
namespace r2 {

// A row code is a byte offset: bit 28 set -> into the shared-memory row table (slot s at
// s * ld * 8, +16 for odd s: see the prologue), else into the level's factor (id * ld * 8).
// Both must stay below 2^28 bytes (root2_eligible).
constexpr uint32_t kHot = 1u << 28;
constexpr uint32_t kIdMask = kHot - 1u;
constexpr int kDShift = 29;                 // record word 0: closing depth d in bits 29..31
// One CTA per SM.  Threads per CTA by tree order (B200 sweeps, profiles/ab_r02/): N = 4
// keeps three register-held levels and needs ~126 registers (512 threads); N = 3 fits 80
// (768 threads: more rows in flight).
#ifndef SB_ROOT2_THREADS4
#define SB_ROOT2_THREADS4 512
#endif
#ifndef SB_ROOT2_THREADS3
#define SB_ROOT2_THREADS3 768
#endif
template <int N>
struct Threads { static constexpr int k = (N == 3) ? SB_ROOT2_THREADS3 : SB_ROOT2_THREADS4; };
#ifndef SB_ROOT2_B
#define SB_ROOT2_B 48
#endif
constexpr int kBMax = SB_ROOT2_B;           // leaves per staged batch (at most)
#ifndef SB_ROOT2_RECBUDGET_KB
#define SB_ROOT2_RECBUDGET_KB 200
#endif
constexpr int kRecBudget = SB_ROOT2_RECBUDGET_KB * 1024;  // record buffers of all groups (at most)
constexpr int kSmemBudget = 225 * 1024;     // dynamic shared memory per CTA

struct d4 { double x, y, z, w; };

template <int N>
struct Args {
  const uint4* rec;                 // nnz records
  const uint32_t* cid[N];           // level 0: output row ids; 1..N-3: coded ids (+1 pad)
  const uint32_t* ids[N];           // plain node ids (level 0: output rows; N-2: tail fiber)
  const double* fac[N];             // factor at level l (fac[0] unused)
  uint32_t nodes[N];
  double* out;
  const uint32_t* tab;              // chunk table (ensure_chunk_table)
  const uint32_t* hot;              // K entries: (level << 28) | id, ~0u = empty slot
  uint32_t K;
  uint32_t nnz, nchunks, chunk, ld;
  // Guided work units over the chunk table: units 0..nbig-1 take `unit` consecutive table
  // chunks each, the rest one chunk each (the last few percent of the leaves go out in small
  // pieces, so groups finish together); nunits = nbig + nchunks - nbig * unit.
  uint32_t unit, nbig, nunits;
  int R;
  int accumulate;                   // add into the owned rows (later leaf tiles)
  const int* conv;
  unsigned* work;                   // dynamic chunk counter (nullptr: static)
  unsigned work_base;
};

__device__ __forceinline__ d4 ldg_row(const double* p) {
  d4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
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
__device__ __forceinline__ d4 mask_pad(d4 v, int col, int R) {
  if (col + 0 >= R) v.x = 0.0;
  if (col + 1 >= R) v.y = 0.0;
  if (col + 2 >= R) v.z = 0.0;
  if (col + 3 >= R) v.w = 0.0;
  return v;
}
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
__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int P>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(P) : "memory");
}

// Cold-row load: L1::no_allocate (the hot rows are in shared memory).  SB_ROOT2_COLD_LD
// overrides it for A/B runs (e.g. L1-allocating "ld.global.nc.v4.f64").
#ifndef SB_ROOT2_COLD_LD
#define SB_ROOT2_COLD_LD "ld.global.nc.L1::no_allocate.v4.f64"
#endif
// Predicated row gather (no branch, one code path for the whole warp): a hot code reads the
// lane's two 16-byte halves from shared memory (sa0, sa1: 32-bit shared addresses), a cold
// one reads 32 bytes from global memory (gp); `en` = false loads nothing (outputs undefined).
__device__ __forceinline__ d4 gather_pred(bool en, bool hot, uint32_t sa0, uint32_t sa1,
                                          const double* gp) {
  d4 r;
  asm("{\n\t.reg .pred pe, ph, pc;\n\t"
      "setp.ne.b32 pe, %7, 0;\n\t"
      "setp.ne.and.b32 ph, %4, 0, pe;\n\t"
      "setp.eq.and.b32 pc, %4, 0, pe;\n\t"
      "@ph ld.shared.v2.f64 {%0,%1}, [%5];\n\t"
      "@ph ld.shared.v2.f64 {%2,%3}, [%6];\n\t"
      "@pc " SB_ROOT2_COLD_LD " {%0,%1,%2,%3}, [%8];\n\t}"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
      : "r"((uint32_t)hot), "r"(sa0), "r"(sa1), "r"((uint32_t)en), "l"(gp));
  return r;
}
// As gather_pred, always enabled (leaf rows).
__device__ __forceinline__ d4 gather_on(bool hot, uint32_t sa0, uint32_t sa1, const double* gp) {
  d4 r;
  asm("{\n\t.reg .pred ph;\n\t"
      "setp.ne.b32 ph, %4, 0;\n\t"
      "@ph ld.shared.v2.f64 {%0,%1}, [%5];\n\t"
      "@ph ld.shared.v2.f64 {%2,%3}, [%6];\n\t"
      "@!ph " SB_ROOT2_COLD_LD " {%0,%1,%2,%3}, [%7];\n\t}"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
      : "r"((uint32_t)hot), "r"(sa0), "r"(sa1), "l"(gp));
  return r;
}
__device__ __forceinline__ uint4 lds_u4(uint32_t sa) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(sa));
  return r;
}

// Record batches moved by the TMA engine (one cp.async.bulk per batch and group, completion on
// an mbarrier; SB_ROOT2_TMA=1) or by per-lane 16-byte cp.async (0).
#ifndef SB_ROOT2_TMA
#define SB_ROOT2_TMA 1
#endif
#ifndef SB_ROOT2_EVICT
#define SB_ROOT2_EVICT 1  // record batches with an L2 evict-first cache hint (0: without, A/B)
#endif
__device__ __forceinline__ void mbar_init(uint32_t mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
}
__device__ __forceinline__ void bulk_batch(uint32_t dst, const void* src, uint32_t bytes,
                                           uint32_t mb) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic reads
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
               : "memory");
#if SB_ROOT2_EVICT
  // the tree is read once per launch: evict-first in L2, so it does not displace factor rows
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
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W%=;\n\t}" ::"r"(mb), "r"(parity) : "memory");
}

template <int G, int T>
struct Lanes {
  static constexpr int kPerWarp = 32 / G;
  static constexpr int kGroups = T / 32 * kPerWarp;
};

// Shared memory: [hot rows: K x ld doubles][per group: 2 x kB records + 16-byte skew].
// The skew puts the same record index of the groups sharing a warp into different bank
// windows (their broadcast reads then share a wavefront).  kB: the largest batch (48 on
// B200 sweeps, profiles/ab_r02/) whose buffers for every group fit kRecBudget (narrow groups
// are many per CTA).
constexpr int group_rec_bytes(int b) { return 2 * b * 16 + 16; }
template <int G, int T>
__host__ __device__ constexpr int batch_leaves() {
  return Lanes<G, T>::kGroups * group_rec_bytes(kBMax) <= kRecBudget ? kBMax
       : Lanes<G, T>::kGroups * group_rec_bytes(32) <= kRecBudget    ? 32
       : Lanes<G, T>::kGroups * group_rec_bytes(16) <= kRecBudget    ? 16
                                                                      : 8;
}
template <int G, int T>
__host__ __device__ constexpr int rec_smem_bytes() {
  // + two 8-byte mbarriers per group (TMA record batches), after all groups' tables
  return Lanes<G, T>::kGroups * (group_rec_bytes(batch_leaves<G, T>()) + (SB_ROOT2_TMA ? 16 : 0));
}
template <int G, int T>
inline uint32_t hot_capacity(int ld) {
  const long free_b = (long)kSmemBudget - rec_smem_bytes<G, T>();
  return free_b > 0 ? (uint32_t)(free_b / ((long)ld * 8)) : 0u;
}

template <int N, int G, int U>
__global__ void __launch_bounds__(Threads<N>::k, 1) mttkrp_root2_kernel(const Args<N> a) {
  using L = Lanes<G, Threads<N>::k>;
  constexpr int kB = batch_leaves<G, Threads<N>::k>();
  constexpr int kGroupRecBytes = group_rec_bytes(kB);
  extern __shared__ __align__(16) unsigned char smem2[];
  if (a.conv && *a.conv) return;
  double* hotrows = reinterpret_cast<double*>(smem2);
  const uint32_t ld = a.ld;
  // ---- prologue: the hot rows of this launch's factors into shared memory
  {
    const uint32_t slots = ld / 4;
    const uint32_t total = a.K * slots;
    for (uint32_t e = threadIdx.x; e < total; e += blockDim.x) {
      const uint32_t s = e / slots, c4 = e - s * slots;
      const uint32_t h = a.hot[s];
      if (h == ~0u) continue;
      const uint32_t l = h >> 28, id = h & kIdMask;
      const d4 r = ldg_row(a.fac[l] + (size_t)id * ld + 4 * c4);
      // odd slots keep the two 16-byte halves of each 32-byte lane chunk swapped, so that
      // even and odd rows read in one instruction touch complementary bank sets
      double2* dst = reinterpret_cast<double2*>(hotrows + (size_t)s * ld + 4 * c4);
      dst[s & 1] = make_double2(r.x, r.y);
      dst[(s & 1) ^ 1] = make_double2(r.z, r.w);
    }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int gw = lane / G;
  if (gw >= L::kPerWarp) return;  // lanes beyond the packed groups
  const int q = lane - gw * G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  const uint32_t gib = (threadIdx.x >> 5) * L::kPerWarp + gw;
  const uint32_t group = blockIdx.x * L::kGroups + gib;
  const uint32_t ngroups = gridDim.x * L::kGroups;
  unsigned char* recbase = smem2 + (size_t)a.K * ld * 8 + (size_t)gib * kGroupRecBytes;
  uint4* buf0 = reinterpret_cast<uint4*>(recbase);
  const uint32_t rec_sa = (uint32_t)__cvta_generic_to_shared(recbase);
#if SB_ROOT2_TMA
  const uint32_t mbar_sa = (uint32_t)__cvta_generic_to_shared(
      smem2 + (size_t)a.K * ld * 8 + (size_t)L::kGroups * kGroupRecBytes + (size_t)gib * 16);
  if (q == 0) {
    mbar_init(mbar_sa);
    mbar_init(mbar_sa + 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp(gmask);
  uint32_t phase = 0;  // bit w: parity of the next completion of buffer w's mbarrier
#endif
  const bool active = 4u * q < ld;
  const uint32_t col = 4u * q;
  const uint32_t colc = active ? col : 0u;
  // Row gathers: hot codes from the shared-memory table (32-bit shared addresses; the
  // first half of a lane's 32-byte chunk sits at +16 in odd slots, see the prologue), cold
  // ones from global memory; predicated, so the warp runs one path whatever its groups mix.
  const uint32_t hot_sa = (uint32_t)__cvta_generic_to_shared(hotrows) + 8u * colc;
  // this lane's column chunk of every gathered level's factor (loop-invariant bases)
  const char* facb[N];
#pragma unroll
  for (int l = 1; l < N; ++l) facb[l] = reinterpret_cast<const char*>(a.fac[l] + colc);
  auto gather_en = [&](int l, uint32_t code, bool en) -> d4 {
    const uint32_t x = code & kIdMask;
    const uint32_t sa0 = hot_sa + x;
    return gather_pred(en, (code & kHot) != 0u, sa0, sa0 ^ 16u,
                       reinterpret_cast<const double*>(facb[l] + x));
  };
  auto gather = [&](int l, uint32_t code) -> d4 {
    const uint32_t x = code & kIdMask;
    const uint32_t sa0 = hot_sa + x;
    return gather_on((code & kHot) != 0u, sa0, sa0 ^ 16u,
                     reinterpret_cast<const double*>(facb[l] + x));
  };
  auto next_chunk = [&](uint32_t prev, bool first) -> uint32_t {
    if (a.work == nullptr) return first ? group : prev + ngroups;
    uint32_t v = 0;
    if (q == 0) v = atomicAdd(a.work, 1u) - a.work_base;
    return __shfl_sync(gmask, v, gw * G);
  };
  auto issue_batch = [&](uint32_t kb, uint32_t nb, int which) {
#if SB_ROOT2_TMA
    if (q == 0) bulk_batch(rec_sa + (uint32_t)which * (kB * 16u), a.rec + kb, nb * 16u,
                           mbar_sa + 8u * (uint32_t)which);
#else
    uint4* dst = buf0 + which * kB;
    for (uint32_t j = q; j < nb; j += G) cp_async16(dst + j, a.rec + kb + j);
    cp_async_commit();
#endif
  };

  constexpr int NM = (N > 3) ? (N - 3) : 1;  // levels 1..N-3 with a register-held open row
  for (uint32_t u = next_chunk(0, true); u < a.nunits; u = next_chunk(u, false)) {
    const uint32_t c = u < a.nbig ? u * a.unit : a.nbig * a.unit + (u - a.nbig);
    const uint32_t cn = u < a.nbig ? a.unit : 1u;
    const uint32_t k0 = c * a.chunk;
    const uint32_t k1 = min(k0 + cn * a.chunk, a.nnz);
    uint32_t base[N - 1];
#pragma unroll
    for (int l = 0; l < N - 1; ++l) base[l] = a.tab[(size_t)c * N + l];
    bool head = (a.tab[(size_t)c * N + N - 1] & 1u) != 0;  // first slice began earlier
    // (cid[0] = the output row ids, cid[1..N-3] coded ids; each padded by one entry, so the
    // one-ahead loads need no bounds test)
    uint32_t rid = a.cid[0][base[0]];
    uint32_t nrid = a.cid[0][base[0] + 1];
    d4 mrow[NM];
    uint32_t nid[NM];
#pragma unroll
    for (int l = 1; l <= N - 3; ++l) {
      mrow[l - 1] = gather(l, a.cid[l][base[l]]);
      nid[l - 1] = a.cid[l][base[l] + 1];
    }
    const uint32_t fib0 = base[N - 2];
    uint32_t nfib = 0;
    d4 acc[N - 1];
#pragma unroll
    for (int l = 0; l < N - 1; ++l) acc[l] = d4{0, 0, 0, 0};
    uint32_t last_d = N - 1;

    issue_batch(k0, min((uint32_t)kB, k1 - k0), 0);
    int which = 0;
    for (uint32_t kb = k0; kb < k1; kb += kB, which ^= 1) {
      const uint32_t nb = min((uint32_t)kB, k1 - kb);
#if SB_ROOT2_TMA
      if (kb + kB < k1) issue_batch(kb + kB, min((uint32_t)kB, k1 - kb - kB), which ^ 1);
      mbar_wait(mbar_sa + 8u * (uint32_t)which, (phase >> which) & 1u);
      phase ^= 1u << which;
#else
      if (kb + kB < k1) {
        issue_batch(kb + kB, min((uint32_t)kB, k1 - kb - kB), which ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp(gmask);
#endif
      const uint32_t rb_sa = rec_sa + (uint32_t)which * (kB * 16u);
      // One leaf: its record (shared memory) and gathered rows.  Past the batch end the
      // last record is re-read and made inert (v = 0, no close, no gathers).
      struct Leaf { d4 row, frow; uint32_t d; double v; };
      auto fetch = [&](uint32_t t) -> Leaf {
        const bool valid = t < nb;
        const uint4 r = lds_u4(rb_sa + 16u * min(t, nb - 1));
        Leaf f;
        f.d = valid ? (r.x >> kDShift) : (uint32_t)(N - 1);
        f.v = valid ? __hiloint2double((int)r.w, (int)r.z) : 0.0;
        f.row = gather_en(N - 1, r.x & (kHot | kIdMask), valid);
        f.frow = gather_en(N - 2, r.y, f.d <= (uint32_t)(N - 2));
        return f;
      };
      auto consume = [&](const Leaf& f, bool valid) {
        const uint32_t d = f.d;
        if (valid) fma4(acc[N - 2], f.v, f.row);
        if (d <= (uint32_t)(N - 2)) {
          fma4v(acc[N - 3], acc[N - 2], f.frow);
          acc[N - 2] = d4{0, 0, 0, 0};
          ++nfib;
#pragma unroll
          for (int l = N - 3; l >= 1; --l) {
            if (d <= (uint32_t)l) {
              fma4v(acc[l - 1], acc[l], mrow[l - 1]);
              acc[l] = d4{0, 0, 0, 0};
              ++base[l];
              mrow[l - 1] = gather(l, nid[l - 1]);
              nid[l - 1] = ld_u32(a.cid[l] + base[l] + 1);
            }
          }
          if (d == 0) {
            double* dst = a.out + (size_t)rid * ld + col;
            d4 r = mask_pad(acc[0], col, a.R);
            if (active) {
              if (head) {
                atomic_row(dst, r);
              } else {
                if (a.accumulate) {
                  const d4 o = d4{dst[0], dst[1], dst[2], dst[3]};
                  r = d4{r.x + o.x, r.y + o.y, r.z + o.z, r.w + o.w};
                }
                st_row(dst, r);
              }
            }
            head = false;
            acc[0] = d4{0, 0, 0, 0};
            ++base[0];
            rid = nrid;
            nrid = ld_u32(a.cid[0] + base[0] + 1);
          }
        }
        if (valid) last_d = d;
      };
      // Two-stage software pipeline: the rows of the next leaf are in flight while this one
      // is accumulated and its closes are handled (two register sets, no moves).
      Leaf A = fetch(0), B;
      for (uint32_t t = 0; t < nb; t += 2) {
        B = fetch(t + 1);
        consume(A, true);
        A = fetch(t + 2);
        consume(B, t + 1 < nb);
      }
      __syncwarp(gmask);  // every lane is done with this buffer before it is refilled
    }
    // ---- chunk end: the still-open nodes of the last slice go out with atomics
    if (last_d > 0) {
      if (last_d > (uint32_t)(N - 2)) {  // open fiber
        const uint32_t fid = a.ids[N - 2][fib0 + nfib];
        const d4 r = ldg_row(a.fac[N - 2] + colc + (size_t)fid * ld);
        fma4v(acc[N - 3], acc[N - 2], r);
      }
#pragma unroll
      for (int l = N - 3; l >= 1; --l)
        if ((uint32_t)l < last_d) fma4v(acc[l - 1], acc[l], mrow[l - 1]);
      if (active) atomic_row(a.out + (size_t)rid * ld + col, mask_pad(acc[0], col, a.R));
    }
  }
}

}  // namespace r2
}  // namespace sb
