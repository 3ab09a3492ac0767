// mttkrp.cu — root-mode CSF MTTKRP for sm_100a (PAPER.md:182-185,
// Alg. 1 lines 5/8/11; "no-lock" root traversal PAPER.md:469).
//
//   M[i, :] = sum_{slices i} sum_{fibers} ( sum_{leaves} v * A_leaf[k, :] ) (*) A_mid[j, :] ...
//
// Design:
//  * Work unit = a fixed chunk of CH consecutive leaves of the CSF, handled by a lane
//    group of G lanes (G = next pow2 of ld/4; each lane owns 4 consecutive columns
//    and moves them with one 256-bit load).  Fixed-size leaf chunks balance the
//    power-law slices (a 13.8M-nonzero slice is just many chunks) — SURVEY.md §8(a')1a.
//  * A group walks its chunk in batches of 32 leaves.  Per batch, lane-parallel: load
//    windows of leaf ids/values (streamed, L1 no-allocate) and of every internal
//    level's ptr, turn them into 32-bit "node closes here" masks (segment flags derived
//    from ptr, §8(a')2), and resolve for every leaf how many levels it closes and the
//    ids of the closed nodes; the result goes to a per-group shared-memory table.
//  * Then the group runs the batch's leaves in order with register accumulators per
//    level: a leaf row is FMA'd into the fiber accumulator; a closing node multiplies
//    its accumulator by its own factor row and pushes it one level up; a closing slice
//    writes its output row.  The rows of U leaves (and of the nodes they close) are
//    issued before any is consumed (Little's law, §8(a')4).
//  * Slices wholly inside a chunk are written with plain 256-bit stores (conflict-free:
//    rows are owned); the <= 2 slices per chunk that cross a chunk seam are accumulated
//    with fp64 atomics into the zero-filled output (outside the per-leaf loop).
#include <algorithm>

#include "csf.hpp"
#include "mttkrp.hpp"

namespace sb {

namespace {

template <int N>
struct Args {
  const uint32_t* ids[N];
  const uint32_t* ptr[N];     // levels 0..N-2
  const double* fac[N];       // fac[l] = factor of mode perm[l] (l >= 1)
  uint32_t nodes[N];
  const double* vals;
  double* out;
  const uint32_t* tab;
  double* seam;               // nchunks x ld: the chunk's first slice when it began earlier
  uint32_t nnz, nchunks, chunk;
  uint32_t ld;
  int R;
};

struct d4 { double x, y, z, w; };

__device__ __forceinline__ d4 ldg_row(const double* p) {
  d4 r;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
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
#pragma unroll
  for (int o = G / 2; o >= 1; o >>= 1) m |= __shfl_xor_sync(gmask, m, o, G);
  return m;
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

// Per-leaf record written by the lane-parallel phase.  Word 0: leaf factor row id;
// word 1: closing depth d (levels d..N-2 close at this leaf; N-1 = none) | 0x100 if the
// closing slice is the chunk's first slice and began in an earlier chunk (its row goes
// to the chunk's seam row and is added to the output with atomics at the chunk end);
// word 2: output row (if d == 0); words 3..: ids of the closed nodes at levels 1..N-2.
template <int N>
struct MetaLayout {
  static constexpr int kWords = ((3 + (N - 2)) + 3) / 4 * 4;
  static constexpr int kVec = kWords / 4;
};

constexpr int kBatch = 32;
constexpr int kBlock = 256;

template <int N>
__host__ __device__ constexpr int group_smem_words() {
  return MetaLayout<N>::kWords * kBatch + 2 * kBatch;  // meta + values (doubles)
}

// NM = N-2 internal levels below the root that carry factor rows (>= 1 for N >= 3).
template <int N, int G, int U, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) mttkrp_root_kernel(const Args<N> a) {
  constexpr int E = kBatch / G;  // window entries per lane
  constexpr int NM = N - 2;
  constexpr int MV = MetaLayout<N>::kVec;
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x & 31;
  const int q = lane & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const uint32_t gib = threadIdx.x / G;  // group in block
  uint32_t* gs = smem + gib * group_smem_words<N>();
  uint4* meta = reinterpret_cast<uint4*>(gs);
  double* sval = reinterpret_cast<double*>(gs + MetaLayout<N>::kWords * kBatch);
  const uint32_t group = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const uint32_t ngroups = gridDim.x * blockDim.x / G;
  const bool active = 4u * q < a.ld;
  const uint32_t col = 4u * q;
  // Idle lanes (4q >= ld) re-read column 0..3 so every load is unconditional and valid.
  const uint32_t colc = active ? col : 0u;
  const double* __restrict__ fleaf = a.fac[N - 1] + colc;

  for (uint32_t c = group; c < a.nchunks; c += ngroups) {
    const uint32_t k0 = c * a.chunk;
    const uint32_t k1 = min(k0 + a.chunk, a.nnz);
    uint32_t base[N - 1];
#pragma unroll
    for (int l = 0; l < N - 1; ++l) base[l] = a.tab[(size_t)c * N + l];
    const bool first_partial = a.tab[(size_t)c * N + N - 1] & 1u;
    const uint32_t slice0 = base[0];
    d4 acc[N - 1];
#pragma unroll
    for (int l = 0; l < N - 1; ++l) acc[l] = d4{0, 0, 0, 0};
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

#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t t = q + e * G;
        uint32_t w[MetaLayout<N>::kWords];
#pragma unroll
        for (int z = 0; z < MetaLayout<N>::kWords; ++z) w[z] = 0u;
        double v = 0.0;
        uint32_t dep = N - 1;
        if (t < nb) {
          w[0] = ld_stream_u32(a.ids[N - 1] + kb + t);
          v = ld_stream_f64(a.vals + kb + t);
          if ((msk[N - 2] >> t) & 1u) {
            uint32_t li = __popc(msk[N - 2] & lowmask(t));
            uint32_t node = base[N - 2] + li;
            dep = N - 2;
            if (NM >= 1) w[3 + (N - 2) - 1] = a.ids[N - 2][node];
#pragma unroll
            for (int l = N - 3; l >= 0; --l) {
              if (dep == (uint32_t)(l + 1) && ((msk[l] >> li) & 1u)) {
                li = __popc(msk[l] & lowmask(li));
                node = base[l] + li;
                dep = l;
                if (l >= 1) w[3 + l - 1] = a.ids[l][node];
                else {
                  if (first_partial && node == slice0) { dep |= 0x100u; w[2] = c; }
                  else w[2] = a.ids[0][node];
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
        d4 mid[U][NM];
        uint32_t dep[U], orow[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t t = t0 + u;
          uint32_t w[MetaLayout<N>::kWords];
#pragma unroll
          for (int z = 0; z < MV; ++z) {
            const uint4 m4 = meta[t * MV + z];
            w[4 * z] = m4.x; w[4 * z + 1] = m4.y; w[4 * z + 2] = m4.z; w[4 * z + 3] = m4.w;
          }
          v[u] = sval[t];
          dep[u] = w[1];
          orow[u] = w[2];
          row[u] = ldg_row(fleaf + (size_t)w[0] * a.ld);
#pragma unroll
          for (int l = 1; l <= NM; ++l)
            if ((w[1] & 0xffu) <= (uint32_t)l)
              mid[u][l - 1] = ldg_row(a.fac[l] + colc + (size_t)w[3 + l - 1] * a.ld);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (t0 + u < nb) {
            const uint32_t d = dep[u] & 0xffu;
            fma4(acc[N - 2], v[u], row[u]);
#pragma unroll
            for (int l = NM; l >= 1; --l) {
              if (d <= (uint32_t)l) {
                fma4v(acc[l - 1], acc[l], mid[u][l - 1]);
                acc[l] = d4{0, 0, 0, 0};
              }
            }
            if (d == 0) {
              double* dst = (dep[u] & 0x100u) ? a.seam : a.out;
              if (active) st_row(dst + (size_t)orow[u] * a.ld + col, mask_pad(acc[0], col, a.R));
              acc[0] = d4{0, 0, 0, 0};
            }
          }
        }
      }
      last_dep = (int)(meta[(nb - 1) * MV].y & 0xffu);
      __syncwarp(gmask);
#pragma unroll
      for (int l = 0; l < N - 1; ++l) base[l] += cnt[l];
    }
    // Chunk seams: the first slice (if it began earlier) and the still-open levels
    // (< last_dep) of the last slice go out through fp64 atomics.
    if (first_partial && base[0] != slice0 && active) {  // the first slice closed here
      const double* sp = a.seam + (size_t)c * a.ld + col;  // written by this same lane
      const d4 r = d4{sp[0], sp[1], sp[2], sp[3]};
      atomic_row(a.out + (size_t)a.ids[0][slice0] * a.ld + col, r);
    }
    if (last_dep > 0) {
#pragma unroll
      for (int l = NM; l >= 1; --l) {
        if (l < last_dep) {
          const uint32_t nid = a.ids[l][base[l]];
          const d4 r = ldg_row(a.fac[l] + colc + (size_t)nid * a.ld);
          fma4v(acc[l - 1], acc[l], r);
        }
      }
      if (active) {
        const uint32_t i = a.ids[0][base[0]];
        atomic_row(a.out + (size_t)i * a.ld + col, mask_pad(acc[0], col, a.R));
      }
    }
  }
}

template <int N, int G, int U, int MINB>
void launch_t(splatt_ctx* ctx, DevCsf& c, const double* const* fac_by_mode, double* out,
              int ld, int R, int chunk) {
  Args<N> a{};
  for (int l = 0; l < N; ++l) {
    a.ids[l] = c.ids[l].p;
    a.ptr[l] = (l < N - 1) ? c.ptr[l].p : nullptr;
    a.fac[l] = fac_by_mode[c.perm[l]];
    a.nodes[l] = (uint32_t)c.nodes[l];
  }
  a.vals = c.vals.p;
  a.out = out;
  a.tab = c.tab.p;
  if (c.seam.n < c.nchunks * (size_t)ld) c.seam.alloc(c.nchunks * (size_t)ld, ctx->stream);
  a.seam = c.seam.p;
  a.nnz = (uint32_t)c.nnz;
  a.nchunks = (uint32_t)c.nchunks;
  a.chunk = (uint32_t)chunk;
  a.ld = (uint32_t)ld;
  a.R = R;
  // 256 threads per block unless the per-group tables would exceed 160 KB (many small
  // groups with many levels); the kernel indexes groups by blockDim, not kBlock.
  int threads = kBlock;
  while (threads > 64 && (size_t)(threads / G) * group_smem_words<N>() * 4 > 160 * 1024)
    threads /= 2;
  const int groups_per_block = threads / G;
  const size_t smem = (size_t)groups_per_block * group_smem_words<N>() * 4;
  static bool attr = false;
  if (!attr) {
    SB_CUDA(cudaFuncSetAttribute(mttkrp_root_kernel<N, G, U, MINB>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr = true;
  }
  const uint64_t blocks = ceil_div(c.nchunks, groups_per_block);
  mttkrp_root_kernel<N, G, U, MINB>
      <<<(unsigned)std::max<uint64_t>(1, blocks), threads, smem, ctx->stream>>>(a);
  SB_CHECK_LAUNCH(ctx);
}

#ifndef SB_MTTKRP_U
#define SB_MTTKRP_U 4
#endif
#ifndef SB_MTTKRP_MINB
#define SB_MTTKRP_MINB 2
#endif

template <int N>
void launch_n(splatt_ctx* ctx, DevCsf& c, const double* const* f, double* out, int ld,
              int R, int chunk) {
  const int slots = ld / 4;
#ifndef SB_MTTKRP_U4
#define SB_MTTKRP_U4 2
#endif
#ifndef SB_MTTKRP_MINB4
#define SB_MTTKRP_MINB4 2
#endif
  constexpr int U = (N == 3) ? SB_MTTKRP_U : (N == 4 ? SB_MTTKRP_U4 : 2);
  constexpr int MB = (N == 3) ? SB_MTTKRP_MINB : (N == 4 ? SB_MTTKRP_MINB4 : 1);
  if (slots <= 2) launch_t<N, 2, U, MB>(ctx, c, f, out, ld, R, chunk);
  else if (slots <= 4) launch_t<N, 4, U, MB>(ctx, c, f, out, ld, R, chunk);
  else if (slots <= 8) launch_t<N, 8, U, MB>(ctx, c, f, out, ld, R, chunk);
  else if (slots <= 16) launch_t<N, 16, U, MB>(ctx, c, f, out, ld, R, chunk);
  else launch_t<N, 32, U, MB>(ctx, c, f, out, ld, R, chunk);
}

}  // namespace

int mttkrp_chunk_leaves(int N, int ld) {
  (void)N;
  (void)ld;
  return 512;
}

double mttkrp_alg_bytes(const DevCsf& c, int R) {
  // B_alg = CSF index/value bytes + gathered factor-row bytes:
  // 12 B per leaf (id + value), 8 B per internal node (id + ptr) and per slice, plus
  // 8 R bytes per gathered row (one per leaf and one per internal node below the root).
  double nodes_below_root = 0.0;
  for (int l = 1; l < c.N - 1; ++l) nodes_below_root += (double)c.nodes[l];
  const double nnz = (double)c.nnz;
  return 12.0 * nnz + 8.0 * nodes_below_root + 8.0 * (double)c.nodes[0] +
         8.0 * R * (nnz + nodes_below_root);
}

void mttkrp_root(splatt_ctx* ctx, DevCsf& c, const double* const* fac_by_mode, double* out,
                 uint64_t out_rows, int ld, int R, EventTimer* tm, int cat) {
  if (ld % 4 != 0) fail(SPLATT_ERR_BADINPUT, "internal: ld must be a multiple of 4");
  const int chunk = mttkrp_chunk_leaves(c.N, ld);
  ensure_chunk_table(ctx, c, chunk);
  SB_CUDA(cudaMemsetAsync(out, 0, out_rows * (size_t)ld * sizeof(double), ctx->stream));
  if (tm) tm->begin(cat);
  switch (c.N) {
    case 3: launch_n<3>(ctx, c, fac_by_mode, out, ld, R, chunk); break;
    case 4: launch_n<4>(ctx, c, fac_by_mode, out, ld, R, chunk); break;
    case 5: launch_n<5>(ctx, c, fac_by_mode, out, ld, R, chunk); break;
    case 6: launch_n<6>(ctx, c, fac_by_mode, out, ld, R, chunk); break;
    case 7: launch_n<7>(ctx, c, fac_by_mode, out, ld, R, chunk); break;
    case 8: launch_n<8>(ctx, c, fac_by_mode, out, ld, R, chunk); break;
    default: fail(SPLATT_ERR_BADINPUT, "nmodes out of range");
  }
  if (tm) tm->end();
}

}  // namespace sb
