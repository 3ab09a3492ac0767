// mttkrp.cu — CSF MTTKRP host entry points and the N = 3 instantiations (SURVEY.md §8(a)
// a6, §8(f) NEXT-1).  The kernel is mttkrp_kernel.cuh.
#include <algorithm>
#include <vector>

#include "mttkrp.hpp"
#include "mttkrp_kernel.cuh"

namespace sb {

#ifndef SB_MTTKRP_U
#define SB_MTTKRP_U 2
#endif
#ifndef SB_MTTKRP_MINB
#define SB_MTTKRP_MINB 3
#endif

void mttkrp_launch_n3(splatt_ctx* ctx, DevCsf& c, int D, const double* const* f, double* out,
                      int ld, int R, int chunk, int acc) {
  constexpr int U = SB_MTTKRP_U, MB = SB_MTTKRP_MINB;
  switch (D) {
    case 0: return mk::launch_g<3, 0, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    case 1: return mk::launch_g<3, 1, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    case 2: return mk::launch_g<3, 2, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    default: fail(SPLATT_ERR_BADINPUT, "level out of range");
  }
}

// Leaves per work unit (measured on B200 with dynamic chunk assignment: N = 3 best at 384
// (c2 +3.8% over 256; 320 and 448+ worse, profiles/ab_r01/chunks_dyn.txt), N = 4 at 1024
// (+1.8% over 512, 1536 -6%); shorter chunks balance better, longer ones amortise the
// per-chunk setup and seam rows).
#ifndef SB_MTTKRP_CHUNK3
#define SB_MTTKRP_CHUNK3 384
#endif
#ifndef SB_MTTKRP_CHUNK3_LONG
#define SB_MTTKRP_CHUNK3_LONG 512
#endif
#ifndef SB_MTTKRP_CHUNK3_NONROOT
#define SB_MTTKRP_CHUNK3_NONROOT 256  // trees also run at non-root levels (ONE: 43.3 vs 46.7 ms at 384)
#endif
#ifndef SB_MTTKRP_CHUNK
#define SB_MTTKRP_CHUNK 1024
#endif

// N = 3: trees with long fibers (>= 4 leaves per level-(N-2) node on average, e.g. c3's
// modes 1/2 at ~8) take longer chunks (512): the per-chunk setup and seam rows are amortised
// over more leaves (c3 +7.8% with static scheduling; c2's ~2.9-leaf fibers lose 12% at 512;
// profiles/ab_r01/sweep18.txt, chunks_dyn.txt).  SPLATT_CHUNK overrides.
#ifndef SB_MTTKRP_LONG_FIBER
#define SB_MTTKRP_LONG_FIBER 4
#endif
int mttkrp_chunk_leaves(const DevCsf& c) {
  if (const char* e = getenv("SPLATT_CHUNK")) {
    const int v = atoi(e);
    if (v >= 32 && v % 32 == 0) return v;
  }
  if (c.N != 3) return SB_MTTKRP_CHUNK;
  if (c.nonroot) return SB_MTTKRP_CHUNK3_NONROOT;
  const uint64_t fibers = std::max<uint64_t>(1, c.nodes[c.N - 2]);
  return c.nnz >= (uint64_t)SB_MTTKRP_LONG_FIBER * fibers ? SB_MTTKRP_CHUNK3_LONG : SB_MTTKRP_CHUNK3;
}

double mttkrp_alg_bytes(const DevCsf& c, int R, int level) {
  // B_alg = CSF index/value bytes + factor-row bytes: 12 B per leaf
  // (id + value), 8 B per internal node (id + ptr), plus 8 R bytes per gathered factor
  // row — one per node of every level except the output level D and the root (root:
  // SURVEY's formula exactly) — and, for D > 0, 8 R bytes per output-row update (one
  // atomic row per level-D node; a root MTTKRP writes each owned row once, not counted).
  const int N = c.N;
  double internal = 0.0;
  for (int l = 0; l < N - 1; ++l) internal += (double)c.nodes[l];
  double rows = 0.0;
  for (int l = 0; l < N; ++l)
    if (l != level && l != 0) rows += (double)c.nodes[l];
  if (level > 0) rows += (double)c.nodes[0] + (double)c.nodes[level];
  return 12.0 * (double)c.nnz + 8.0 * internal + 8.0 * R * rows;
}

double mttkrp_min_bytes(const DevCsf& c, int R, int level, const uint64_t* distinct) {
  // Compulsory traffic of one launch: the tree once (12 B per leaf, 8 B per internal node),
  // every factor row the launch references once (distinct[m] rows of mode m: the root node
  // count of mode m's own tree when one exists, else min(I_m, nodes at its level) — an upper
  // bound), and the output matrix written once (I_D rows).  SURVEY.md §7 hard part 3.
  const int N = c.N;
  double internal = 0.0;
  for (int l = 0; l < N - 1; ++l) internal += (double)c.nodes[l];
  double rows = (double)c.dims[level];
  for (int l = 0; l < N; ++l)
    if (l != level) rows += (double)distinct[c.perm[l]];
  return 12.0 * (double)c.nnz + 8.0 * internal + 8.0 * R * rows;
}

namespace {

__global__ void id_histogram_kernel(const uint32_t* __restrict__ ids, uint64_t n,
                                    uint32_t* __restrict__ cnt) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ids[j]], 1u);
}

// The kHotRows most frequent ids of CSF level `level` (ties -> lower id), once per tree.
void ensure_hot(splatt_ctx* ctx, DevCsf& c, int level) {
  if (c.hot_ready[level]) return;
  const uint64_t I = c.dims[level], n = c.nodes[level];
  DevBuf<uint32_t> cnt(I, ctx->stream);
  SB_CUDA(cudaMemsetAsync(cnt.p, 0, I * 4, ctx->stream));
  const uint64_t blocks = std::min<uint64_t>(ceil_div(n, 256), (uint64_t)ctx->num_sms * 8);
  id_histogram_kernel<<<(unsigned)std::max<uint64_t>(1, blocks), 256, 0, ctx->stream>>>(
      c.ids[level].p, n, cnt.p);
  SB_CHECK_LAUNCH(ctx);
  std::vector<uint32_t> h(I);
  SB_CUDA(cudaMemcpyAsync(h.data(), cnt.p, I * 4, cudaMemcpyDeviceToHost, ctx->stream));
  host_sync(ctx);
  std::vector<uint32_t> idx(I);
  for (uint64_t i = 0; i < I; ++i) idx[i] = (uint32_t)i;
  const size_t k = std::min<size_t>(kHotRows, I);
  std::partial_sort(idx.begin(), idx.begin() + k, idx.end(), [&](uint32_t a, uint32_t b) {
    return h[a] != h[b] ? h[a] > h[b] : a < b;
  });
  for (int j = 0; j < kHotRows; ++j)
    c.hot[level][j] = ((size_t)j < k && h[idx[j]] > 1) ? idx[j] : ~0u;
  c.hot_ready[level] = true;
}

// Deterministic chunk seams: every chunk whose first slice closed in it (head) sums, in a
// fixed order, the tails of the chunks the slice spans and its own head row into the output
// row (the only writer of that row).  One warp per chunk, lanes over columns; the span start
// is found 32 chunks per step (ballot).  Spans longer than kLongSpan chunks (a power-law
// slice can cover thousands) are queued for seam_long_kernel, which splits them over a
// block.  The summation order is a function of the span alone (4 interleaved partial sums
// per lane; 8 contiguous warp ranges for long spans), so the result is bitwise reproducible.
constexpr int kLongSpan = 64;
static_assert(kLongSpan >= mk::kLongSpanMin, "long-span list sized for kLongSpanMin");

__device__ __forceinline__ double sum_tails(const double* __restrict__ tail, uint64_t k0,
                                            uint64_t k1, int ld, int col) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  uint64_t k = k0;
  for (; k + 4 <= k1; k += 4) {
    a0 += tail[k * ld + col];
    a1 += tail[(k + 1) * ld + col];
    a2 += tail[(k + 2) * ld + col];
    a3 += tail[(k + 3) * ld + col];
  }
  for (; k < k1; ++k) a0 += tail[k * ld + col];
  return (a0 + a1) + (a2 + a3);
}

__global__ void seam_combine_kernel(const double* __restrict__ head, const double* __restrict__ tail,
                                    const uint32_t* __restrict__ headrow,
                                    const uint32_t* __restrict__ tailrow, uint64_t nchunks, int ld,
                                    double* __restrict__ out, int accumulate, const int* conv,
                                    uint32_t* __restrict__ longcnt, uint64_t* __restrict__ longlist) {
  if (conv && *conv) return;
  const uint64_t c = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (c >= nchunks) return;
  const uint32_t s = headrow[c];
  if (s == ~0u) return;
  uint64_t c0 = c;
  for (;;) {  // chunks c0-1, c0-2, ... whose open tail is slice s
    const int64_t k = (int64_t)c0 - 1 - lane;
    const unsigned m = __ballot_sync(0xffffffffu, k >= 0 && tailrow[k] == s);
    if (m == 0xffffffffu) { c0 -= 32; continue; }
    c0 -= (uint64_t)(__ffs(~m) - 1);
    break;
  }
  if (c - c0 > (uint64_t)kLongSpan) {
    if (lane == 0) {
      const uint32_t e = atomicAdd(longcnt, 1u);
      longlist[2 * (uint64_t)e] = c;
      longlist[2 * (uint64_t)e + 1] = c0;
    }
    return;
  }
  for (int col = lane; col < ld; col += 32) {
    const double acc = sum_tails(tail, c0, c, ld, col) + head[c * ld + col];
    double* o = out + (size_t)s * ld + col;
    *o = accumulate ? *o + acc : acc;
  }
}

// Long spans: one block (8 warps) per span, warp w sums the w-th of 8 contiguous ranges,
// the partials are added in warp order.
__global__ void __launch_bounds__(256) seam_long_kernel(
    const double* __restrict__ head, const double* __restrict__ tail,
    const uint32_t* __restrict__ headrow, int ld, double* __restrict__ out, int accumulate,
    const int* conv, const uint32_t* __restrict__ longcnt,
    const uint64_t* __restrict__ longlist) {
  if (conv && *conv) return;
  __shared__ double part[8][SPLATT_MAX_RANK];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t n = *longcnt;
  for (uint32_t e = blockIdx.x; e < n; e += gridDim.x) {
    const uint64_t c = longlist[2 * (uint64_t)e], c0 = longlist[2 * (uint64_t)e + 1];
    const uint64_t span = c - c0;
    const uint64_t k0 = c0 + span * w / 8, k1 = c0 + span * (w + 1) / 8;
    for (int col = lane; col < ld; col += 32) part[w][col] = sum_tails(tail, k0, k1, ld, col);
    __syncthreads();
    if (w == 0) {
      const uint32_t s = headrow[c];
      for (int col = lane; col < ld; col += 32) {
        double acc = 0.0;
        for (int v = 0; v < 8; ++v) acc += part[v][col];
        acc += head[c * ld + col];
        double* o = out + (size_t)s * ld + col;
        *o = accumulate ? *o + acc : acc;
      }
    }
    __syncthreads();
  }
}

}  // namespace

// Leaf tiles for a ROOT traversal whose leaf factor does not fit in L2 (NEXT-4), when the
// context enables them (splatt_ctx_set_leaf_tiling): T tiles of at most `leaf_tile_frac` of
// the L2 capacity each.
int leaf_tiles(splatt_ctx* ctx, const DevCsf& c, int ld) {
  const double frac = ctx->leaf_tile_frac;  // auto (< 0) outside an ALS run: off
  if (!(frac > 0.0)) return 1;
  const double leaf_bytes = (double)c.dims[c.N - 1] * ld * 8.0;
  const double budget = frac * (double)(ctx->l2_bytes ? ctx->l2_bytes : (126u << 20));
  if (leaf_bytes <= budget || c.nnz < (1u << 20)) return 1;
  return (int)std::min<double>(8.0, std::ceil(leaf_bytes / budget));
}

// ROOT gather cache policy: SPLATT_L1_ALLOC=0/1 forces it (A/B runs and
// tests), else the caller's request, else the tree's timed choice.
bool l1_allocate(const DevCsf& c, int request) {
  if (const char* e = getenv("SPLATT_L1_ALLOC")) return *e == '1';
  if (request >= 0) return request == 1;
  return c.l1a == 1;
}

void mttkrp_prepare(splatt_ctx* ctx, DevCsf& c, int level, int ld) {
  if (c.nnz == 0) return;
  if (level == 0) {
    const int T = leaf_tiles(ctx, c, ld);
    if (T > 1 && c.tiles.empty()) tile_tree(ctx, c, T);
    for (auto& t : c.tiles) {
      const bool v2 = t->nnz && root2_eligible(ctx, *t, ld);
      ensure_chunk_table(ctx, *t, v2 ? root2_table_chunk() : mttkrp_chunk_leaves(*t));
      if (v2) ensure_root_plan(ctx, *t, ld);
    }
    if (!c.tiles.empty()) return;
  }
  const bool v2 = level == 0 && root2_eligible(ctx, c, ld);
  ensure_chunk_table(ctx, c, v2 ? root2_table_chunk() : mttkrp_chunk_leaves(c));
  if (v2) ensure_root_plan(ctx, c, ld);
  if (level > 0) ensure_hot(ctx, c, level);
}

void mttkrp_level(splatt_ctx* ctx, DevCsf& c, int level, const double* const* fac_by_mode,
                  double* out, uint64_t out_rows, int ld, int R, EventTimer* tm, int cat,
                  int l1a_request) {
  if (ld % 4 != 0) fail(SPLATT_ERR_BADINPUT, "internal: ld must be a multiple of 4");
  if (level < 0 || level >= c.N) fail(SPLATT_ERR_BADINPUT, "internal: level out of range");
  if (tm) tm->gap();  // the zero-fill is not part of the timed kernel
  SB_CUDA(cudaMemsetAsync(out, 0, out_rows * (size_t)ld * sizeof(double), ctx->stream));
  if (c.nnz == 0) return;
  mttkrp_prepare(ctx, c, level, ld);
  const int l1a = (level == 0 && l1_allocate(c, l1a_request)) ? 2 : 0;
  auto launch = [&](DevCsf& t, int accumulate) {
    accumulate |= l1a;
    const int chunk = (int)t.tab_chunk;  // the tree's chunk table (mttkrp_prepare)
    if (level == 0 && t.plan && t.plan->ld == ld && t.plan->ready && root2_eligible(ctx, t, ld)) {
      mttkrp_root2_launch(ctx, t, fac_by_mode, out, ld, R, accumulate & 1);
      return;
    }
    switch (c.N) {
      case 3: mttkrp_launch_n3(ctx, t, level, fac_by_mode, out, ld, R, chunk, accumulate); break;
      case 4: mttkrp_launch_n4(ctx, t, level, fac_by_mode, out, ld, R, chunk, accumulate); break;
      default: mttkrp_launch_nx(ctx, t, level, fac_by_mode, out, ld, R, chunk, accumulate); break;
    }
    if (level == 0 && ctx->deterministic) {
      // seamrows: head rows | tail rows | long-span count | (pad) | long-span (c, c0) pairs
      uint32_t* longcnt = t.seamrows.p + 2 * t.nchunks;
      uint64_t* longlist = reinterpret_cast<uint64_t*>(t.seamrows.p + 2 * t.nchunks + 2);
      SB_CUDA(cudaMemsetAsync(longcnt, 0, sizeof(uint32_t), ctx->stream));
      const unsigned blocks = (unsigned)ceil_div(t.nchunks, 8);
      seam_combine_kernel<<<std::max(1u, blocks), 256, 0, ctx->stream>>>(
          t.seam.p, t.tail.p, t.seamrows.p, t.seamrows.p + t.nchunks, t.nchunks, ld, out,
          accumulate & 1, ctx->d_conv, longcnt, longlist);
      SB_CHECK_LAUNCH(ctx);
      seam_long_kernel<<<(unsigned)ctx->num_sms, 256, 0, ctx->stream>>>(
          t.seam.p, t.tail.p, t.seamrows.p, ld, out, accumulate & 1, ctx->d_conv, longcnt,
          longlist);
      SB_CHECK_LAUNCH(ctx);
    }
  };
  if (tm) tm->begin(cat);
  if (level == 0 && !c.tiles.empty()) {
    for (size_t t = 0; t < c.tiles.size(); ++t) launch(*c.tiles[t], t > 0);
  } else {
    launch(c, 0);
  }
  if (tm) tm->end();
}

}  // namespace sb
