// csf.cu — device COO -> CSF builder.
//
// For CSF_n with level order perm (root n first): the nonzeros are put in the
// lexicographic order of (ind[perm[0]], ..., ind[perm[N-1]]), ties by input position
// (stable), using LSD radix sorts of packed composite keys (one 64-bit pass group when
// the coordinate bits fit, else several stable groups, least significant first).
// Level-l nodes are the maximal runs of equal (perm[0..l]) prefixes: a start flag per
// position, an inclusive scan numbering the nodes, and a scatter of ids/ptr.  All
// integer work, so the result is bit-exact against any correct implementation.
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>

#include "csf.hpp"

namespace sb {

namespace {

struct IndSet {
  const uint32_t* p[SPLATT_MAX_NMODES];
  uint64_t dims[SPLATT_MAX_NMODES];
  int N;
};

__global__ void validate_kernel(IndSet s, uint64_t nnz, int* bad) {
  int local = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    for (int m = 0; m < s.N; ++m) local |= (s.p[m][j] >= s.dims[m]);
  }
  if (__any_sync(0xffffffffu, local) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// Composite key of levels [lo, hi) (level order), most significant = lo: bit fields
// (coordinate << shift[l]), or — `mixed`, one key group only — the mixed-radix number
// sum_l c_l * stride[l] with stride[l] = prod_{m > l} I_m, whose ceil(log2 prod I) bits can
// save a radix pass (c5: 57 -> 56 bits, 8 -> 7 passes).  Both orders are the lexicographic
// order of the coordinates (c_l < I_l).
struct KeySpec {
  const uint32_t* src[SPLATT_MAX_NMODES];  // per level (already in level order)
  int shift[SPLATT_MAX_NMODES];
  uint64_t stride[SPLATT_MAX_NMODES];
  int lo, hi;
  bool mixed;
};

// Mixed-radix digits of a key: c[l] = (k / stride[l]) mod I_l for l = N-1 down to 0, by
// successive division (a double-precision quotient corrected to the exact one; k < 2^63).
struct MixedRadix {
  uint32_t dim[SPLATT_MAX_NMODES];
  double inv[SPLATT_MAX_NMODES];  // 1 / dim
  int N;
};
__device__ __forceinline__ void mixed_decode(const MixedRadix& mr, uint64_t k, uint32_t* c) {
  for (int l = mr.N - 1; l >= 0; --l) {
    const uint64_t d = mr.dim[l];
    if (d == 1) { c[l] = 0; continue; }
    uint64_t q = (uint64_t)((double)k * mr.inv[l]);
    long long r = (long long)(k - q * d);
    while (r < 0) { --q; r += (long long)d; }
    while (r >= (long long)d) { ++q; r -= (long long)d; }
    c[l] = (uint32_t)r;
    k = q;
  }
}

// Also (vbits != nullptr, first group only) the values' bits, carried through the sort.
__global__ void pack_keys_kernel(KeySpec ks, uint64_t nnz, const uint32_t* __restrict__ order,
                                 uint64_t* __restrict__ keys, uint32_t* __restrict__ pos,
                                 const double* __restrict__ vin, uint64_t* __restrict__ vbits) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = order ? order[j] : (uint32_t)j;
    uint64_t k = 0;
    if (ks.mixed) {
      for (int l = ks.lo; l < ks.hi; ++l) k += (uint64_t)ks.src[l][q] * ks.stride[l];
    } else {
      for (int l = ks.lo; l < ks.hi; ++l) k |= (uint64_t)ks.src[l][q] << ks.shift[l];
    }
    keys[j] = k;
    if (vbits) vbits[j] = (uint64_t)__double_as_longlong(vin[j]);
    else if (!order) pos[j] = (uint32_t)j;
  }
}

struct CoordOut {
  const uint32_t* src[SPLATT_MAX_NMODES];
  uint32_t* dst[SPLATT_MAX_NMODES];
  int N;
};

__global__ void gather_kernel(CoordOut co, uint64_t nnz, const uint32_t* __restrict__ P,
                              const double* __restrict__ vin, double* __restrict__ vout) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = P[j];
    for (int l = 0; l < co.N; ++l) co.dst[l][j] = co.src[l][q];
    vout[j] = vin[q];
  }
}

struct BitSet { int b[SPLATT_MAX_NMODES]; };

// coordinate of level l at sorted position j = bits of the sorted composite key.
__global__ void decode_kernel(KeySpec ks, BitSet bs, MixedRadix mr, CoordOut co, uint64_t nnz,
                              const uint64_t* __restrict__ keys, const uint32_t* __restrict__ P,
                              const double* __restrict__ vin, double* __restrict__ vout,
                              double2* __restrict__ kv) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[j];
    if (ks.mixed) {
      uint32_t c[SPLATT_MAX_NMODES];
      mixed_decode(mr, k, c);
      for (int l = 0; l < co.N; ++l) co.dst[l][j] = c[l];
    } else {
      for (int l = 0; l < co.N; ++l) {
        const uint64_t m = bs.b[l] >= 64 ? ~0ull : ((1ull << bs.b[l]) - 1ull);
        co.dst[l][j] = (uint32_t)((k >> ks.shift[l]) & m);
      }
    }
    const double v = P ? vin[P[j]] : vin[j];  // (no P: the values travelled with the keys)
    vout[j] = v;
    if (kv) kv[j] = make_double2(__longlong_as_double((long long)k), v);
  }
}

// node[l][j] = 1 iff a level-l node starts at sorted position j (prefix 0..l changed).
struct FlagOut {
  const uint32_t* c[SPLATT_MAX_NMODES];
  uint32_t* node[SPLATT_MAX_NMODES];
  int N;
};

__device__ __forceinline__ uint32_t plan_code(const RootPlanRecOut& ro, uint64_t off, uint32_t id) {
  // (read-only during the build's level kernels: the non-coherent path lets these loads
  // move ahead of the record stores)
  const uint32_t s = __ldg(ro.slotmap + off + id);  // (root2.cuh's row code: byte offset, bit 28 = hot)
  return s != ~0u ? ((1u << 28) | (s * ro.ldb + ((s & 1u) << 4))) : id * ro.ldb;
}

// Also, with a ROOT plan under construction (ro.rec), leaf j's record: d = the first level
// whose coordinate differs from leaf j+1 (the shallowest node ending at j; 0 at the last
// leaf, N-1 if none), the codes of its leaf row and of the fiber closing here, its value.
__global__ void level_flags_kernel(FlagOut f, uint64_t nnz, RootPlanRecOut ro) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    if (ro.rec) {
      uint32_t dc = (uint32_t)(f.N - 1);
      if (j + 1 == nnz) {
        dc = 0;
      } else {
        for (int l = f.N - 2; l >= 0; --l)
          if (f.c[l][j + 1] != f.c[l][j]) dc = (uint32_t)l;
      }
      const uint32_t code = plan_code(ro, ro.off_leaf, f.c[f.N - 1][j]);
      const uint32_t fcode =
          dc <= (uint32_t)(f.N - 2) ? plan_code(ro, ro.off_fiber, f.c[f.N - 2][j]) : 0u;
      const double v = ro.vals[j];
      ro.rec[j] = make_uint4(code | (dc << 29), fcode, (uint32_t)__double2loint(v),
                             (uint32_t)__double2hiint(v));
    }
    int d = f.N;  // first level whose coordinate differs from position j-1
    if (j == 0) {
      d = 0;
    } else {
      for (int l = f.N - 1; l >= 0; --l)
        if (f.c[l][j] != f.c[l][j - 1]) d = l;
    }
    for (int l = 0; l < f.N - 1; ++l) f.node[l][j] = (d <= l) ? 1u : 0u;
  }
}

// ---- Levels of a tree in two passes over its sorted coordinates, without node-number arrays
// (the derived trees).  The leaves are split into contiguous ranges of whole
// 32-leaf rows, one per warp of a full grid.  Pass 1 counts the node starts of every internal
// level in each range (ballots); a scan turns the counts into each range's first node index
// per level (and the level totals, which size ids/ptr); pass 2 walks each range row by row,
// numbers the starts by ballot + popc on top of the range's running index — no block-level
// synchronisation anywhere — and writes ids/ptr (and a ROOT plan's per-leaf records) directly.
constexpr int kLvThreads = 256;
constexpr int kLvWarps = kLvThreads / 32;

struct LevelIn {
  const uint32_t* c[SPLATT_MAX_NMODES];  // sorted coordinates per level (nnz each)
  int N;
};

// First level l <= N-2 whose coordinate at leaf j differs from leaf j-1 (0 at j = 0; N-1:
// none, i.e. only a new leaf starts at j).
template <int N>
__device__ __forceinline__ int first_diff(const LevelIn& li, uint64_t j) {
  if (j == 0) return 0;
  int d = N - 1;
#pragma unroll
  for (int l = N - 2; l >= 0; --l)
    if (__ldg(li.c[l] + j) != __ldg(li.c[l] + j - 1)) d = l;
  return d;
}

// counts[l * nwr + w] = node starts of level l among the leaves of warp range w.
template <int N>
__global__ void __launch_bounds__(kLvThreads) level_count_kernel(LevelIn li, uint64_t nnz,
                                                                 uint64_t range, uint32_t nwr,
                                                                 uint32_t* __restrict__ counts) {
  constexpr int L = N - 1;
  const uint32_t w = blockIdx.x * kLvWarps + (threadIdx.x >> 5);
  if (w >= nwr) return;
  const int lane = threadIdx.x & 31;
  const uint64_t r0 = w * range, r1 = min(nnz, r0 + range);
  uint32_t cnt[L];
#pragma unroll
  for (int l = 0; l < L; ++l) cnt[l] = 0u;
  for (uint64_t j0 = r0; j0 < r1; j0 += 32) {
    const uint64_t j = j0 + lane;
    const int d = (j < r1) ? first_diff<N>(li, j) : N - 1;
#pragma unroll
    for (int l = 0; l < L; ++l) cnt[l] += (uint32_t)__popc(__ballot_sync(0xffffffffu, d <= l));
  }
  if (lane < L) {
#pragma unroll
    for (int l = 0; l < L; ++l)
      if (lane == l) counts[(size_t)l * nwr + w] = cnt[l];
  }
}

// In place, one CTA of 1024 threads per level: counts[l][w] -> sum over ranges w' < w;
// totals[l] = the level's node count.
__global__ void __launch_bounds__(1024) level_scan_kernel(uint32_t* __restrict__ counts,
                                                          uint32_t nwr,
                                                          uint32_t* __restrict__ totals) {
  __shared__ uint32_t ws[32];
  uint32_t* c = counts + (size_t)blockIdx.x * nwr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t carry = 0u;
  for (uint32_t b = 0; b < nwr; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < nwr ? c[i] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = ws[lane];
      uint32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      ws[lane] = xi - x;
    }
    __syncthreads();
    const uint32_t excl = carry + ws[warp] + incl - v;
    if (i < nwr) c[i] = excl;
    const uint32_t last = __shfl_sync(0xffffffffu, excl + v, 31);  // (warp 31's: the chunk's end)
    __syncthreads();
    if (warp == 31 && lane == 0) ws[0] = last;
    __syncthreads();
    carry = ws[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// flag[k] = 1 iff a level-j node starts at leaf k (inclusive-scanned into node numbers).
template <int N>
__global__ void level_start_kernel(LevelIn li, uint64_t nnz, int j, uint32_t* __restrict__ flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (uint64_t)gridDim.x * blockDim.x)
    flag[k] = (first_diff<N>(li, k) <= j) ? 1u : 0u;
}

struct LevelOut {
  uint32_t* ids[SPLATT_MAX_NMODES];
  uint32_t* ptr[SPLATT_MAX_NMODES];
};

// Pass 2: warp w walks its range in rows of 32 consecutive leaves (coalesced loads and record
// stores).  A leaf's node starts at level l are the ballot of (d <= l) over its row; its node
// index is the range's first index + the starts of the earlier rows + of the lower lanes of its
// row.
template <int N>
__global__ void __launch_bounds__(kLvThreads) level_write_kernel(LevelIn li, uint64_t nnz,
                                                                 uint64_t range, uint32_t nwr,
                                                                 const uint32_t* __restrict__ bases,
                                                                 const uint32_t* __restrict__ totals,
                                                                 LevelOut lo, RootPlanRecOut ro) {
  constexpr int L = N - 1;
  const uint32_t w = blockIdx.x * kLvWarps + (threadIdx.x >> 5);
  if (w >= nwr) return;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t r0 = w * range, r1 = min(nnz, r0 + range);
  uint32_t next[L];  // index of the range's next start per level
#pragma unroll
  for (int l = 0; l < L; ++l) next[l] = __ldg(bases + (size_t)l * nwr + w);
  for (uint64_t j0 = r0; j0 < r1; j0 += 32) {
    const uint64_t j = j0 + lane;
    const bool valid = j < r1;
    const int d = valid ? first_diff<N>(li, j) : N - 1;
    uint32_t k[L];
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const uint32_t b = __ballot_sync(0xffffffffu, d <= l);
      k[l] = next[l] + (uint32_t)__popc(b & lt);
      next[l] += (uint32_t)__popc(b);
    }
    int dn = 0;  // d of leaf j+1: the shallowest node ending at leaf j (0 at the last leaf)
    if (ro.rec) dn = __shfl_down_sync(0xffffffffu, d, 1);
    if (!valid) continue;
    // nodes starting at leaf j: levels d .. L-1, each one's first child starts here too
#pragma unroll
    for (int l = 0; l < L; ++l) {
      if (l >= d) {
        lo.ids[l][k[l]] = __ldg(li.c[l] + j);
        lo.ptr[l][k[l]] = (l == L - 1) ? (uint32_t)j : k[l + 1 < L ? l + 1 : l];
      }
    }
    if (ro.rec) {
      if (lane == 31 || j + 1 >= r1) dn = (j + 1 < nnz) ? first_diff<N>(li, j + 1) : 0;
      const uint32_t dc = (uint32_t)dn;
      const uint32_t code = plan_code(ro, ro.off_leaf, __ldg(li.c[N - 1] + j));
      const uint32_t fcode =
          dc <= (uint32_t)(N - 2) ? plan_code(ro, ro.off_fiber, __ldg(li.c[N - 2] + j)) : 0u;
      const double v = __ldg(ro.vals + j);
      ro.rec[j] = make_uint4(code | (dc << 29), fcode, (uint32_t)__double2loint(v),
                             (uint32_t)__double2hiint(v));
    }
    if (j + 1 == nnz) {
#pragma unroll
      for (int l = 0; l < L; ++l)
        lo.ptr[l][totals[l]] = (l + 1 < L) ? totals[l + 1] : (uint32_t)nnz;
    }
  }
}

// After the inclusive scans node[l][j] = 1 + index of the level-l node containing j.
// All internal levels in one pass (each node array is read once, instead of once as the
// level's and once as its parent's child numbering).
struct LevelScatter {
  const uint32_t* node[SPLATT_MAX_NMODES];  // levels 0..N-2
  const uint32_t* c[SPLATT_MAX_NMODES];
  uint32_t* ids[SPLATT_MAX_NMODES];
  uint32_t* ptr[SPLATT_MAX_NMODES];
  uint64_t nodes[SPLATT_MAX_NMODES];        // levels 0..N-1 (N-1: nnz)
  int N;
};
__global__ void scatter_levels_kernel(LevelScatter ls, uint64_t nnz) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t child = (uint32_t)j + 1u;  // 1-based index of leaf j's node one level down
    for (int l = ls.N - 2; l >= 0; --l) {
      const uint32_t k = ls.node[l][j];
      const bool start = (j == 0) || (ls.node[l][j - 1] != k);
      if (!start) break;  // a node starting at j starts at every deeper level too
      ls.ids[l][k - 1] = ls.c[l][j];
      ls.ptr[l][k - 1] = child - 1u;
      child = k;
    }
    if (j == 0)
      for (int l = 0; l < ls.N - 1; ++l) ls.ptr[l][ls.nodes[l]] = (uint32_t)ls.nodes[l + 1];
  }
}

struct PtrSet {
  const uint32_t* ptr[SPLATT_MAX_NMODES];
  uint64_t nodes[SPLATT_MAX_NMODES];
  int N;
};

// Largest i in [0, n) with ptr[i] <= x (ptr has n+1 non-decreasing entries, ptr[0] = 0).
__device__ __forceinline__ uint32_t find_node(const uint32_t* __restrict__ ptr, uint64_t n,
                                              uint32_t x) {
  uint64_t lo = 0, hi = n;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (ptr[mid] <= x) lo = mid; else hi = mid;
  }
  return (uint32_t)lo;
}

__global__ void chunk_table_kernel(PtrSet ps, uint64_t nnz, int chunk, uint64_t nchunks,
                                   uint32_t* __restrict__ tab) {
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int N = ps.N;
  const uint32_t k0 = (uint32_t)(c * (uint64_t)chunk);
  uint32_t b[SPLATT_MAX_NMODES];
  b[N - 2] = find_node(ps.ptr[N - 2], ps.nodes[N - 2], k0);
  bool starts = ps.ptr[N - 2][b[N - 2]] == k0;
  for (int l = N - 3; l >= 0; --l) {
    b[l] = find_node(ps.ptr[l], ps.nodes[l], b[l + 1]);
    starts = starts && (ps.ptr[l][b[l]] == b[l + 1]);
  }
  for (int l = 0; l <= N - 2; ++l) tab[c * N + l] = b[l];
  tab[c * N + N - 1] = starts ? 0u : 1u;
}

inline int grid_for(splatt_ctx* ctx, uint64_t n, int block = 256) {
  const uint64_t want = ceil_div(n, block);
  const uint64_t cap = (uint64_t)ctx->num_sms * 16;
  return (int)std::max<uint64_t>(1, std::min(want, cap));
}

int bits_for(uint64_t dim) {
  if (dim <= 1) return 0;
  int b = 0;
  uint64_t v = dim - 1;
  while (v) { ++b; v >>= 1; }
  return b;
}

}  // namespace

void csf_perm(int N, const uint64_t* dims, int root, int* perm) {
  std::vector<int> rest;
  for (int m = 0; m < N; ++m)
    if (m != root) rest.push_back(m);
  std::stable_sort(rest.begin(), rest.end(), [&](int a, int b) { return dims[a] < dims[b]; });
  int k = 0;
  if (root >= 0) perm[k++] = root;  // root < 0: every mode by ascending length
  for (int m : rest) perm[k++] = m;
}

void csf_policy(int N, const uint64_t* dims, int policy, int* ncsf, int* roots, int* mode_csf,
                int* mode_level) {
  if (policy == SPLATT_CSF_ALL) {
    *ncsf = N;
    for (int n = 0; n < N; ++n) { roots[n] = n; mode_csf[n] = n; mode_level[n] = 0; }
    return;
  }
  SB_REQUIRE(policy == SPLATT_CSF_ONE || policy == SPLATT_CSF_TWO, "unknown CSF policy");
  int order[SPLATT_MAX_NMODES];
  csf_perm(N, dims, -1, order);  // all modes by ascending length (no root)
  *ncsf = (policy == SPLATT_CSF_ONE) ? 1 : 2;
  roots[0] = order[0];
  for (int l = 0; l < N; ++l) { mode_csf[order[l]] = 0; mode_level[order[l]] = l; }
  if (policy == SPLATT_CSF_TWO) {
    roots[1] = order[N - 1];
    mode_csf[order[N - 1]] = 1;
    mode_level[order[N - 1]] = 0;
  }
}

void validate_coo_enqueue(splatt_ctx* ctx, const uint32_t* const* d_ind, uint64_t nnz, int N,
                          const uint64_t* dims, int* d_bad) {
  IndSet s{};
  for (int m = 0; m < N; ++m) { s.p[m] = d_ind[m]; s.dims[m] = dims[m]; }
  s.N = N;
  SB_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), ctx->stream));
  validate_kernel<<<grid_for(ctx, nnz), 256, 0, ctx->stream>>>(s, nnz, d_bad);
  SB_CHECK_LAUNCH(ctx);
}

bool validate_coo_device(splatt_ctx* ctx, const uint32_t* const* d_ind, uint64_t nnz, int N,
                         const uint64_t* dims) {
  DevBuf<int> bad(1, ctx->stream);
  validate_coo_enqueue(ctx, d_ind, nnz, N, dims, bad.p);
  int h = 0;
  SB_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  host_sync(ctx);
  return h == 0;
}

namespace {

// The nonzeros of one tree in its lexicographic order: per level the sorted coordinate, and
// the values.  coord[N-1] and vals become the tree's leaf arrays (finish_levels).
struct SortedTree {
  DevBuf<uint32_t> coord[SPLATT_MAX_NMODES];
  DevBuf<double> vals;
  // Q-sorted (composite key, value) pairs, one 16-byte record per nonzero (one key group
  // only): a derived tree gathers one record per nonzero through its permutation instead of
  // N coordinates and a value (N + 1 random reads, each a DRAM burst).
  DevBuf<double2> kv;
  int shift[SPLATT_MAX_NMODES] = {0}, bits[SPLATT_MAX_NMODES] = {0};
  bool mixed = false;  // kv keys are mixed-radix (KeySpec::mixed), decoded with `mr`
  MixedRadix mr{};
};

struct KvOut {
  uint32_t* dst[SPLATT_MAX_NMODES];  // tree levels 1..N-1
  int shift[SPLATT_MAX_NMODES], bits[SPLATT_MAX_NMODES];
  int qlev[SPLATT_MAX_NMODES];       // mixed keys: the Q level of each tree level
  bool mixed;
  MixedRadix mr;
  int N;
};

// Derived tree: level l (>= 1) coordinate and value of sorted position j from the Q-sorted
// record kv[P[j]] (one 16-byte read).
__global__ void gather_kv_kernel(KvOut ko, uint64_t nnz, const uint32_t* __restrict__ P,
                                 const double2* __restrict__ kv, double* __restrict__ vout) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double2 r = kv[P[j]];
    const uint64_t k = (uint64_t)__double_as_longlong(r.x);
    if (ko.mixed) {
      uint32_t c[SPLATT_MAX_NMODES];
      mixed_decode(ko.mr, k, c);
      for (int l = 1; l < ko.N; ++l) ko.dst[l][j] = c[ko.qlev[l]];
    } else {
      for (int l = 1; l < ko.N; ++l) {
        const uint64_t m = ko.bits[l] >= 64 ? ~0ull : ((1ull << ko.bits[l]) - 1ull);
        ko.dst[l][j] = (uint32_t)((k >> ko.shift[l]) & m);
      }
    }
    vout[j] = r.y;
  }
}

__global__ void iota_kernel(uint32_t* __restrict__ p, uint64_t n) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    p[j] = (uint32_t)j;
}

// dst[l][j] = src[l][P[j]] for levels [1, N) and vout[j] = vin[P[j]].
__global__ void gather_levels_kernel(CoordOut co, uint64_t nnz, const uint32_t* __restrict__ P,
                                     const double* __restrict__ vin, double* __restrict__ vout) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nnz;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = P[j];
    for (int l = 1; l < co.N; ++l) co.dst[l][j] = co.src[l][q];
    vout[j] = vin[q];
  }
}

constexpr uint64_t kBlockLeaves = 8;  // mean leaves per node for the block move
// Derived tree rooted at Q's level j (1 <= j <= N-2), by blocks: the Q-ordered leaves of one
// level-j node stay together and in order, so a stable sort of the leaves by the level-j
// coordinate is a stable sort of the F_j level-j NODES by that coordinate, followed by a
// block move of their leaves (F_j << nnz: c5's mode-2 tree sorts 4M keys instead of 150M).
__global__ void node_keys_kernel(const uint32_t* __restrict__ node_j,
                                 const uint32_t* __restrict__ coord_j, uint64_t nnz,
                                 uint32_t* __restrict__ key, uint32_t* __restrict__ start,
                                 uint32_t* __restrict__ idx) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t n1 = node_j[k];
    if (k == 0 || node_j[k - 1] != n1) {
      key[n1 - 1] = coord_j[k];
      start[n1 - 1] = (uint32_t)k;
      idx[n1 - 1] = n1 - 1;
    }
  }
}
// leaves of the i-th node in sorted order
__global__ void node_sizes_kernel(const uint32_t* __restrict__ sidx,
                                  const uint32_t* __restrict__ start, uint64_t F, uint64_t nnz,
                                  uint32_t* __restrict__ sz) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < F;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t n = sidx[i];
    sz[i] = (n + 1 < F ? start[n + 1] : (uint32_t)nnz) - start[n];
  }
}
__global__ void node_newstart_kernel(const uint32_t* __restrict__ sidx,
                                     const uint32_t* __restrict__ off, uint64_t F,
                                     uint32_t* __restrict__ newstart) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < F;
       i += (uint64_t)gridDim.x * blockDim.x)
    newstart[sidx[i]] = off[i];
}
// leaf k (Q order) -> its position in the derived order; the derived tree's root coordinate
__global__ void node_dest_kernel(const uint32_t* __restrict__ node_j,
                                 const uint32_t* __restrict__ coord_j,
                                 const uint32_t* __restrict__ start,
                                 const uint32_t* __restrict__ newstart, uint64_t nnz,
                                 uint32_t* __restrict__ perm, uint32_t* __restrict__ root) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t n = node_j[k] - 1u;
    const uint32_t d = newstart[n] + ((uint32_t)k - start[n]);
    perm[d] = (uint32_t)k;
    root[d] = coord_j[k];
  }
}

// Full sort of the COO into the order of `perm`: packed composite keys (one or more <= 64-bit
// groups, LSD), stable radix sort of (key, position), then decode / gather into t (allocated
// by the caller, alloc_sorted).
// If t.kv is allocated (one key group), the decode also writes the (key, value) records.
void sort_full(splatt_ctx* ctx, const uint32_t* const* d_ind, const double* d_vals, uint64_t nnz,
               int N, const uint64_t* dims, const int* perm, SortedTree& t, PhaseTrace& tr) {
  cudaStream_t st = ctx->stream;
  int bits[SPLATT_MAX_NMODES];
  const uint32_t* lvl_src[SPLATT_MAX_NMODES];
  for (int l = 0; l < N; ++l) {
    bits[l] = bits_for(dims[perm[l]]);
    lvl_src[l] = d_ind[perm[l]];
  }
  // Key groups, least significant first: levels [lo, hi) with <= 64 bits in total.
  std::vector<std::pair<int, int>> groups;
  {
    int hi = N, acc = 0;
    for (int l = N - 1; l >= 0; --l) {
      if (acc + bits[l] > 64) { groups.push_back({l + 1, hi}); hi = l + 1; acc = 0; }
      acc += bits[l];
    }
    groups.push_back({0, hi});
  }
  // One key group: a mixed-radix key when its fewer bits save a radix pass.
  bool mixed = false;
  int mixed_bits = 0;
  uint64_t stride[SPLATT_MAX_NMODES] = {0};
  if (groups.size() == 1) {
    int total = 0;
    for (int l = 0; l < N; ++l) total += bits[l];
    unsigned __int128 prod = 1;
    for (int l = N - 1; l >= 0; --l) {
      stride[l] = (uint64_t)prod;
      prod *= (unsigned __int128)std::max<uint64_t>(1, dims[perm[l]]);
    }
    while (mixed_bits < 64 && ((unsigned __int128)1 << mixed_bits) < prod) ++mixed_bits;
    mixed = (mixed_bits + 7) / 8 < (total + 7) / 8 && !getenv("SPLATT_BUILD_PACKED");
  }
  const int grid = grid_for(ctx, nnz);
  ArenaScope tmp_scope(current_arena(), true);  // sort buffers: released on return
  // SPLATT_BUILD_CARRY (A/B runs): with one key group and the values on the device, the
  // values' bits travel with the keys (8-byte payload) and the decode reads them in order
  // instead of gathering them through the permutation.  Measured a tie on c5 (sort +3.0 ms,
  // decode -2.7 ms; profiles/ab_r02/README.md), so the default keeps 4-byte positions.
  const bool carry = groups.size() == 1 && !ctx->vals_pending && getenv("SPLATT_BUILD_CARRY");
  DevBuf<uint64_t> kA(nnz, st), kB(nnz, st);
  DevBuf<uint32_t> pA(carry ? 0 : nnz, st), pB(carry ? 0 : nnz, st);
  DevBuf<uint64_t> vA(carry ? nnz : 0, st), vB(carry ? nnz : 0, st);
  tr.mark("alloc");
  uint32_t* order = nullptr;  // current permutation (sorted position -> input position)
  for (size_t g = 0; g < groups.size(); ++g) {
    KeySpec ks{};
    ks.lo = groups[g].first;
    ks.hi = groups[g].second;
    int sh = 0;
    for (int l = ks.hi - 1; l >= ks.lo; --l) { ks.src[l] = lvl_src[l]; ks.shift[l] = sh; sh += bits[l]; }
    ks.mixed = mixed;
    for (int l = 0; l < N; ++l) ks.stride[l] = stride[l];
    const int total = mixed ? mixed_bits : sh;
    if (carry) {
      pack_keys_kernel<<<grid, 256, 0, st>>>(ks, nnz, nullptr, kA.p, nullptr, d_vals, vA.p);
      SB_CHECK_LAUNCH(ctx);
      radix_sort_pairs(ctx, kA.p, vA.p, kB.p, vB.p, kA.p, vA.p, nnz, 0, total);
      break;
    }
    // order == nullptr: first group, positions are the identity (written into pA).
    pack_keys_kernel<<<grid, 256, 0, st>>>(ks, nnz, order, kA.p, pA.p, nullptr, nullptr);
    SB_CHECK_LAUNCH(ctx);
    uint32_t* pin = order ? order : pA.p;
    uint32_t* pout = (pin == pB.p) ? pA.p : pB.p;
    // (kA, pin) are scratch once read: they serve as the sort's alternate buffers
    radix_sort_pairs(ctx, kA.p, pin, kB.p, pout, kA.p, pin, nnz, 0, total);
    order = pout;
  }
  tr.mark("pack+sort");
  // Sorted coordinates per level and the permuted values.  With one key group the
  // coordinates are decoded from the sorted keys (sequential reads); otherwise they are
  // gathered through the permutation.
  CoordOut co{};
  co.N = N;
  for (int l = 0; l < N; ++l) {
    co.src[l] = lvl_src[l];
    co.dst[l] = t.coord[l].p;
  }
  wait_vals(ctx);  // a host-staged value upload overlapped the sort
  if (groups.size() == 1) {
    KeySpec ks{};
    int sh = 0;
    for (int l = N - 1; l >= 0; --l) { ks.shift[l] = sh; sh += bits[l]; }
    for (int l = 0; l < N; ++l) ks.src[l] = nullptr;
    ks.lo = 0;
    ks.hi = N;
    ks.mixed = mixed;
    MixedRadix mr{};
    mr.N = N;
    for (int l = 0; l < N; ++l) {
      mr.dim[l] = (uint32_t)std::max<uint64_t>(1, dims[perm[l]]);
      mr.inv[l] = 1.0 / (double)mr.dim[l];
    }
    if (t.kv.p) {
      for (int l = 0; l < N; ++l) { t.shift[l] = ks.shift[l]; t.bits[l] = bits[l]; }
      t.mixed = mixed;
      t.mr = mr;
    }
    decode_kernel<<<grid, 256, 0, st>>>(ks, BitSet{{bits[0], bits[1], bits[2], bits[3], bits[4],
                                                    bits[5], bits[6], bits[7]}},
                                        mr, co, nnz, kB.p, carry ? nullptr : order,
                                        carry ? reinterpret_cast<const double*>(vB.p) : d_vals,
                                        t.vals.p, t.kv.p);
  } else {
    gather_kernel<<<grid, 256, 0, st>>>(co, nnz, order, d_vals, t.vals.p);
  }
  SB_CHECK_LAUNCH(ctx);
  tr.mark("decode");
}

// Allocate the sorted-coordinate arrays of a tree: coord[N-1] and vals from `out_arena`
// (they become the tree's leaf arrays), the rest from the current (scratch) arena.
void alloc_sorted(splatt_ctx* ctx, SortedTree& t, uint64_t nnz, int N, Arena* out_arena,
                  bool leaf_to_out) {
  cudaStream_t st = ctx->stream;
  for (int l = 0; l < N - 1; ++l) t.coord[l].alloc(nnz, st);
  ArenaScope o(leaf_to_out ? out_arena : current_arena(), false);
  t.coord[N - 1].alloc(nnz, st);
  t.vals.alloc(nnz, st);
}

// Levels of a tree from its sorted coordinates: "prefix 0..l changed" flags, inclusive scans
// numbering the nodes, one host sync for the node counts, scatter of ids/ptr.  Moves
// t.coord[N-1] and t.vals into the tree.
// A tree's node numbering: node[l][j] = 1 + index of the level-l node containing sorted
// position j (inclusive scans of "prefix 0..l changed" flags), and the node counts.
struct LevelNumbering {
  DevBuf<uint32_t> node[SPLATT_MAX_NMODES];
  uint64_t counts[SPLATT_MAX_NMODES] = {0};
  bool plan = false;  // a ROOT plan is under construction (its records written by the flags)
};

// Flags (+ the ROOT plan's records), scans, one host sync for the node counts.  The node
// arrays come from the current arena (the caller's scope).
void number_levels(splatt_ctx* ctx, SortedTree& t, uint64_t nnz, int N, DevCsf& out,
                   Arena* out_arena, LevelNumbering& nb, PhaseTrace& tr) {
  cudaStream_t st = ctx->stream;
  const int grid = grid_for(ctx, nnz);
  FlagOut fo{};
  fo.N = N;
  for (int l = 0; l < N; ++l) fo.c[l] = t.coord[l].p;
  for (int l = 0; l < N - 1; ++l) { nb.node[l].alloc(nnz, st); fo.node[l] = nb.node[l].p; }
  RootPlanRecOut ro;
  if (ctx->build_plan_ld > 0) {
    ArenaScope o(out_arena, false);  // the plan lives as long as the tree
    nb.plan = root_plan_begin(ctx, out, fo.c, t.vals.p, ctx->build_plan_ld, &ro);
  }
  level_flags_kernel<<<grid, 256, 0, st>>>(fo, nnz, ro);
  SB_CHECK_LAUNCH(ctx);
  {
    ArenaScope tmp_scope(current_arena(), true);
    size_t temp_bytes = 0;
    SB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, nb.node[0].p, nb.node[0].p,
                                          (int)nnz, st));
    DevBuf<uint8_t> temp(temp_bytes, st);
    for (int l = 0; l < N - 1; ++l)
      SB_CUDA(cub::DeviceScan::InclusiveSum(temp.p, temp_bytes, nb.node[l].p, nb.node[l].p,
                                            (int)nnz, st));
  }
  tr.mark("flags+scan");
  std::vector<uint32_t> counts(N, 0);
  for (int l = 0; l < N - 1; ++l)
    SB_CUDA(cudaMemcpyAsync(&counts[l], nb.node[l].p + (nnz - 1), 4, cudaMemcpyDeviceToHost, st));
  host_sync(ctx);
  for (int l = 0; l < N - 1; ++l) nb.counts[l] = counts[l];
  nb.counts[N - 1] = nnz;
}

// Scatter of ids/ptr, the ROOT plan's node-id arrays; moves t.coord[N-1] and t.vals into the
// tree.
void complete_levels(splatt_ctx* ctx, SortedTree& t, uint64_t nnz, int N, DevCsf& out,
                     Arena* out_arena, LevelNumbering& nb, PhaseTrace& tr) {
  cudaStream_t st = ctx->stream;
  const int grid = grid_for(ctx, nnz);
  for (int l = 0; l < N; ++l) out.nodes[l] = nb.counts[l];
  LevelScatter ls{};
  ls.N = N;
  for (int l = 0; l < N - 1; ++l) {
    {
      ArenaScope o(out_arena, false);
      out.ids[l].alloc(out.nodes[l], st);
      out.ptr[l].alloc(out.nodes[l] + 1, st);
    }
    ls.node[l] = nb.node[l].p;
    ls.c[l] = t.coord[l].p;
    ls.ids[l] = out.ids[l].p;
    ls.ptr[l] = out.ptr[l].p;
  }
  for (int l = 0; l < N; ++l) ls.nodes[l] = out.nodes[l];
  scatter_levels_kernel<<<grid, 256, 0, st>>>(ls, nnz);
  SB_CHECK_LAUNCH(ctx);
  tr.mark("scatter");
  if (nb.plan) {
    ArenaScope o(out_arena, false);
    root_plan_end(ctx, out);
    tr.mark("root plan");
  }
  out.ids[N - 1] = std::move(t.coord[N - 1]);
  out.vals = std::move(t.vals);
  out.tab_chunk = 0;
  out.nchunks = 0;
  out.tab.release();
}

// Levels of a tree from its sorted coordinates by the two-pass count / write kernels (no
// node-number arrays): counts per range, one host sync for the level sizes, then ids / ptr
// (and a ROOT plan's records) written directly.  Moves t.coord[N-1] and t.vals into the tree.
// Pass 1 of the level kernels (counts, scan, one host sync for the level sizes).
struct LevelCounts {
  DevBuf<uint32_t> counts, totals;  // per-range first indices (after the scan), level sizes
  uint64_t range = 0;
  uint32_t nwr = 0;
  std::vector<uint32_t> h;          // level sizes on the host
};

void count_levels(splatt_ctx* ctx, const SortedTree& t, uint64_t nnz, int N, LevelCounts& lc) {
  cudaStream_t st = ctx->stream;
  const int L = N - 1;
  LevelIn li{};
  li.N = N;
  for (int l = 0; l < N; ++l) li.c[l] = t.coord[l].p;
  // one range of whole rows per warp of a full grid (8 CTAs of 8 warps per SM)
  const uint64_t W = (uint64_t)ctx->num_sms * 8 * kLvWarps;
  const uint64_t range = ceil_div(ceil_div(nnz, W), 32) * 32;
  const uint32_t nwr = (uint32_t)ceil_div(nnz, range);
  const unsigned blocks = (unsigned)ceil_div(nwr, kLvWarps);
  lc.range = range;
  lc.nwr = nwr;
  lc.counts.alloc((size_t)nwr * L, st);
  lc.totals.alloc(L, st);
  DevBuf<uint32_t>& counts = lc.counts;
  DevBuf<uint32_t>& totals = lc.totals;
  auto count = [&](auto kern) {
    kern<<<blocks, kLvThreads, 0, st>>>(li, nnz, range, nwr, counts.p);
  };
  switch (N) {
    case 3: count(level_count_kernel<3>); break;
    case 4: count(level_count_kernel<4>); break;
    case 5: count(level_count_kernel<5>); break;
    case 6: count(level_count_kernel<6>); break;
    case 7: count(level_count_kernel<7>); break;
    default: count(level_count_kernel<8>); break;
  }
  SB_CHECK_LAUNCH(ctx);
  level_scan_kernel<<<L, 1024, 0, st>>>(counts.p, nwr, totals.p);
  SB_CHECK_LAUNCH(ctx);
  lc.h.assign(L, 0);
  SB_CUDA(cudaMemcpyAsync(lc.h.data(), totals.p, L * 4, cudaMemcpyDeviceToHost, st));
  host_sync(ctx);
}

// Levels of a tree by the two-pass count / write kernels (`pre`: pass 1 already run).
void write_levels(splatt_ctx* ctx, SortedTree& t, uint64_t nnz, int N, DevCsf& out,
                  Arena* out_arena, PhaseTrace& tr, LevelCounts* pre = nullptr) {
  cudaStream_t st = ctx->stream;
  const int L = N - 1;
  LevelIn li{};
  li.N = N;
  for (int l = 0; l < N; ++l) li.c[l] = t.coord[l].p;
  RootPlanRecOut ro;
  bool plan = false;
  if (ctx->build_plan_ld > 0) {
    ArenaScope o(out_arena, false);  // the plan lives as long as the tree
    plan = root_plan_begin(ctx, out, li.c, t.vals.p, ctx->build_plan_ld, &ro);
  }
  LevelCounts own;
  LevelCounts& lc = pre ? *pre : own;
  if (!pre) count_levels(ctx, t, nnz, N, lc);
  tr.mark("level counts");
  const std::vector<uint32_t>& h = lc.h;
  const uint64_t range = lc.range;
  const uint32_t nwr = lc.nwr;
  const unsigned blocks = (unsigned)ceil_div(nwr, kLvWarps);
  DevBuf<uint32_t>& counts = lc.counts;
  DevBuf<uint32_t>& totals = lc.totals;
  LevelOut lo{};
  for (int l = 0; l < L; ++l) {
    out.nodes[l] = h[l];
    ArenaScope o(out_arena, false);
    out.ids[l].alloc(out.nodes[l], st);
    out.ptr[l].alloc(out.nodes[l] + 1, st);
    lo.ids[l] = out.ids[l].p;
    lo.ptr[l] = out.ptr[l].p;
  }
  out.nodes[N - 1] = nnz;
  auto write = [&](auto kern) {
    kern<<<blocks, kLvThreads, 0, st>>>(li, nnz, range, nwr, counts.p, totals.p, lo, ro);
  };
  switch (N) {
    case 3: write(level_write_kernel<3>); break;
    case 4: write(level_write_kernel<4>); break;
    case 5: write(level_write_kernel<5>); break;
    case 6: write(level_write_kernel<6>); break;
    case 7: write(level_write_kernel<7>); break;
    default: write(level_write_kernel<8>); break;
  }
  SB_CHECK_LAUNCH(ctx);
  tr.mark("level write");
  if (plan) {
    ArenaScope o(out_arena, false);
    root_plan_end(ctx, out);
    tr.mark("root plan");
  }
  out.ids[N - 1] = std::move(t.coord[N - 1]);
  out.vals = std::move(t.vals);
  out.tab_chunk = 0;
  out.nchunks = 0;
  out.tab.release();
}

// Levels of a tree from its sorted coordinates (write_levels; number_levels +
// complete_levels when SPLATT_BUILD_SCATTER is set, for A/B runs).
void finish_levels(splatt_ctx* ctx, SortedTree& t, uint64_t nnz, int N, DevCsf& out,
                   Arena* out_arena, PhaseTrace& tr) {
  ArenaScope tmp_scope(current_arena(), true);
  if (nnz > 0 && !getenv("SPLATT_BUILD_SCATTER")) {
    write_levels(ctx, t, nnz, N, out, out_arena, tr);
    return;
  }
  LevelNumbering nb;
  number_levels(ctx, t, nnz, N, out, out_arena, nb, tr);
  complete_levels(ctx, t, nnz, N, out, out_arena, nb, tr);
}

// `arena`: the allocator the tree's arrays come from (nullptr: the stream-ordered pool); the
// tree's lazily built members (chunk table, seam rows, tiles) are taken from it too.
void init_tree(DevCsf& out, int N, uint64_t nnz, const uint64_t* dims, int root, Arena* arena) {
  out.N = N;
  out.nnz = nnz;
  out.arena = arena;
  csf_perm(N, dims, root, out.perm);
  for (int l = 0; l < N; ++l) {
    out.hot_ready[l] = false;
    out.dims[l] = dims[out.perm[l]];
  }
}

}  // namespace

void build_csf(splatt_ctx* ctx, const uint32_t* const* d_ind, const double* d_vals, uint64_t nnz,
               int N, const uint64_t* dims, int root, DevCsf& out) {
  DevCsf* o[1] = {&out};
  build_csf_set(ctx, d_ind, d_vals, nnz, N, dims, &root, 1, o);
}

void build_csf_set(splatt_ctx* ctx, const uint32_t* const* d_ind, const double* d_vals,
                   uint64_t nnz, int N, const uint64_t* dims, const int* roots, int ntrees,
                   DevCsf* const* outs) {
  cudaStream_t st = ctx->stream;
  PhaseTrace tr(st, "csf_build");
  if (nnz >= (1ull << 31)) fail(SPLATT_ERR_UNSUPPORTED, "nnz >= 2^31 not supported");
  // Inside a library call with an arena (cpd_als): temporaries come from the scratch arena,
  // released when this build returns; the trees themselves from the caller's arena.
  Arena* const out_arena = current_arena();
  if (out_arena && !ctx->arena_scratch) ctx->arena_scratch = new Arena();
  ArenaScope scratch(out_arena ? ctx->arena_scratch : nullptr, true);
  // (not the scratch arena made current above: the trees outlive this build)
  for (int k = 0; k < ntrees; ++k) init_tree(*outs[k], N, nnz, dims, roots[k], out_arena);
  // One full sort, in the order Q of all modes by ascending length (the tree rooted at the
  // shortest mode).  Every tree rooted at r has level order (r, Q without r), so its order is
  // a STABLE sort of the Q-ordered nonzeros by their mode-r coordinate alone — a 32-bit key
  // of ceil(log2 I_r) bits instead of the full composite key.  Ties (equal mode-r
  // coordinates) keep the Q order, i.e. (Q without r) lexicographically, then input position
  // for duplicates: bit-identical to sorting each tree's full key.
  int Q[SPLATT_MAX_NMODES], qlev[SPLATT_MAX_NMODES];
  csf_perm(N, dims, -1, Q);
  for (int l = 0; l < N; ++l) qlev[Q[l]] = l;
  int qtree = -1;
  for (int k = 0; k < ntrees; ++k)
    if (roots[k] == Q[0]) qtree = k;
  SortedTree tq;
  alloc_sorted(ctx, tq, nnz, N, out_arena, qtree >= 0);
  int total_bits = 0;
  for (int l = 0; l < N; ++l) total_bits += bits_for(dims[l]);
  if (ntrees > (qtree >= 0 ? 1 : 0) && total_bits <= 64) tq.kv.alloc(nnz, st);
  sort_full(ctx, d_ind, d_vals, nnz, N, dims, Q, tq, tr);
  const int grid = grid_for(ctx, nnz);
  // The Q tree's node numbering first when a derived tree can be built by node blocks (its
  // root at Q level 1..N-2); its scatter / plan completion comes last, as before.
  bool blocks = false;
  for (int k = 0; k < ntrees && qtree >= 0; ++k)
    if (k != qtree && qlev[roots[k]] >= 1 && qlev[roots[k]] <= N - 2) blocks = true;
  // (the numbering is needed anyway; only its node counts decide, per tree, below)
  if (getenv("SPLATT_BUILD_NOBLOCKS")) blocks = false;  // A/B runs: leaf re-sorts only
  // Q's level sizes (pass 1 of its level kernels, reused at its write below) decide the
  // block trees; their per-leaf node numbers at the root level are flag + scan.
  LevelCounts qc;
  LevelNumbering qn;
  if (blocks) {
    count_levels(ctx, tq, nnz, N, qc);
    for (int l = 0; l < N - 1; ++l) qn.counts[l] = qc.h[l];
    qn.counts[N - 1] = nnz;
    for (int k = 0; k < ntrees; ++k) {
      const int j = qlev[roots[k]];
      if (k == qtree || j < 1 || j > N - 2 || nnz < kBlockLeaves * qn.counts[j] || qn.node[j].p)
        continue;
      qn.node[j].alloc(nnz, st);
      LevelIn li{};
      li.N = N;
      for (int l = 0; l < N; ++l) li.c[l] = tq.coord[l].p;
      auto start = [&](auto kern) { kern<<<grid, 256, 0, st>>>(li, nnz, j, qn.node[j].p); };
      switch (N) {
        case 3: start(level_start_kernel<3>); break;
        case 4: start(level_start_kernel<4>); break;
        case 5: start(level_start_kernel<5>); break;
        case 6: start(level_start_kernel<6>); break;
        case 7: start(level_start_kernel<7>); break;
        default: start(level_start_kernel<8>); break;
      }
      SB_CHECK_LAUNCH(ctx);
      ArenaScope tmp_scope(current_arena(), true);
      size_t tb = 0;
      SB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, qn.node[j].p, qn.node[j].p, (int)nnz, st));
      DevBuf<uint8_t> temp(tb, st);
      SB_CUDA(cub::DeviceScan::InclusiveSum(temp.p, tb, qn.node[j].p, qn.node[j].p, (int)nnz, st));
    }
    tr.mark("Q levels");
  }
  for (int k = 0; k < ntrees; ++k) {
    if (k == qtree) continue;
    DevCsf& out = *outs[k];
    const int r = roots[k];
    const int j = qlev[r];
    ArenaScope tree_scope(current_arena(), true);
    SortedTree tr_;
    alloc_sorted(ctx, tr_, nnz, N, out_arena, true);
    {
      ArenaScope sort_scope(current_arena(), true);
      DevBuf<uint32_t> perm_out(nnz, st);
      const int nb = std::max(1, bits_for(dims[r]));
      // (blocks only where they are long: the block move scatters each node's leaves
      // together, so ~2-leaf nodes would turn it into a random scatter — c5's mode-1 tree,
      // 77M nodes: 11.8 ms against 5.0 for the leaf re-sort)
      if (blocks && j >= 1 && j <= N - 2 && nnz >= kBlockLeaves * qn.counts[j]) {
        const uint64_t F = qn.counts[j];
        DevBuf<uint32_t> key(F, st), skey(F, st), idx(F, st), sidx(F, st), start(F, st),
            sz(F, st), off(F, st), newstart(F, st);
        node_keys_kernel<<<grid, 256, 0, st>>>(qn.node[j].p, tq.coord[j].p, nnz, key.p, start.p,
                                               idx.p);
        SB_CHECK_LAUNCH(ctx);
        size_t tb2 = 0;
        SB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, sz.p, off.p, (int)F, st));
        DevBuf<uint8_t> temp(tb2, st);
        radix_sort_pairs(ctx, key.p, idx.p, skey.p, sidx.p, key.p, idx.p, F, 0, nb);
        const int gF = grid_for(ctx, F);
        node_sizes_kernel<<<gF, 256, 0, st>>>(sidx.p, start.p, F, nnz, sz.p);
        SB_CHECK_LAUNCH(ctx);
        SB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb2, sz.p, off.p, (int)F, st));
        node_newstart_kernel<<<gF, 256, 0, st>>>(sidx.p, off.p, F, newstart.p);
        SB_CHECK_LAUNCH(ctx);
        node_dest_kernel<<<grid, 256, 0, st>>>(qn.node[j].p, tq.coord[j].p, start.p, newstart.p,
                                               nnz, perm_out.p, tr_.coord[0].p);
        SB_CHECK_LAUNCH(ctx);
      } else {
        DevBuf<uint32_t> pos(nnz, st), tk(nnz, st);
        iota_kernel<<<grid, 256, 0, st>>>(pos.p, nnz);
        SB_CHECK_LAUNCH(ctx);
        radix_sort_pairs(ctx, tq.coord[j].p, pos.p, tr_.coord[0].p, perm_out.p, tk.p, pos.p, nnz,
                         0, nb);
      }
      if (tq.kv.p) {
        KvOut ko{};
        ko.N = N;
        ko.mixed = tq.mixed;
        ko.mr = tq.mr;
        for (int l = 1; l < N; ++l) {
          ko.dst[l] = tr_.coord[l].p;
          ko.shift[l] = tq.shift[qlev[out.perm[l]]];
          ko.bits[l] = tq.bits[qlev[out.perm[l]]];
          ko.qlev[l] = qlev[out.perm[l]];
        }
        gather_kv_kernel<<<grid, 256, 0, st>>>(ko, nnz, perm_out.p, tq.kv.p, tr_.vals.p);
      } else {
        CoordOut co{};
        co.N = N;
        for (int l = 1; l < N; ++l) {
          co.src[l] = tq.coord[qlev[out.perm[l]]].p;
          co.dst[l] = tr_.coord[l].p;
        }
        gather_levels_kernel<<<grid, 256, 0, st>>>(co, nnz, perm_out.p, tq.vals.p, tr_.vals.p);
      }
      SB_CHECK_LAUNCH(ctx);
      tr.mark("derived sort");
    }
    finish_levels(ctx, tr_, nnz, N, out, out_arena, tr);
  }
  if (qtree >= 0) {
    if (blocks) write_levels(ctx, tq, nnz, N, *outs[qtree], out_arena, tr, &qc);
    else finish_levels(ctx, tq, nnz, N, *outs[qtree], out_arena, tr);
  }
}

namespace {

// flag[ptr[j]] = 1 for the F child-range starts of a level (flag zeroed by the caller).
__global__ void mark_starts_kernel(const uint32_t* __restrict__ ptr, uint64_t F,
                                   uint32_t* __restrict__ flag) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < F;
       j += (uint64_t)gridDim.x * blockDim.x)
    flag[ptr[j]] = 1u;
}

// out[k] = table[idx[k] - 1] (idx from an inclusive scan of start flags: 1-based).
__global__ void gather_minus1_kernel(const uint32_t* __restrict__ table,
                                     const uint32_t* __restrict__ idx, uint64_t n,
                                     uint32_t* __restrict__ out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x)
    out[k] = table[idx[k] - 1u];
}

// Tile key and position per leaf, and the per-tile counts: a shared-memory histogram per
// block, one global atomic per block and tile (T <= 8; per-leaf global atomics on T
// counters serialised: 100M leaves took ~45 ms).
__global__ void tile_key_kernel(const uint32_t* __restrict__ leaf, uint64_t n, uint64_t rows,
                                int T, uint32_t* __restrict__ key, uint32_t* __restrict__ pos,
                                unsigned long long* __restrict__ cnt) {
  __shared__ unsigned int h[8];
  if (threadIdx.x < 8) h[threadIdx.x] = 0u;
  __syncthreads();
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(leaf[k] / rows);
    key[k] = t;
    pos[k] = (uint32_t)k;
    atomicAdd(&h[t], 1u);
  }
  __syncthreads();
  if ((int)threadIdx.x < T && h[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

}  // namespace

void tile_tree(splatt_ctx* ctx, DevCsf& c, int T) {
  cudaStream_t st = ctx->stream;
  PhaseTrace tr(st, "tile_tree");
  const int N = c.N;
  const uint64_t nnz = c.nnz;
  const uint64_t rows = (c.dims[N - 1] + T - 1) / T;
  Arena* const out_arena = c.arena;  // the tiles live as long as the tree
  if (out_arena && !ctx->arena_scratch) ctx->arena_scratch = new Arena();
  ArenaScope scratch(out_arena ? ctx->arena_scratch : nullptr, true);
  const int grid = grid_for(ctx, nnz);
  // 1. per-leaf node index and coordinate of every internal level (start flags + scans)
  DevBuf<uint32_t> node(nnz, st), lvl[SPLATT_MAX_NMODES], tmp(nnz, st);
  size_t tb = 0;
  SB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, tmp.p, tmp.p, (int)nnz, st));
  DevBuf<uint8_t> temp(tb, st);
  SB_CUDA(cudaMemsetAsync(node.p, 0, nnz * 4, st));
  mark_starts_kernel<<<grid, 256, 0, st>>>(c.ptr[N - 2].p, c.nodes[N - 2], node.p);
  SB_CHECK_LAUNCH(ctx);
  SB_CUDA(cub::DeviceScan::InclusiveSum(temp.p, tb, node.p, node.p, (int)nnz, st));  // 1-based
  for (int l = N - 2; l >= 0; --l) {
    lvl[l].alloc(nnz, st);
    gather_minus1_kernel<<<grid, 256, 0, st>>>(c.ids[l].p, node.p, nnz, lvl[l].p);
    SB_CHECK_LAUNCH(ctx);
    if (l == 0) break;
    // parent (level l-1) of every level-l node, then of every leaf
    const uint64_t F = c.nodes[l];
    DevBuf<uint32_t> par(F, st);
    SB_CUDA(cudaMemsetAsync(par.p, 0, F * 4, st));
    mark_starts_kernel<<<grid_for(ctx, c.nodes[l - 1]), 256, 0, st>>>(c.ptr[l - 1].p,
                                                                      c.nodes[l - 1], par.p);
    SB_CHECK_LAUNCH(ctx);
    SB_CUDA(cub::DeviceScan::InclusiveSum(temp.p, tb, par.p, par.p, (int)F, st));
    gather_minus1_kernel<<<grid, 256, 0, st>>>(par.p, node.p, nnz, tmp.p);  // parent + 1
    SB_CHECK_LAUNCH(ctx);
    std::swap(node, tmp);  // whole buffers: one may be arena memory, the other pooled
  }
  // 2. stable order by tile (the tree order inside each tile is kept)
  DevBuf<uint32_t> key(nnz, st), key2(nnz, st), pos(nnz, st), perm(nnz, st);
  DevBuf<unsigned long long> cnt(T, st);
  SB_CUDA(cudaMemsetAsync(cnt.p, 0, T * 8, st));
  tile_key_kernel<<<grid, 256, 0, st>>>(c.ids[N - 1].p, nnz, rows, T, key.p, pos.p, cnt.p);
  SB_CHECK_LAUNCH(ctx);
  int bits = 1;
  while ((1 << bits) < T) ++bits;
  radix_sort_pairs(ctx, key.p, pos.p, key2.p, perm.p, key.p, pos.p, nnz, 0, bits);
  std::vector<unsigned long long> hcnt(T);
  SB_CUDA(cudaMemcpyAsync(hcnt.data(), cnt.p, T * 8, cudaMemcpyDeviceToHost, st));
  host_sync(ctx);
  tr.mark("expand+order");
  // 3. every tile: gather its coordinates / values (tree order), then its levels
  c.tiles.clear();
  uint64_t off = 0;
  for (int t = 0; t < T; ++t) {
    const uint64_t n = hcnt[t];
    if (n == 0) continue;
    auto tile = std::make_unique<DevCsf>();
    tile->N = N;
    tile->nnz = n;
    tile->arena = out_arena;
    for (int l = 0; l < N; ++l) {
      tile->perm[l] = c.perm[l];
      tile->dims[l] = c.dims[l];
      tile->hot_ready[l] = false;
    }
    ArenaScope tile_scope(current_arena(), true);
    SortedTree ts;
    alloc_sorted(ctx, ts, n, N, out_arena, true);
    CoordOut co{};
    co.N = N;
    for (int l = 0; l < N; ++l) {
      co.src[l] = (l < N - 1) ? lvl[l].p : c.ids[N - 1].p;
      co.dst[l] = ts.coord[l].p;
    }
    gather_kernel<<<grid_for(ctx, n), 256, 0, st>>>(co, n, perm.p + off, c.vals.p, ts.vals.p);
    SB_CHECK_LAUNCH(ctx);
    finish_levels(ctx, ts, n, N, *tile, out_arena, tr);
    c.tiles.push_back(std::move(tile));
    off += n;
  }
  c.tile_rows = rows;
}

void ensure_chunk_table(splatt_ctx* ctx, DevCsf& c, int chunk) {
  if (c.tab_chunk == chunk && c.tab.p) return;
  c.nchunks = ceil_div(c.nnz, chunk);
  ArenaScope own(c.arena, false);  // lives as long as the tree
  c.tab.alloc(c.nchunks * c.N, ctx->stream);
  PtrSet ps{};
  ps.N = c.N;
  for (int l = 0; l < c.N - 1; ++l) { ps.ptr[l] = c.ptr[l].p; ps.nodes[l] = c.nodes[l]; }
  chunk_table_kernel<<<(unsigned)ceil_div(c.nchunks, 256), 256, 0, ctx->stream>>>(
      ps, c.nnz, chunk, c.nchunks, c.tab.p);
  SB_CHECK_LAUNCH(ctx);
  c.tab_chunk = chunk;
}

}  // namespace sb
