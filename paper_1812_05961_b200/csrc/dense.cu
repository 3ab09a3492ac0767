// dense.cu — the small fp64 kernels of each ALS mode update.
//
// Alg. 1 per mode n: V = *_{m!=n} G_m (line 4), A_n = M V^dagger
// (line 5, realised as potrf/potrs), normalise columns into lambda
// (line 6), Gram refresh, and the fit (line 13).  Readings: DESIGN.md §2 (C-7 pivot
// threshold / ridge, C-8 norm schedule, C-10 fit identity).
//
// Structure: one CTA forms V = *G and inverts it by Gauss-Jordan
// elimination without pivoting (V is SPD; its k-th pivot is the k-th Cholesky pivot squared,
// so the C-7 pivot test and ridge retry apply unchanged); persistent CTAs solve slabs of
// rows X = M V^-1 (fp64 tensor cores, DMMA) and, while a solved slab is still on chip, add
// its partial Gram, column max |a| and fit inner product <M_i, A_i>; partials are reduced
// in a fixed order, so every result is deterministic.
#include <algorithm>
#include <cmath>

#include "dense.hpp"

namespace sb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_factor_kernel(double* __restrict__ A, uint64_t I, int R, int ld,
                                   uint64_t seed, uint64_t base) {
  const uint64_t total = I * (uint64_t)ld;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / ld;
    const int r = (int)(e % ld);
    double v = 0.0;
    if (r < R) {
      const uint64_t k = base + i * (uint64_t)R + (uint64_t)r;
      const uint64_t z = splitmix_mix(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
      v = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    }
    A[e] = v;
  }
}

// Deterministic block sum: per-thread strided partials, then a fixed shared-memory tree.
__device__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void sumsq_partial_kernel(const double* __restrict__ v, uint64_t n,
                                     double* __restrict__ part) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x)
    acc = fma(v[j], v[j], acc);
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int P, double* out) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  for (int p = threadIdx.x; p < P; p += blockDim.x) acc += part[p];
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) out[0] = s;
}

// One CTA: V = *_{m != n} G_m (ascending m) and V^-1 (Alg. 1 line 5's V^dagger,
// PAPER.md:194; V is SPD, so V^dagger = V^-1) by in-place Gauss-Jordan elimination without
// pivoting.  On an SPD matrix the k-th Gauss-Jordan pivot is the k-th Schur-complement
// diagonal d_k = V_kk - sum_{m<k} L_km^2, i.e. the square of the k-th Cholesky pivot, so
// the failure test of C-7 applies unchanged: fail if d_k <= 1e-12 * max_j V_jj; on failure
// retry once with V + (1e-12 * trace(V) / R) I; a second failure sets *status.  Output:
// Vinv, ld x ld (row-major, zero pad rows/columns >= R).  Each step is one parallel pass
// over the matrix (two barriers), so the kernel is R short steps, not R^2 serial ones.
__global__ void hadamard_inverse_kernel(const double* __restrict__ G_all, int N, int n, int R,
                                        int ld, double* __restrict__ Vinv, int* status,
                                        const double* __restrict__ sig, double* __restrict__ tau,
                                        const int* conv) {
  extern __shared__ double sm[];
  if (conv && *conv) return;
  double* A = sm;            // R x R working matrix
  double* prow = A + R * R;  // pivot row of the current step (R)
  double* pcol = prow + R;   // pivot column of the current step (R)
  __shared__ int failed;
  __shared__ double mxd, ridge;
  const int RR = R * R;
  for (int attempt = 0; attempt < 2; ++attempt) {
    __syncthreads();
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {  // V (re-read for the retry)
      double p = 1.0;
      bool first = true;
      for (int m = 0; m < N; ++m) {
        if (m == n) continue;
        const double g = G_all[(size_t)m * RR + e];
        p = first ? g : p * g;
        first = false;
      }
      A[e] = p;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      failed = 0;
      double mx = 0.0, tr = 0.0;
      for (int j = 0; j < R; ++j) { mx = fmax(mx, A[j * R + j]); tr += A[j * R + j]; }
      if (attempt == 0) {
        ridge = 1e-12 * tr / R;
        mxd = mx;
      } else {
        for (int j = 0; j < R; ++j) A[j * R + j] += ridge;
        mxd = mx + ridge;
      }
    }
    __syncthreads();
    const double th = 1e-12 * mxd;  // 1e-12 x max diagonal of the matrix being inverted
    for (int k = 0; k < R; ++k) {
      const double d = A[k * R + k];
      if (!(d > th)) { failed = 1; break; }  // uniform: every thread reads the same d
      const double inv = 1.0 / d;
      for (int j = threadIdx.x; j < R; j += blockDim.x) {
        prow[j] = (j == k) ? inv : A[k * R + j] * inv;
        pcol[j] = (j == k) ? 0.0 : A[j * R + k];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < RR; e += blockDim.x) {
        const int i = e / R, j = e % R;
        if (i == k) {
          A[e] = prow[j];
        } else if (j == k) {
          A[e] = -pcol[i] * inv;
        } else {
          A[e] = fma(-pcol[i], prow[j], A[e]);
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (!failed) break;
  }
  if (failed) {
    if (threadIdx.x == 0) *status = 1;
    return;
  }
  // tau_i = prod_{m != n} sig_m[i]: the column scale mapping the MTTKRP of the stored
  // (unnormalised) factors to that of the normalised ones
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    double t = 1.0;
    if (sig)
      for (int m = 0; m < N; ++m)
        if (m != n) t *= sig[(size_t)m * R + i];
    prow[i] = t;
    tau[i] = t;
  }
  __syncthreads();
  // symmetrise (the elimination rounds the two triangles differently), scale row i by tau_i
  // (x = (m o tau) V^-1 = m (diag(tau) V^-1)) and pad to ld
  for (int e = threadIdx.x; e < ld * ld; e += blockDim.x) {
    const int i = e / ld, j = e % ld;
    double v = 0.0;
    if (i < R && j < R) v = prow[i] * (0.5 * (A[i * R + j] + A[j * R + i]));
    Vinv[e] = v;
  }
}

// ------------------------------------------------- row solves + Gram + colmax
// Per row m (length R): x = m V^-1 (line 5, with V^-1 from hadamard_cholesky), computed by
// a lane group of G lanes (lane q owns columns 4q..4q+3, 256-bit shared-memory operands),
// so every output is an independent length-R dot product (no serial substitution chain).
// inner += m . x (the row's share of <X, Z>, C-10).  CTAs walk tiles of T = RPG x groups
// rows staged in shared memory with cp.async (stride ld+2 doubles: conflict-free 128-bit
// accesses); the solved tile replaces the staged rows, is written back coalesced and,
// while still in shared memory, every thread accumulates a 4x4 block of the partial Gram
// (rows split into S subsets when there are fewer block pairs than threads) and a
// column-max |a| over a row subset.  Without `solve` the kernel only reads A (initial
// Grams).  Partials are reduced in a fixed order (reduce_stats_kernel): deterministic.
__device__ __forceinline__ void block_pair(int q, int nb, int& rb, int& cb) {
  int r = 0;
  while (q >= nb - r) { q -= nb - r; ++r; }
  rb = r;
  cb = r + q;
}

struct RowsArgs {
  const double* M;
  double* A;
  uint64_t lo, hi, ntiles;
  int R, ld, T;
  const double* Vinv;
  const double* tau;  // R column scales of M (stored -> true MTTKRP), folded into Vinv's rows
  const int* status;
  const int* conv;  // ALS converged: skip (splatt_ctx::d_conv)
  double* part;  // gridDim.x x stats_len(R)
  bool solve;
  PeerRows peers;  // n = 0: none
};

#ifndef SB_SOLVE_RPG
#define SB_SOLVE_RPG 4
#endif
constexpr int kRPG = SB_SOLVE_RPG;  // rows per lane group per tile

// BT threads per CTA; tiles of T = (BT / G) * kRPG rows, double-buffered: the next tile's
// rows are copied (cp.async) while the current one is solved.
template <int kMaxBP, int G, int BT>  // kMaxBP: 1 when <= BT block pairs, else 3
__global__ void __launch_bounds__(BT, kMaxBP == 1 ? (BT == 128 ? 4 : 2) : 1)
    solve_gram_kernel(const RowsArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[BT];
  const int R = a.R, ld = a.ld, ldp = ld + 2, T = a.T;
  const size_t SL = (size_t)R * R + R + 1;
  double* out = a.part + (size_t)blockIdx.x * SL;
  double* Ws = sm;                                   // ld x ld if solve (zero pads)
  const int nb = ld / 4;
  const int nbp = nb * (nb + 1) / 2;
  const int S = nbp >= BT ? 1 : BT / nbp;
  const size_t tile_sz = (size_t)T * ldp;
  double* taus = Ws + (a.solve ? ld * ld : 0);       // ld (solve only)
  double* tiles = taus + (a.solve ? ld : 0);         // 2 x T x ldp (+ combine area)
  if (a.solve)
    for (int r = threadIdx.x; r < ld; r += blockDim.x) taus[r] = (r < R) ? a.tau[r] : 0.0;
  const bool dead = (a.status && *a.status) || (a.conv && *a.conv);
  if (a.solve && !dead) {  // Vinv is ld x ld with zero pads: one contiguous async copy
    const unsigned base = (unsigned)__cvta_generic_to_shared(Ws);
    for (int e = threadIdx.x; e < ld * ld / 2; e += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + 16 * e),
                   "l"(a.Vinv + 2 * e));
  }
  const double* src = a.solve ? a.M : a.A;
  const int half = ld / 2;  // 16-byte pairs per row
  auto load_tile = [&](uint64_t tI, double* buf) {
    if (tI < a.ntiles && !dead) {
      const uint64_t row0 = a.lo + tI * T;
      const uint64_t left = a.hi - row0;
      const int nrows = left < (uint64_t)T ? (int)left : T;
      const double* gsrc = src + row0 * ld;
      for (int e = threadIdx.x; e < nrows * half; e += blockDim.x) {
        const int r = e / half, c = 2 * (e % half);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(buf + r * ldp + c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gsrc + 2 * e));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int q = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  const int col = 4 * q;
  const bool active = col < ld;
  const int s_id = (S > 1) ? (int)threadIdx.x / nbp : 0;
  int rb[kMaxBP], cb[kMaxBP];
  double g[kMaxBP][16];
#pragma unroll
  for (int k = 0; k < kMaxBP; ++k) {
    const int qq = (S > 1) ? (int)threadIdx.x % nbp + k * nbp : (int)threadIdx.x + k * BT;
    rb[k] = cb[k] = -1;
    if ((S > 1 ? (k == 0 && s_id < S) : qq < nbp)) block_pair(qq, nb, rb[k], cb[k]);
#pragma unroll
    for (int z = 0; z < 16; ++z) g[k][z] = 0.0;
  }
  // column max: thread -> column cm (< CW, CW = pow2 >= R) over row subset cs of CS
  const int CW = R <= 32 ? 32 : (R <= 64 ? 64 : 128);
  const int CS = BT / CW;
  const int cm = threadIdx.x % CW, cs = threadIdx.x / CW;
  double cmax = 0.0, inner = 0.0;
  load_tile(blockIdx.x, tiles);
  int cur = 0;
  for (uint64_t tI = blockIdx.x; tI < a.ntiles && !dead; tI += gridDim.x, cur ^= 1) {
    const uint64_t row0 = a.lo + tI * T;
    const uint64_t left = a.hi - row0;
    const int nrows = left < (uint64_t)T ? (int)left : T;
    double* tile = tiles + cur * tile_sz;
    load_tile(tI + gridDim.x, tiles + (cur ^ 1) * tile_sz);  // prefetch the next tile
    asm volatile("cp.async.wait_group 1;" ::: "memory");      // this tile (and Vinv) landed
    __syncthreads();
    if (a.solve) {
      // x[u][0..3] = sum_k m_u[k] Vinv[k][col..col+3] for the group's kRPG rows: each
      // Vinv operand is loaded once per k for all kRPG rows (register blocking).
      double x[kRPG][4];
#pragma unroll
      for (int u = 0; u < kRPG; ++u) x[u][0] = x[u][1] = x[u][2] = x[u][3] = 0.0;
      const int r0 = grp * kRPG;
      if (active && r0 < nrows) {
        const double* wc = Ws + col;
        const double* m0 = tile + r0 * ldp;
        int k = 0;
        for (; k + 1 < R; k += 2) {
          const double2 w0a = *reinterpret_cast<const double2*>(wc + k * ld);
          const double2 w0b = *reinterpret_cast<const double2*>(wc + k * ld + 2);
          const double2 w1a = *reinterpret_cast<const double2*>(wc + (k + 1) * ld);
          const double2 w1b = *reinterpret_cast<const double2*>(wc + (k + 1) * ld + 2);
#pragma unroll
          for (int u = 0; u < kRPG; ++u) {
            const double2 mv = *reinterpret_cast<const double2*>(m0 + u * ldp + k);
            x[u][0] = fma(mv.x, w0a.x, x[u][0]);
            x[u][1] = fma(mv.x, w0a.y, x[u][1]);
            x[u][2] = fma(mv.x, w0b.x, x[u][2]);
            x[u][3] = fma(mv.x, w0b.y, x[u][3]);
            x[u][0] = fma(mv.y, w1a.x, x[u][0]);
            x[u][1] = fma(mv.y, w1a.y, x[u][1]);
            x[u][2] = fma(mv.y, w1b.x, x[u][2]);
            x[u][3] = fma(mv.y, w1b.y, x[u][3]);
          }
        }
        if (k < R) {
          const double2 wa = *reinterpret_cast<const double2*>(wc + k * ld);
          const double2 wb = *reinterpret_cast<const double2*>(wc + k * ld + 2);
#pragma unroll
          for (int u = 0; u < kRPG; ++u) {
            const double mk = m0[u * ldp + k];
            x[u][0] = fma(mk, wa.x, x[u][0]);
            x[u][1] = fma(mk, wa.y, x[u][1]);
            x[u][2] = fma(mk, wb.x, x[u][2]);
            x[u][3] = fma(mk, wb.y, x[u][3]);
          }
        }
#pragma unroll
        for (int u = 0; u < kRPG; ++u)
          if (r0 + u < nrows)
#pragma unroll
            for (int z = 0; z < 4; ++z)
              if (col + z < R) inner = fma(m0[u * ldp + col + z] * taus[col + z], x[u][z], inner);
      }
      __syncthreads();  // every group has read its m rows
#pragma unroll
      for (int u = 0; u < kRPG; ++u) {
        const int r = r0 + u;
        if (r < nrows && active) {
          double2* d = reinterpret_cast<double2*>(tile + r * ldp + col);
          d[0] = make_double2(x[u][0], x[u][1]);
          d[1] = make_double2(x[u][2], x[u][3]);
        }
      }
      __syncthreads();
      double2* dst = reinterpret_cast<double2*>(a.A + row0 * ld);
      for (int e = threadIdx.x; e < nrows * half; e += blockDim.x)
        dst[e] = *reinterpret_cast<const double2*>(tile + (e / half) * ldp + 2 * (e % half));
      for (int q = 0; q < a.peers.n; ++q) {  // fused all-gather: the peers' copies of the rows
        double2* pd = reinterpret_cast<double2*>(a.peers.p[q] + row0 * ld);
        for (int e = threadIdx.x; e < nrows * half; e += blockDim.x)
          pd[e] = *reinterpret_cast<const double2*>(tile + (e / half) * ldp + 2 * (e % half));
      }
    }
#pragma unroll
    for (int k = 0; k < kMaxBP; ++k) {
      if (rb[k] < 0) continue;
      const int c0 = 4 * rb[k], c1 = 4 * cb[k];
      for (int r = s_id; r < nrows; r += S) {
        const double* row = tile + r * ldp;
        const double2 u01 = *reinterpret_cast<const double2*>(row + c0);
        const double2 u23 = *reinterpret_cast<const double2*>(row + c0 + 2);
        const double2 w01 = *reinterpret_cast<const double2*>(row + c1);
        const double2 w23 = *reinterpret_cast<const double2*>(row + c1 + 2);
        const double u[4] = {u01.x, u01.y, u23.x, u23.y};
        const double w[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) g[k][i * 4 + j] = fma(u[i], w[j], g[k][i * 4 + j]);
      }
    }
    if (cm < R)
      for (int r = cs; r < nrows; r += CS) cmax = fmax(cmax, fabs(tile[r * ldp + cm]));
    __syncthreads();  // the buffer is refilled by the next iteration's prefetch
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (S > 1) {  // combine the row subsets (reuses the tile area)
    double* comb = tiles;
    __syncthreads();
    if (rb[0] >= 0)
      for (int z = 0; z < 16; ++z) comb[((size_t)s_id * nbp + threadIdx.x % nbp) * 16 + z] = g[0][z];
    __syncthreads();
    if ((int)threadIdx.x < nbp) {
      for (int z = 0; z < 16; ++z) {
        double acc = 0.0;
        for (int s2 = 0; s2 < S; ++s2) acc += comb[((size_t)s2 * nbp + threadIdx.x) * 16 + z];
        g[0][z] = acc;
      }
    } else {
      rb[0] = -1;
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxBP; ++k) {
    if (rb[k] < 0) continue;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        const int r = 4 * rb[k] + i, c2 = 4 * cb[k] + j;
        if (r < R && c2 < R && r <= c2) {
          out[(size_t)r * R + c2] = g[k][i * 4 + j];
          out[(size_t)c2 * R + r] = g[k][i * 4 + j];
        }
      }
  }
  // column max over the CS row subsets (fixed order), via the shared reduction buffer
  __syncthreads();
  red[threadIdx.x] = cmax;
  __syncthreads();
  if ((int)threadIdx.x < R) {
    double mx = 0.0;
    for (int c = 0; c < CS; ++c) mx = fmax(mx, red[c * CW + threadIdx.x]);
    out[(size_t)R * R + 1 + threadIdx.x] = mx;
  }
  __syncthreads();
  const double tot = block_sum(inner, red);
  if (threadIdx.x == 0) out[(size_t)R * R] = tot;
}

// ------------------------------------- row solves + Gram on the fp64 tensor cores (DMMA)
// The same contract as solve_gram_kernel for R <= 8 NT, as two small dense contractions
// per slab of 8 rows (mma.sync m8n8k4 f64 — tcgen05 has no fp64 kind, so this is the
// sm_100a fp64 tensor-core path):  X = M_slab (8 x ld) . Vinv (ld x 8NT)  and
// G~ += X^T X.  Every warp works alone on its own slabs (rows lo + 8s .. +8), staged with
// cp.async into a two-slab ring (row stride ldp = 8NT + 4 doubles: conflict-free fragment
// loads for both products); the row solve's A operand comes from the staged M rows, its B
// operand (Vinv, ld x 8NT, zero pads) from shared memory; the solved slab replaces the M
// rows in shared memory (for the Gram's fragments and a coalesced write-back); column max
// |x| and <M o tau, X> are taken from the accumulator registers.  Warps are combined in
// fixed order at the end, so the per-CTA partial is deterministic.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NT>
struct MmaShape {
  static constexpr int RP = 8 * NT;        // padded columns
  static constexpr int LDP = RP + 4;       // slab row stride (doubles)
  static constexpr int NP = NT * (NT + 1) / 2;  // upper-triangular 8x8 Gram tiles
};

#ifndef SB_MMA_MINB
#define SB_MMA_MINB 1
#endif
constexpr int mma_minb(int NT) { return NT <= 5 ? SB_MMA_MINB : 1; }
template <int NT, int W>
__global__ void __launch_bounds__(W * 32, mma_minb(NT)) solve_gram_mma_kernel(const RowsArgs a) {
  using Sh = MmaShape<NT>;
  constexpr int RP = Sh::RP, LDP = Sh::LDP, NP = Sh::NP;
  constexpr int KS = RP / 4;  // k-steps upper bound (ld <= RP)
  extern __shared__ __align__(16) double sm[];
  const int R = a.R, ld = a.ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* Ws = sm;                                  // ld x RP (solve)
  double* taus = Ws + (a.solve ? (size_t)ld * RP : 0);  // RP
  double* slabs = taus + RP;                        // W x 2 x 8 x LDP
  slabs = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(slabs) + 15) & ~uintptr_t(15));
  double* mine = slabs + (size_t)warp * 2 * 8 * LDP;
  const bool dead = (a.status && *a.status) || (a.conv && *a.conv);
  // columns ld..LDP-1 of the warp's slab ring stay zero (cp.async fills columns < ld)
  for (int e = lane; e < 2 * 8 * (LDP - ld); e += 32)
    mine[(e / (LDP - ld)) * LDP + ld + e % (LDP - ld)] = 0.0;
  __syncwarp();
  const uint64_t nslabs = (a.hi - a.lo + 7) / 8;
  const uint64_t stride = (uint64_t)gridDim.x * W;
  const double* src = a.solve ? a.M : a.A;
  const int half = ld / 2;
  auto load_slab = [&](uint64_t sI, double* buf) {
    if (sI < nslabs && !dead) {
      const uint64_t row0 = a.lo + sI * 8;
      for (int e = lane; e < 8 * half; e += 32) {
        const int r = e / half, c = 2 * (e % half);
        const bool in = row0 + r < a.hi;
        const double* gp = src + (in ? (row0 + r) * ld + c : 0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(buf + r * LDP + c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(gp),
                     "r"(in ? 16 : 0));
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  uint64_t sI = (uint64_t)blockIdx.x * W + warp;
  load_slab(sI, mine);  // in flight while Vinv is staged
  if (a.solve) {
    for (int e = threadIdx.x; e < ld * RP; e += blockDim.x) {
      const int k = e / RP, n = e % RP;
      Ws[e] = (n < ld) ? a.Vinv[(size_t)k * ld + n] : 0.0;
    }
    for (int c = threadIdx.x; c < RP; c += blockDim.x) taus[c] = (c < R) ? a.tau[c] : 0.0;
  }
  __syncthreads();

  double gacc[NP][2];
#pragma unroll
  for (int p = 0; p < NP; ++p) gacc[p][0] = gacc[p][1] = 0.0;
  double cm[NT][2];
#pragma unroll
  for (int n = 0; n < NT; ++n) cm[n][0] = cm[n][1] = 0.0;
  double inner = 0.0;
  const int ks = ld / 4;

  int cur = 0;
  for (; sI < nslabs && !dead; sI += stride, cur ^= 1) {
    double* buf = mine + cur * 8 * LDP;
    load_slab(sI + stride, mine + (cur ^ 1) * 8 * LDP);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const uint64_t row0 = a.lo + sI * 8;
    const int nrows = (a.hi - row0) < 8 ? (int)(a.hi - row0) : 8;
    if (a.solve) {
      double c[NT][2];
#pragma unroll
      for (int n = 0; n < NT; ++n) c[n][0] = c[n][1] = 0.0;
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        if (k < ks) {
          const int kc = 4 * k + t;
          const double av = (kc < R) ? buf[g * LDP + kc] : 0.0;
          const double* wrow = Ws + (size_t)kc * RP + g;
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma(c[n][0], c[n][1], av, wrow[n * 8]);
        }
      }
      // <M o tau, X> for this slab, then the solved rows replace the M rows
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double2 m2 = *reinterpret_cast<const double2*>(buf + g * LDP + n * 8 + 2 * t);
        const double2 t2 = *reinterpret_cast<const double2*>(taus + n * 8 + 2 * t);
        inner = fma(m2.x * t2.x, c[n][0], inner);
        inner = fma(m2.y * t2.y, c[n][1], inner);
        cm[n][0] = fmax(cm[n][0], fabs(c[n][0]));
        cm[n][1] = fmax(cm[n][1], fabs(c[n][1]));
      }
      __syncwarp();
#pragma unroll
      for (int n = 0; n < NT; ++n)
        *reinterpret_cast<double2*>(buf + g * LDP + n * 8 + 2 * t) = make_double2(c[n][0], c[n][1]);
      __syncwarp();
      double2* dst = reinterpret_cast<double2*>(a.A + row0 * ld);
      for (int e = lane; e < nrows * half; e += 32)
        dst[e] = *reinterpret_cast<const double2*>(buf + (e / half) * LDP + 2 * (e % half));
      for (int q = 0; q < a.peers.n; ++q) {  // fused all-gather: the peers' copies of the rows
        double2* pd = reinterpret_cast<double2*>(a.peers.p[q] + row0 * ld);
        for (int e = lane; e < nrows * half; e += 32)
          pd[e] = *reinterpret_cast<const double2*>(buf + (e / half) * LDP + 2 * (e % half));
      }
    } else {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double2 x2 = *reinterpret_cast<const double2*>(buf + g * LDP + n * 8 + 2 * t);
        cm[n][0] = fmax(cm[n][0], fabs(x2.x));
        cm[n][1] = fmax(cm[n][1], fabs(x2.y));
      }
    }
    // G~ += X^T X over the slab's 8 rows (rows past hi are zero)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      double f[NT];
#pragma unroll
      for (int b = 0; b < NT; ++b) f[b] = buf[(kk * 4 + t) * LDP + b * 8 + g];
      int p = 0;
#pragma unroll
      for (int bi = 0; bi < NT; ++bi)
#pragma unroll
        for (int bj = bi; bj < NT; ++bj, ++p) dmma(gacc[p][0], gacc[p][1], f[bi], f[bj]);
    }
    __syncwarp();  // the buffer is refilled two slabs later
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  // column max over the 8 row lanes (g), inner over the warp: fixed shuffle trees
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int o = 4; o <= 16; o <<= 1) cm[n][i] = fmax(cm[n][i], __shfl_xor_sync(0xffffffffu, cm[n][i], o));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) inner += __shfl_xor_sync(0xffffffffu, inner, o);

  // combine: every warp parks its raw fragments (NP x 32 lanes x 2 | RP colmax | inner) in
  // its own region of the (now dead) shared memory, then all threads sum each element over
  // the warps in fixed order and scatter it into the CTA partial (both triangles).
  constexpr int CL = NP * 64 + RP + 1, CLS = (CL + 1) & ~1;
  __syncthreads();
  double* park = sm + (size_t)warp * CLS;
#pragma unroll
  for (int p = 0; p < NP; ++p)
    *reinterpret_cast<double2*>(park + p * 64 + 2 * lane) = make_double2(gacc[p][0], gacc[p][1]);
  if (g == 0)
#pragma unroll
    for (int n = 0; n < NT; ++n)
      *reinterpret_cast<double2*>(park + NP * 64 + n * 8 + 2 * t) = make_double2(cm[n][0], cm[n][1]);
  if (lane == 0) park[NP * 64 + RP] = inner;
  __syncthreads();
  const size_t SL = (size_t)R * R + R + 1;
  double* out = a.part + (size_t)blockIdx.x * SL;
  for (int e = threadIdx.x; e < CL; e += blockDim.x) {
    const bool is_max = e >= NP * 64 && e < NP * 64 + RP;
    double v = sm[e];
    for (int w = 1; w < W; ++w) {
      const double x = sm[(size_t)w * CLS + e];
      v = is_max ? fmax(v, x) : v + x;
    }
    if (e < NP * 64) {
      int p = e >> 6, bi = 0;
      while (p >= NT - bi) { p -= NT - bi; ++bi; }
      const int bj = bi + p, ln = (e & 63) >> 1;
      const int r = bi * 8 + (ln >> 2), c2 = bj * 8 + 2 * (ln & 3) + (e & 1);
      if (r < R && c2 < R) {
        out[(size_t)r * R + c2] = v;
        if (bi != bj) out[(size_t)c2 * R + r] = v;
      }
    } else if (is_max) {
      const int c2 = e - NP * 64;
      if (c2 < R) out[(size_t)R * R + 1 + c2] = v;
    } else {
      out[(size_t)R * R] = v;
    }
  }
}

// stats[e] = fixed-order reduction over P partials: one warp per element, lane l sums
// partials l, l+32, ... then a fixed shuffle tree (sum; max for the colmax entries).
__device__ void lambda_gram_body(const double* st, int R, int first, double* lambda, double* G,
                                 double* inner_out, double* sig, double* lam);

__device__ __forceinline__ void reduce_stats_element(const double* __restrict__ part, int P,
                                                     int R, double* __restrict__ out, size_t e) {
  const size_t SL = (size_t)R * R + R + 1;
  const int lane = threadIdx.x & 31;
  const bool is_max = e > (size_t)R * R;
  double acc = 0.0;
  for (int p = lane; p < P; p += 32) {
    const double v = part[(size_t)p * SL + e];
    acc = is_max ? fmax(acc, v) : acc + v;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double v = __shfl_down_sync(0xffffffffu, acc, o);
    acc = is_max ? fmax(acc, v) : acc + v;
  }
  if (lane == 0) out[e] = acc;
}

__global__ void reduce_stats_kernel(const double* __restrict__ part, int P, int R,
                                    double* __restrict__ out, const int* conv) {
  if (conv && *conv) return;
  const size_t SL = (size_t)R * R + R + 1;
  const size_t e = blockIdx.x * (size_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (e >= SL) return;
  reduce_stats_element(part, P, R, out, e);
}

// reduce_stats_kernel + lambda_gram_kernel in one launch: the last CTA to finish its
// elements (atomic ticket after a fence) computes lambda / G_n / sig from the reduced
// statistics.  *ticket must be 0 on entry and is 0 again on exit.
__global__ void reduce_lambda_kernel(const double* __restrict__ part, int P, int R,
                                     double* __restrict__ out, int first, double* lambda,
                                     double* G, double* inner_out, double* sig,
                                     unsigned* ticket, const int* conv) {
  extern __shared__ double lam[];
  __shared__ bool last;
  if (conv && *conv) return;  // uniform: no block takes a ticket
  const size_t SL = (size_t)R * R + R + 1;
  const size_t e = blockIdx.x * (size_t)(blockDim.x / 32) + threadIdx.x / 32;
  if (e < SL) reduce_stats_element(part, P, R, out, e);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  lambda_gram_body(out, R, first, lambda, G, inner_out, sig, lam);
  if (threadIdx.x == 0) *ticket = 0u;
}

// a8 + a9 from the reduced statistics: lambda (iteration 1: 2-norm = sqrt(G~_rr); later
// max(1, colmax)), the normalised Gram G_n = G~ / (lambda lambda^T), the inner product, and
// the column scale sig_r = 1 / lambda_r (1 for a zero column) that maps the stored,
// unnormalised rows to the normalised factor (A_n = stored * diag(sig)): the rows are never
// rescaled in memory.  One CTA; lam: R doubles of shared memory.
__device__ void lambda_gram_body(const double* st, int R, int first, double* lambda, double* G,
                                 double* inner_out, double* sig, double* lam) {
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    // __ldcg: st may have been written by other CTAs of this launch (reduce_lambda_kernel)
    const double l = first ? sqrt(__ldcg(st + (size_t)r * R + r))
                           : fmax(1.0, __ldcg(st + (size_t)R * R + 1 + r));
    lam[r] = l;
    lambda[r] = l;
    if (sig) sig[r] = l > 0.0 ? 1.0 / l : 1.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int r = e / R, c = e % R;
    const double u = __ldcg(st + (size_t)min(r, c) * R + max(r, c));
    const double lr = lam[r] > 0.0 ? lam[r] : 1.0;
    const double lc = lam[c] > 0.0 ? lam[c] : 1.0;
    G[e] = u / (lr * lc);
  }
  if (threadIdx.x == 0 && inner_out) inner_out[0] = __ldcg(st + (size_t)R * R);
}

__global__ void lambda_gram_kernel(const double* __restrict__ st, int R, int first,
                                   double* __restrict__ lambda, double* __restrict__ G,
                                   double* inner_out, double* sig, const int* conv) {
  extern __shared__ double lam[];
  if (conv && *conv) return;
  lambda_gram_body(st, R, first, lambda, G, inner_out, sig, lam);
}

__global__ void gram_from_stats_kernel(const double* __restrict__ st, int R, double* G) {
  for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < R * R; e += blockDim.x * gridDim.x) {
    const int r = e / R, c = e % R;
    G[e] = st[(size_t)min(r, c) * R + max(r, c)];
  }
}

__global__ void scale_kernel(double* __restrict__ A, uint64_t lo, uint64_t hi, int R, int ld,
                             const double* __restrict__ lambda) {
  const uint64_t total = (hi - lo) * (uint64_t)ld;
  double* base = A + lo * ld;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % ld);
    if (r < R) {
      const double l = lambda[r];
      if (l > 0.0) base[e] = base[e] / l;
    }
  }
}

// fit_out = fit_hist + (it - 1).  With conv (tol > 0): skip once converged, and mark
// convergence (C-11: |fit_it - fit_{it-1}| < tol, it >= 2) by writing `it` to *conv.
__global__ void fit_kernel(const double* __restrict__ G_all, int N, int R,
                           const double* __restrict__ lambda, const double* inner,
                           const double* normx_sq, double* fit_out, int it, double tol,
                           int* conv) {
  __shared__ double sh[kThreads];
  if (conv && *conv) return;
  const int RR = R * R;
  double acc = 0.0;
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    double h = lambda[e / R] * lambda[e % R];
    for (int m = 0; m < N; ++m) h *= G_all[(size_t)m * RR + e];
    acc += h;
  }
  const double zz = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    const double nx = normx_sq[0];
    const double res = fmax(0.0, nx + zz - 2.0 * inner[0]);
    const double f = 1.0 - sqrt(res) / sqrt(nx);
    fit_out[0] = f;
    if (conv && it >= 2 && fabs(f - fit_out[-1]) < tol) *conv = it;
  }
}

// nu_r = ||A_n[:, r]|| of the normalised factor A_n = stored * diag(sig); the output rows
// are stored / d with d_r = (nu_r > 0 ? nu_r : 1) / sig_r, and lambda_r *= nu_r (C-12).
__global__ void fold_norms_kernel(const double* __restrict__ G, int R, double* lambda,
                                  double* d, const double* __restrict__ sig) {
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const double v = sqrt(G[(size_t)r * R + r]);
    d[r] = (v > 0.0 ? v : 1.0) / (sig ? sig[r] : 1.0);
    if (v > 0.0) lambda[r] *= v;
  }
}

__global__ void fill_kernel(double* __restrict__ p, size_t n, double v) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x)
    p[e] = v;
}

int grid_stride_blocks(splatt_ctx* ctx, uint64_t n) {
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n, kThreads),
                                                       (uint64_t)ctx->num_sms * 8));
}

}  // namespace

void init_factor(splatt_ctx* ctx, double* A, uint64_t I, int R, int ld, uint64_t seed,
                 uint64_t base) {
  init_factor_kernel<<<grid_stride_blocks(ctx, I * ld), kThreads, 0, ctx->stream>>>(A, I, R, ld,
                                                                                    seed, base);
  SB_CHECK_LAUNCH(ctx);
}

void norm_sq(splatt_ctx* ctx, const double* vals, uint64_t nnz, double* d_out) {
  const int P = std::min<int>(grid_stride_blocks(ctx, nnz), kThreads * 4);
  DevBuf<double> part(P, ctx->stream);
  sumsq_partial_kernel<<<P, kThreads, 0, ctx->stream>>>(vals, nnz, part.p);
  SB_CHECK_LAUNCH(ctx);
  sum_partials_kernel<<<1, kThreads, 0, ctx->stream>>>(part.p, P, d_out);
  SB_CHECK_LAUNCH(ctx);
}

void hadamard_inverse(splatt_ctx* ctx, const double* G_all, int N, int n, int R, int ld,
                      double* Vinv, int* status, const double* sig, double* tau,
                      cudaStream_t stream) {
  const size_t smem = ((size_t)R * R + 2 * R) * sizeof(double);
  set_max_dynamic_smem((const void*)hadamard_inverse_kernel, (128 * 128 + 2 * 128) * 8);
  hadamard_inverse_kernel<<<1, 1024, smem, stream ? stream : ctx->stream>>>(G_all, N, n, R, ld,
                                                                          Vinv, status, sig, tau,
                                                                          ctx->d_conv);
  SB_CHECK_LAUNCH(ctx);
}

namespace {

// Block size: 128 threads (4 CTAs/SM) while a CTA's threads cover every 4x4 Gram block pair
// (ld <= 60), else 256 (and 3 pairs per thread beyond 256 pairs, ld > 88).
template <int KB, int G, int BT>
void launch_rows(const RowsArgs& a, int P, size_t smem, cudaStream_t s) {
  set_max_dynamic_smem((const void*)solve_gram_kernel<KB, G, BT>, 200 * 1024);
  solve_gram_kernel<KB, G, BT><<<P, BT, smem, s>>>(a);
}

template <int KB, int BT>
void launch_rows_g(int G, const RowsArgs& a, int P, size_t smem, cudaStream_t s) {
  switch (G) {
    case 2: return launch_rows<KB, 2, BT>(a, P, smem, s);
    case 4: return launch_rows<KB, 4, BT>(a, P, smem, s);
    case 8: return launch_rows<KB, 8, BT>(a, P, smem, s);
    case 16: return launch_rows<KB, 16, BT>(a, P, smem, s);
    default: return launch_rows<KB, 32, BT>(a, P, smem, s);
  }
}

#ifndef SB_MMA_W
#define SB_MMA_W 8
#endif
constexpr int mma_warps(int NT) { return NT <= 5 ? SB_MMA_W : 8; }

template <int NT>
void launch_rows_mma_t(const RowsArgs& a, int P, size_t smem, cudaStream_t s) {
  constexpr int W = mma_warps(NT);
  set_max_dynamic_smem((const void*)solve_gram_mma_kernel<NT, W>, 220 * 1024);
  solve_gram_mma_kernel<NT, W><<<P, W * 32, smem, s>>>(a);
}

void launch_rows_mma(int NT, const RowsArgs& a, int P, size_t smem, cudaStream_t s) {
  switch (NT) {
    case 1: return launch_rows_mma_t<1>(a, P, smem, s);
    case 2: return launch_rows_mma_t<2>(a, P, smem, s);
    case 3: return launch_rows_mma_t<3>(a, P, smem, s);
    case 4: return launch_rows_mma_t<4>(a, P, smem, s);
    case 5: return launch_rows_mma_t<5>(a, P, smem, s);
    case 6: return launch_rows_mma_t<6>(a, P, smem, s);
    case 7: return launch_rows_mma_t<7>(a, P, smem, s);
    default: return launch_rows_mma_t<8>(a, P, smem, s);
  }
}

// Fixed-order reduction of the P per-CTA partials (with the lambda / G_n step fused when
// `fuse` is given).
void reduce_rows_stats(splatt_ctx* ctx, const double* part, int P, int R, double* stats,
                       const LambdaOut* fuse, cudaStream_t s) {
  const size_t SL = stats_len(R);
  const unsigned rblocks = (unsigned)ceil_div(SL, kThreads / 32);
  if (fuse) {
    reduce_lambda_kernel<<<rblocks, kThreads, R * sizeof(double), s>>>(
        part, P, R, stats, fuse->first ? 1 : 0, fuse->lambda, fuse->G_n, fuse->inner,
        fuse->sig, fuse->ticket, ctx->d_conv);
  } else {
    reduce_stats_kernel<<<rblocks, kThreads, 0, s>>>(part, P, R, stats, ctx->d_conv);
  }
  SB_CHECK_LAUNCH(ctx);
}

bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && *v != '0';
}

}  // namespace

void rows_solve_stats(splatt_ctx* ctx, const double* M, double* A, uint64_t lo, uint64_t hi,
                      int R, int ld, const double* Vinv, const double* tau, bool solve,
                      bool inner, const int* status, double* stats, const LambdaOut* fuse,
                      const RowsReduce* rr, const PeerRows* peers) {
  // Vinv: ld x ld, zero pads (hadamard_inverse)
  (void)inner;  // the inner product is always produced by the solve (it is free)
  const size_t SL = stats_len(R);
  cudaStream_t s = ctx->stream;
  if (hi <= lo) {
    SB_CUDA(cudaMemsetAsync(stats, 0, SL * sizeof(double), s));
    return;
  }
  // The fixed-order reduction of the per-CTA partials: on this stream, or (rr) on another
  // stream after an event, from rr's persistent partial buffer.
  auto reduce = [&](const double* part, int P) {
    if (rr && part == rr->part) {
      SB_CUDA(cudaEventRecord(rr->ev, s));
      SB_CUDA(cudaStreamWaitEvent(rr->stream, rr->ev, 0));
      if (rr->tm) {
        rr->tm->gap();  // the span starts once the solve is done, not at the last aux span
        rr->tm->begin(rr->cat);
      }
      reduce_rows_stats(ctx, part, P, R, stats, fuse, rr->stream);
      if (rr->tm) rr->tm->end();
    } else {
      reduce_rows_stats(ctx, part, P, R, stats, fuse, s);
    }
  };
  auto part_for = [&](DevBuf<double>& own, int P) -> double* {
    if (rr && (size_t)P * SL <= rr->cap) return rr->part;
    own.alloc((size_t)P * SL, s);
    return own.p;
  };
  const int ldp = ld + 2;
  const int slots = ld / 4;
  const int G = slots <= 2 ? 2 : slots <= 4 ? 4 : slots <= 8 ? 8 : slots <= 16 ? 16 : 32;
  const int nb = ld / 4, nbp = nb * (nb + 1) / 2;
  const int BT = nbp <= 128 ? 128 : 256;
  const int KB = nbp <= BT ? 1 : 3;
  const int S = nbp >= BT ? 1 : BT / nbp;
  const int T = (BT / G) * kRPG;
  // two tile buffers; the subset-combine buffer aliases them
  const size_t tile_doubles = std::max<size_t>(2 * (size_t)T * ldp, (size_t)S * nbp * 16);
  const size_t smem = (solve ? (size_t)ld * ld * 8 + (size_t)ld * 8 : 0) + tile_doubles * 8;
  RowsArgs a{};
  a.M = M;
  a.A = A;
  a.lo = lo;
  a.hi = hi;
  a.R = R;
  a.ld = ld;
  a.T = T;
  a.ntiles = ceil_div(hi - lo, T);
  a.Vinv = Vinv;
  a.tau = tau;
  a.status = status;
  a.conv = ctx->d_conv;
  a.solve = solve;
  if (peers && solve) a.peers = *peers;
#ifndef SB_SOLVE_MAX_PER_SM
#define SB_SOLVE_MAX_PER_SM 3
#endif
  const int max_res = std::min(SB_SOLVE_MAX_PER_SM,
                               KB == 1 ? (BT == 128 ? 4 : 2) : 1);  // __launch_bounds__
  const int per_sm =
      std::max<int>(1, std::min<int>(max_res, (int)((228 * 1024) / (smem + 2048))));
  const int P = (int)std::min<uint64_t>(a.ntiles, (uint64_t)ctx->num_sms * per_sm);
#ifndef SB_SOLVE_MMA
#define SB_SOLVE_MMA 1
#endif
  const int NT = (R + 7) / 8;
  if (SB_SOLVE_MMA && NT <= 8 && !getenv_flag("SPLATT_SOLVE_SIMT")) {
    // fp64 tensor-core path (solve_gram_mma_kernel): one CTA per SM
    const int W = mma_warps(NT);
    const int RP = 8 * NT, LDP = RP + 4;
    const size_t loop_d = (size_t)(solve ? ld : 0) * RP + RP + 2 + (size_t)W * 2 * 8 * LDP;
    const size_t park_d = (size_t)W * (NT * (NT + 1) / 2 * 64 + RP + 2);
    const size_t msmem = std::max(loop_d, park_d) * sizeof(double);
    const uint64_t nslabs = ceil_div(hi - lo, 8);
    a.ntiles = nslabs;
    const int Pm = (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(nslabs, W),
                                                                 (uint64_t)ctx->num_sms * mma_minb(NT)));
    ArenaScope scratch(current_arena() ? ctx->arena_scratch : nullptr, true);  // per-launch
    DevBuf<double> own;
    a.part = part_for(own, Pm);
    launch_rows_mma(NT, a, Pm, msmem, s);
    SB_CHECK_LAUNCH(ctx);
    reduce(a.part, Pm);
    return;
  }
  ArenaScope scratch(current_arena() ? ctx->arena_scratch : nullptr, true);  // per-launch
  DevBuf<double> own;
  a.part = part_for(own, P);
  if (BT == 128) launch_rows_g<1, 128>(G, a, P, smem, s);
  else if (KB == 1) launch_rows_g<1, 256>(G, a, P, smem, s);
  else launch_rows_g<3, 256>(G, a, P, smem, s);
  SB_CHECK_LAUNCH(ctx);
  reduce(a.part, P);
}

size_t rows_partials_cap(splatt_ctx* ctx, int R) {
  return (size_t)4 * ctx->num_sms * stats_len(R);  // every path's P <= 4 x SMs
}

void lambda_gram(splatt_ctx* ctx, const double* stats, int R, bool first, double* lambda,
                 double* G_n, double* inner_out, double* sig) {
  lambda_gram_kernel<<<1, kThreads, R * sizeof(double), ctx->stream>>>(stats, R, first ? 1 : 0,
                                                                       lambda, G_n, inner_out, sig,
                                                                       ctx->d_conv);
  SB_CHECK_LAUNCH(ctx);
}

void gram_from_stats(splatt_ctx* ctx, const double* stats, int R, double* G) {
  gram_from_stats_kernel<<<(unsigned)ceil_div((uint64_t)R * R, kThreads), kThreads, 0,
                           ctx->stream>>>(stats, R, G);
  SB_CHECK_LAUNCH(ctx);
}

void scale_columns(splatt_ctx* ctx, double* A, uint64_t lo, uint64_t hi, int R, int ld,
                   const double* lambda) {
  if (hi <= lo) return;
  scale_kernel<<<grid_stride_blocks(ctx, (hi - lo) * ld), kThreads, 0, ctx->stream>>>(A, lo, hi, R,
                                                                                      ld, lambda);
  SB_CHECK_LAUNCH(ctx);
}

void fit(splatt_ctx* ctx, const double* G_all, int N, int R, const double* lambda,
         const double* inner, const double* normx_sq, double* fit_out, int it, double tol,
         int* conv, cudaStream_t stream) {
  fit_kernel<<<1, kThreads, 0, stream ? stream : ctx->stream>>>(G_all, N, R, lambda, inner,
                                                                normx_sq, fit_out, it, tol, conv);
  SB_CHECK_LAUNCH(ctx);
}

void fill(splatt_ctx* ctx, double* p, size_t n, double v) {
  if (!n) return;
  fill_kernel<<<grid_stride_blocks(ctx, n), kThreads, 0, ctx->stream>>>(p, n, v);
  SB_CHECK_LAUNCH(ctx);
}

void fold_norms(splatt_ctx* ctx, const double* G_n, int R, double* lambda, double* d,
                const double* sig) {
  fold_norms_kernel<<<1, kThreads, 0, ctx->stream>>>(G_n, R, lambda, d, sig);
  SB_CHECK_LAUNCH(ctx);
}

}  // namespace sb
