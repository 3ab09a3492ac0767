// dense.cu — the small fp64 kernels of each ALS mode update.
//
// Alg. 1 per mode n: V = *_{m!=n} G_m (line 4), A_n = M V^dagger
// (line 5, realised as potrf/potrs), normalise columns into lambda
// (line 6), Gram refresh, and the fit (line 13).  Readings: DESIGN.md §2 (C-7 pivot
// threshold / ridge, C-8 norm schedule, C-10 fit identity).
//
// Fusion: the row solve reads each M row once from HBM and, while
// the solved rows are still in shared memory, accumulates the partial Gram, the
// column max |a| and the fit inner product, so lambda / G_n / the fit need no
// further pass over A except the final column scaling.  Reductions run in a fixed
// order (per-CTA partials, then a fixed-order sum), so results are deterministic.
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

// One CTA.  smem: W (R*R) = V; L is built in W's lower triangle while the strict upper
// triangle keeps V (V is exactly symmetric), and diag keeps V's diagonal for the retry.
__global__ void hadamard_cholesky_kernel(const double* __restrict__ G_all, int N, int n, int R,
                                         double* __restrict__ L, int* status) {
  extern __shared__ double sm[];
  double* W = sm;
  double* diag = sm + R * R;
  __shared__ int failed;
  __shared__ double thr, ridge;
  const int RR = R * R;
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    double p = 1.0;
    bool first = true;
    for (int m = 0; m < N; ++m) {
      if (m == n) continue;
      const double g = G_all[(size_t)m * RR + e];
      p = first ? g : p * g;
      first = false;
    }
    W[e] = p;
    if (e / R == e % R) diag[e / R] = p;
  }
  __syncthreads();
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (threadIdx.x == 0) {
      failed = 0;
      if (attempt == 1) {
        double tr = 0.0;
        for (int j = 0; j < R; ++j) tr += diag[j];
        ridge = 1e-12 * tr / R;
      } else {
        ridge = 0.0;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < RR; e += blockDim.x) {
      const int i = e / R, j = e % R;
      if (i == j) W[e] = diag[i] + ridge;
      else if (i > j) W[e] = W[j * R + i];  // restore the lower triangle from the upper
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = 0.0;
      for (int j = 0; j < R; ++j) mx = fmax(mx, W[j * R + j]);
      thr = 1e-12 * mx;
    }
    __syncthreads();
    for (int j = 0; j < R; ++j) {
      if (threadIdx.x == 0) {
        double d = W[j * R + j];
        for (int k = 0; k < j; ++k) d -= W[j * R + k] * W[j * R + k];
        if (d > thr) W[j * R + j] = sqrt(d);
        else failed = 1;
      }
      __syncthreads();
      if (failed) break;
      const double piv = W[j * R + j];
      for (int i = j + 1 + threadIdx.x; i < R; i += blockDim.x) {
        double s = W[i * R + j];
        for (int k = 0; k < j; ++k) s -= W[i * R + k] * W[j * R + k];
        W[i * R + j] = s / piv;
      }
      __syncthreads();
    }
    if (!failed) {
      for (int e = threadIdx.x; e < RR; e += blockDim.x)
        L[e] = (e % R <= e / R) ? W[e] : 0.0;
      return;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *status = 1;
}

struct RowsArgs {
  const double* M;
  double* A;
  uint64_t lo, hi;
  int R, ld, ldp, T;
  uint64_t ntiles;
  const double* L;
  const int* status;
  double* part;  // gridDim.x x stats_len(R)
  bool solve, inner;
};

// Block pair q of the upper block triangle of an nb x nb grid of 4x4 blocks.
__device__ __forceinline__ void block_pair(int q, int nb, int& rb, int& cb) {
  int r = 0;
  while (q >= nb - r) { q -= nb - r; ++r; }
  rb = r;
  cb = r + q;
}

constexpr int kMaxBP = 3;  // ceil(528 / 256) block pairs per thread for R <= 128

__global__ void __launch_bounds__(kThreads) rows_kernel(const RowsArgs a) {
  extern __shared__ double sm[];
  __shared__ double red[kThreads];
  const int R = a.R, ld = a.ld, ldp = a.ldp;
  const size_t SL = (size_t)R * R + R + 1;
  double* part = a.part + (size_t)blockIdx.x * SL;
  if (a.status && *a.status) {
    for (size_t e = threadIdx.x; e < SL; e += blockDim.x) part[e] = 0.0;
    return;
  }
  double* Ls = sm;
  double* tile = sm + (a.solve ? R * R : 0);
  if (a.solve)
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) Ls[e] = a.L[e];
  const int nb = ld / 4;
  const int nbp = nb * (nb + 1) / 2;
  int rb[kMaxBP], cb[kMaxBP];
  double g[kMaxBP][16];
#pragma unroll
  for (int k = 0; k < kMaxBP; ++k) {
    const int q = threadIdx.x + k * blockDim.x;
    rb[k] = cb[k] = -1;
    if (q < nbp) block_pair(q, nb, rb[k], cb[k]);
#pragma unroll
    for (int z = 0; z < 16; ++z) g[k][z] = 0.0;
  }
  double cmax = 0.0, inner = 0.0;
  const double* src = a.solve ? a.M : a.A;
  for (uint64_t tI = blockIdx.x; tI < a.ntiles; tI += gridDim.x) {
    const uint64_t row0 = a.lo + tI * a.T;
    const uint64_t left = a.hi - row0;
    const int nrows = left < (uint64_t)a.T ? (int)left : a.T;
    __syncthreads();
    for (int e = threadIdx.x; e < nrows * ld; e += blockDim.x) {
      const int r = e / ld, c = e % ld;
      tile[r * ldp + c] = src[(row0 + r) * ld + c];
    }
    __syncthreads();
    if (a.solve) {
      if ((int)threadIdx.x < nrows) {
        double* x = tile + threadIdx.x * ldp;
        for (int j = 0; j < R; ++j) {          // L y = m
          double s = x[j];
          for (int k = 0; k < j; ++k) s -= Ls[j * R + k] * x[k];
          x[j] = s / Ls[j * R + j];
        }
        for (int j = R - 1; j >= 0; --j) {     // L^T x = y
          double s = x[j];
          for (int k = j + 1; k < R; ++k) s -= Ls[k * R + j] * x[k];
          x[j] = s / Ls[j * R + j];
        }
      }
      __syncthreads();
      for (int e = threadIdx.x; e < nrows * ld; e += blockDim.x) {
        const int r = e / ld, c = e % ld;
        const double x = (c < R) ? tile[r * ldp + c] : 0.0;
        a.A[(row0 + r) * ld + c] = x;
        if (a.inner && c < R) inner = fma(a.M[(row0 + r) * ld + c], x, inner);
      }
    }
#pragma unroll
    for (int k = 0; k < kMaxBP; ++k) {
      if (rb[k] < 0) continue;
      const int c0 = 4 * rb[k], c1 = 4 * cb[k];
      for (int r = 0; r < nrows; ++r) {
        const double* row = tile + r * ldp;
        double u[4], w[4];
#pragma unroll
        for (int z = 0; z < 4; ++z) { u[z] = row[c0 + z]; w[z] = row[c1 + z]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) g[k][i * 4 + j] = fma(u[i], w[j], g[k][i * 4 + j]);
      }
    }
    if ((int)threadIdx.x < R)
      for (int r = 0; r < nrows; ++r) cmax = fmax(cmax, fabs(tile[r * ldp + threadIdx.x]));
  }
  // Per-CTA partials: symmetric Gram, colmax, inner.
#pragma unroll
  for (int k = 0; k < kMaxBP; ++k) {
    if (rb[k] < 0) continue;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        const int r = 4 * rb[k] + i, s = 4 * cb[k] + j;
        if (r < R && s < R && r <= s) {
          part[(size_t)r * R + s] = g[k][i * 4 + j];
          part[(size_t)s * R + r] = g[k][i * 4 + j];
        }
      }
  }
  if ((int)threadIdx.x < R) part[(size_t)R * R + 1 + threadIdx.x] = cmax;
  const double tot = block_sum(inner, red);
  if (threadIdx.x == 0) part[(size_t)R * R] = tot;
}

__global__ void reduce_stats_kernel(const double* __restrict__ part, int P, int R,
                                    double* __restrict__ out) {
  const size_t SL = (size_t)R * R + R + 1;
  const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (e >= SL) return;
  const bool is_max = e > (size_t)R * R;
  double acc = 0.0;
  for (int p = 0; p < P; ++p) {
    const double v = part[(size_t)p * SL + e];
    acc = is_max ? fmax(acc, v) : acc + v;
  }
  out[e] = acc;
}

__global__ void lambda_gram_kernel(const double* __restrict__ st, int R, int first,
                                   double* __restrict__ lambda, double* __restrict__ G,
                                   double* inner_out) {
  extern __shared__ double lam[];
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const double l = first ? sqrt(st[(size_t)r * R + r]) : fmax(1.0, st[(size_t)R * R + 1 + r]);
    lam[r] = l;
    lambda[r] = l;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int r = e / R, s = e % R;
    const double u = st[(size_t)min(r, s) * R + max(r, s)];
    const double lr = lam[r] > 0.0 ? lam[r] : 1.0;
    const double ls = lam[s] > 0.0 ? lam[s] : 1.0;
    G[e] = u / (lr * ls);
  }
  if (threadIdx.x == 0 && inner_out) inner_out[0] = st[(size_t)R * R];
}

__global__ void gram_from_stats_kernel(const double* __restrict__ st, int R, double* G) {
  for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < R * R; e += blockDim.x * gridDim.x) {
    const int r = e / R, s = e % R;
    G[e] = st[(size_t)min(r, s) * R + max(r, s)];
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

__global__ void fit_kernel(const double* __restrict__ G_all, int N, int R,
                           const double* __restrict__ lambda, const double* inner,
                           const double* normx_sq, double* fit_out) {
  __shared__ double sh[kThreads];
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
    fit_out[0] = 1.0 - sqrt(res) / sqrt(nx);
  }
}

__global__ void fold_norms_kernel(const double* __restrict__ G, int R, double* lambda,
                                  double* nu) {
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const double v = sqrt(G[(size_t)r * R + r]);
    nu[r] = v;
    if (v > 0.0) lambda[r] *= v;
  }
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

void hadamard_cholesky(splatt_ctx* ctx, const double* G_all, int N, int n, int R, double* L,
                       int* status) {
  const size_t smem = ((size_t)R * R + R) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    SB_CUDA(cudaFuncSetAttribute(hadamard_cholesky_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (128 * 128 + 128) * 8));
    attr_set = true;
  }
  hadamard_cholesky_kernel<<<1, kThreads, smem, ctx->stream>>>(G_all, N, n, R, L, status);
  SB_CHECK_LAUNCH(ctx);
}

void rows_solve_stats(splatt_ctx* ctx, const double* M, double* A, uint64_t lo, uint64_t hi,
                      int R, int ld, const double* L, bool solve, bool inner, const int* status,
                      double* stats) {
  const size_t SL = stats_len(R);
  if (hi <= lo) {
    SB_CUDA(cudaMemsetAsync(stats, 0, SL * sizeof(double), ctx->stream));
    return;
  }
  const int ldp = ld + 1;
  const size_t budget = 200 * 1024;
  const size_t lbytes = solve ? (size_t)R * R * 8 : 0;
  int T = (int)std::min<size_t>(256, (budget - lbytes) / ((size_t)ldp * 8));
  T = std::max(32, T / 32 * 32);
  const size_t smem = lbytes + (size_t)T * ldp * 8;
  static bool attr_set = false;
  if (!attr_set) {
    SB_CUDA(cudaFuncSetAttribute(rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(budget + 8 * 1024)));
    attr_set = true;
  }
  RowsArgs a{};
  a.M = M;
  a.A = A;
  a.lo = lo;
  a.hi = hi;
  a.R = R;
  a.ld = ld;
  a.ldp = ldp;
  a.T = T;
  a.ntiles = ceil_div(hi - lo, T);
  a.L = L;
  a.status = status;
  a.solve = solve;
  a.inner = inner;
  const int per_sm = std::max<int>(1, (int)((228 * 1024) / (smem + 2048)));
  const int P = (int)std::min<uint64_t>(a.ntiles, (uint64_t)ctx->num_sms * std::min(per_sm, 2));
  DevBuf<double> part((size_t)P * SL, ctx->stream);
  a.part = part.p;
  rows_kernel<<<P, kThreads, smem, ctx->stream>>>(a);
  SB_CHECK_LAUNCH(ctx);
  reduce_stats_kernel<<<(unsigned)ceil_div(SL, kThreads), kThreads, 0, ctx->stream>>>(part.p, P, R,
                                                                                     stats);
  SB_CHECK_LAUNCH(ctx);
}

void lambda_gram(splatt_ctx* ctx, const double* stats, int R, bool first, double* lambda,
                 double* G_n, double* inner_out) {
  lambda_gram_kernel<<<1, kThreads, R * sizeof(double), ctx->stream>>>(stats, R, first ? 1 : 0,
                                                                       lambda, G_n, inner_out);
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
         const double* inner, const double* normx_sq, double* fit_out) {
  fit_kernel<<<1, kThreads, 0, ctx->stream>>>(G_all, N, R, lambda, inner, normx_sq, fit_out);
  SB_CHECK_LAUNCH(ctx);
}

void fold_norms(splatt_ctx* ctx, const double* G_n, int R, double* lambda, double* nu) {
  fold_norms_kernel<<<1, kThreads, 0, ctx->stream>>>(G_n, R, lambda, nu);
  SB_CHECK_LAUNCH(ctx);
}

}  // namespace sb
