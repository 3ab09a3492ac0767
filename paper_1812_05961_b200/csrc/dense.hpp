// dense.hpp — the small fp64 steps around MTTKRP.
#pragma once
#include "ctx.hpp"

namespace sb {

// Layout of the per-mode statistics vector (all doubles), reduced over rows (and over
// ranks with comm): [0, R*R) Gram of the unnormalised rows (symmetric), [R*R] inner
// product sum M .* A, [R*R+1, R*R+1+R) column max |a|.  The first R*R+1 entries are
// sums, the last R maxima, so one all-reduce of each kind combines ranks.
inline size_t stats_len(int R) { return (size_t)R * R + R + 1; }
inline size_t stats_sum_len(int R) { return (size_t)R * R + 1; }
inline size_t stats_max_off(int R) { return (size_t)R * R + 1; }

// a3: A[i, r] = u(seed, base + i*R + r) for r < R (counter-based splitmix64), pads 0.
void init_factor(splatt_ctx* ctx, double* A, uint64_t I, int R, int ld, uint64_t seed,
                 uint64_t base);

// sum of squares of vals (deterministic two-pass reduction) into d_out[0].
void norm_sq(splatt_ctx* ctx, const double* vals, uint64_t nnz, double* d_out);

// a5 + a7 (factor): V = *_{m != n} G_m (ascending m) and V^-1 (Alg. 1 line 5's
// V^dagger) by Gauss-Jordan elimination without pivoting, whose pivots are the Cholesky
// pivots squared: the C-7 test (pivot <= 1e-12 * max diag) and one 1e-12*trace/R ridge
// retry apply as stated.  G_all: N x R*R.  Vinv: ld x ld (symmetric, zero pads).
// status: set to 1 on failure (never cleared here; Vinv then unwritten).
// The factors are stored unnormalised: A_m = stored_m * diag(sig_m) (sig: N x R, or NULL =
// all ones).  The kernel also forms tau = prod_{m != n} sig_m (written to tau, R) and
// returns Vinv with row i scaled by tau_i, so that x = m_stored Vinv = (m o tau) V^-1.
// Launched on `stream` (default: the context stream).
void hadamard_inverse(splatt_ctx* ctx, const double* G_all, int N, int n, int R, int ld,
                      double* Vinv, int* status, const double* sig, double* tau,
                      cudaStream_t stream = nullptr);

// Outputs of the lambda step when fused into the statistics reduction (see lambda_gram).
struct LambdaOut {
  bool first;
  double* lambda;   // R
  double* G_n;      // R x R
  double* inner;    // 1
  double* sig;      // R: 1 / lambda (1 for a zero column)
  unsigned* ticket; // device counter, 0 on entry and on exit
};

// a7 (solve) + a9/a8/a10 partials: for rows [lo, hi): if solve, A[i,:] = M[i,:] V^-1
// (row times the symmetric inverse from hadamard_inverse, ld x ld); then accumulate the Gram of
// the rows, the column max |A| and (if inner) sum M .* A.  Reduced to stats
// (stats_len(R)).  If !solve, M is ignored and A is only read.  Skipped when *status != 0.
// tau: R column scales of M (from hadamard_inverse; used for <M, A>), NULL when !solve.
// fuse: if non-NULL the reduction kernel also performs lambda_gram (single-rank path).
// rr: run the reduction (and the fused lambda step) on rr->stream after an event recorded
// behind the solve, from the persistent partial buffer rr->part (cap doubles, at least
// rows_partials_cap), so the next MTTKRP on the context stream does not wait for it.  The
// caller orders later users of `stats` / the fused outputs and of rr->part after rr->stream.
struct RowsReduce {
  cudaStream_t stream;
  cudaEvent_t ev;
  double* part;
  size_t cap;
  EventTimer* tm;  // optional span on rr->stream
  int cat;
};
// peers (SPLATT_XCHG_PEER, splatt_b200.h): the other ranks' copies of A; every solved row is
// also stored at the same offset of each (the all-gather of §8(e) step 5 fused into the
// solve: remote stores from inside the kernel, slab by slab).
struct PeerRows {
  double* p[kMaxPeerRanks - 1];
  int n;
};
void rows_solve_stats(splatt_ctx* ctx, const double* M, double* A, uint64_t lo, uint64_t hi,
                      int R, int ld, const double* Vinv, const double* tau, bool solve,
                      bool inner, const int* status, double* stats,
                      const LambdaOut* fuse = nullptr, const RowsReduce* rr = nullptr,
                      const PeerRows* peers = nullptr);
size_t rows_partials_cap(splatt_ctx* ctx, int R);

// a8 + a9: lambda (first: 2-norm = sqrt(G~_rr); else max(1, colmax)), G_n =
// G~ / (lambda lambda^T) (mirrored), inner_out = stats inner, sig = 1 / lambda (the
// stored rows are not rescaled: A_n = stored * diag(sig)).
void lambda_gram(splatt_ctx* ctx, const double* stats, int R, bool first, double* lambda,
                 double* G_n, double* inner_out, double* sig);

// p[0..n) = v.
void fill(splatt_ctx* ctx, double* p, size_t n, double v);

// Mirror the upper Gram of stats into G (R x R) — initial Grams.
void gram_from_stats(splatt_ctx* ctx, const double* stats, int R, double* G);

// A[i, r] /= lambda[r] for lambda[r] > 0, rows [lo, hi).
void scale_columns(splatt_ctx* ctx, double* A, uint64_t lo, uint64_t hi, int R, int ld,
                   const double* lambda);

// a10: fit = 1 - sqrt(max(0, nx + zz - 2 inner)) / sqrt(nx), zz = lambda^T (*_m G_m) lambda.
// fit_out = the iteration's entry of the fit history (it >= 1).  conv (or NULL): device int,
// skip when set, else set to `it` when it >= 2 and |fit - previous fit| < tol (C-11).
void fit(splatt_ctx* ctx, const double* G_all, int N, int R, const double* lambda,
         const double* inner, const double* normx_sq, double* fit_out, int it, double tol,
         int* conv, cudaStream_t stream = nullptr);

// a11 (finalise one mode): nu_r = sqrt(G_n[r,r]); lambda_r *= nu_r (if > 0); d_r =
// (nu_r > 0 ? nu_r : 1) / sig_r is the divisor that turns the stored rows into the output.
void fold_norms(splatt_ctx* ctx, const double* G_n, int R, double* lambda, double* d,
                const double* sig);

}  // namespace sb
