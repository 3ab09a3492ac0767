/*
 * oracle.cpp — plain, slow, obviously-correct CPU CP-ALS over COO (TEST INFRASTRUCTURE).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1812_05961_b200/).
 *
 * Every function follows one step of the method as stated in the paper
 * (arXiv 1812.05961, /root/reference/PAPER.md) and the readings fixed in
 * SURVEY.md §8(c) (C-1..C-14, Q-1..Q-24), restated in DESIGN.md §2:
 *
 *   C-2  init           PAPER.md:191 (Alg. 1 line 2 "initialize A^(n)")
 *   C-3  ||X||^2        PAPER.md:202 (fit, line 13) — plain sum of squares
 *   C-4  Gram A^T A     PAPER.md:193 (Alg. 1 line 4), realised with syrk
 *   C-6  V, MTTKRP      PAPER.md:182-185, 193-200 (Alg. 1 lines 4-11) — DEFINITION:
 *                       M[i,r] = sum_{p: ind_n[p]=i} v_p prod_{m!=n} A_m[ind_m[p], r]
 *   C-7  solve          PAPER.md:194, 387 (V^dagger realised as potrf + potrs)
 *   C-8  normalise      PAPER.md:195 (line 6 "normalize columns ... storing norms as lambda")
 *   C-10 fit            PAPER.md:202, 404 (line 13; formula: SURVEY.md Q-5)
 *   C-11 convergence    PAPER.md:202 ("until fit ceases to improve or max iterations")
 *   C-12 finalise       PAPER.md:203 (line 14 "return lambda, A^(1..3)")
 *   C-13 CSF            PAPER.md:215-218 (compressed sparse fiber tree)
 *   C-14 partition      SURVEY.md §8(e) (optimal contiguous slice split)
 *   C-15 CSF policy     SPEC.md:128-136 (ONE / TWO / ALL allocations)
 *
 * Numbers: fp64 throughout.  Parallelism (OpenMP) only over
 * independent outputs whose own summation order is fixed, so every result is
 * bitwise independent of the thread count.
 *
 * Parity pins for each function live in tests/test_oracle_pins.py (see the header
 * of that file); none of them calls back into this file's arithmetic.
 */
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

enum { OR_OK = 0, OR_BADINPUT = -1, OR_SINGULAR = -3, OR_EMPTY = -6 };

/* ---------------------------------------------------------------- C-2 init */
/* splitmix64 finaliser (public domain, Steele/Lea/Flood) applied to the counter
 * s + (k+1)*gamma; u = top 53 bits * 2^-53.  SURVEY.md §8(c) C-2, Q-7.          */
static uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t oracle_splitmix64_raw(uint64_t seed, uint64_t k) {
    return or_mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ULL);
}
double oracle_u01(uint64_t seed, uint64_t k) {
    return (double)(oracle_splitmix64_raw(seed, k) >> 11) * (1.0 / 9007199254740992.0);
}
/* A_n[i,r] = u(seed, sum_{m<n} I_m R + i R + r), row-major, ld = R. */
void oracle_init_factors(int N, const uint64_t* dims, int R, uint64_t seed, double** A) {
    uint64_t base = 0;
    for (int n = 0; n < N; ++n) {
        for (uint64_t i = 0; i < dims[n]; ++i)
            for (int r = 0; r < R; ++r)
                A[n][i * R + r] = oracle_u01(seed, base + i * (uint64_t)R + (uint64_t)r);
        base += dims[n] * (uint64_t)R;
    }
}

/* ------------------------------------------------------------- C-1 validate */
int oracle_validate(int N, const uint64_t* dims, uint64_t nnz, const uint32_t* const* ind) {
    if (N < 3 || N > 8 || nnz == 0) return OR_BADINPUT;
    for (int m = 0; m < N; ++m) {
        if (dims[m] == 0 || dims[m] >= (1ULL << 32)) return OR_BADINPUT;
        for (uint64_t p = 0; p < nnz; ++p)
            if (ind[m][p] >= dims[m]) return OR_BADINPUT;
    }
    return OR_OK;
}

/* ---------------------------------------------------------------- C-3 ||X||^2 */
double oracle_norm_sq(uint64_t nnz, const double* vals) {
    double s = 0.0;
    for (uint64_t p = 0; p < nnz; ++p) s += vals[p] * vals[p];
    return s;
}

/* ------------------------------------------------------------------ C-4 Gram */
/* G = A^T A; upper triangle summed over i ascending, then mirrored (exactly
 * symmetric).  Parallel over (r,s) pairs only.                  */
void oracle_gram(uint64_t I, int R, const double* A, double* G) {
    const int npairs = R * (R + 1) / 2;
#pragma omp parallel for schedule(dynamic, 1)
    for (int q = 0; q < npairs; ++q) {
        int r = 0, rem = q;
        while (rem >= R - r) { rem -= R - r; ++r; }
        const int s = r + rem;
        double acc = 0.0;
        for (uint64_t i = 0; i < I; ++i) acc += A[i * R + r] * A[i * R + s];
        G[r * R + s] = acc;
        G[s * R + r] = acc;
    }
}

/* V = *_{m != n} G_m, Hadamard product in ascending m (Alg. 1 line 4). */
void oracle_hadamard_except(int N, int R, const double* const* G, int n, double* V) {
    bool first = true;
    for (int m = 0; m < N; ++m) {
        if (m == n) continue;
        for (int e = 0; e < R * R; ++e) V[e] = first ? G[m][e] : V[e] * G[m][e];
        first = false;
    }
}

/* -------------------------------------------------------------- C-6 MTTKRP */
/* Group nonzeros by their mode-n index: stable counting sort of positions p by
 * ind_n[p].  (The oracle's "Sort"; PAPER.md:415 only fixes that some sort happens.)
 * row_ptr has I_n+1 entries, order has nnz entries; within a row p ascends.    */
void oracle_group_by_mode(uint64_t nnz, const uint32_t* ind_n, uint64_t I_n,
                          uint64_t* row_ptr, uint64_t* order) {
    std::fill(row_ptr, row_ptr + I_n + 1, 0);
    for (uint64_t p = 0; p < nnz; ++p) row_ptr[(uint64_t)ind_n[p] + 1]++;
    for (uint64_t i = 0; i < I_n; ++i) row_ptr[i + 1] += row_ptr[i];
    std::vector<uint64_t> next(row_ptr, row_ptr + I_n);
    for (uint64_t p = 0; p < nnz; ++p) order[next[ind_n[p]]++] = p;
}

/* M[i,r] = sum_{p: ind_n[p] = i, p ascending} ((v_p * A_{m1}[.,r]) * A_{m2}[.,r]) ...
 * with m1 < m2 < ... != n.  Rows with no nonzeros are 0.  Factors have ld = R. */
static void mttkrp_grouped(int N, uint64_t I_n, const uint32_t* const* ind, const double* vals,
                           int n, int R, const double* const* A, const uint64_t* row_ptr,
                           const uint64_t* order, double* M) {
#pragma omp parallel
    {
        std::vector<double> acc(R), t(R);
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < (int64_t)I_n; ++i) {
            std::fill(acc.begin(), acc.end(), 0.0);
            for (uint64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
                const uint64_t p = order[q];
                for (int r = 0; r < R; ++r) t[r] = vals[p];
                for (int m = 0; m < N; ++m) {
                    if (m == n) continue;
                    const double* row = A[m] + (uint64_t)ind[m][p] * R;
                    for (int r = 0; r < R; ++r) t[r] = t[r] * row[r];
                }
                for (int r = 0; r < R; ++r) acc[r] += t[r];
            }
            for (int r = 0; r < R; ++r) M[(uint64_t)i * R + r] = acc[r];
        }
    }
}

int oracle_mttkrp(int N, const uint64_t* dims, uint64_t nnz, const uint32_t* const* ind,
                  const double* vals, int n, int R, const double* const* A, double* M) {
    if (n < 0 || n >= N || R < 1) return OR_BADINPUT;
    std::vector<uint64_t> row_ptr(dims[n] + 1), order(nnz);
    oracle_group_by_mode(nnz, ind[n], dims[n], row_ptr.data(), order.data());
    mttkrp_grouped(N, dims[n], ind, vals, n, R, A, row_ptr.data(), order.data(), M);
    return OR_OK;
}

/* --------------------------------------------------------------- C-7 solve */
/* Cholesky-Banachiewicz V = L L^T (no pivoting).  A pivot d_j <= 1e-12 * max_j V_jj
 * fails.  Returns 0 on success.                               */
static int cholesky(int R, const double* V, double* L) {
    double maxd = 0.0;
    for (int j = 0; j < R; ++j) maxd = std::max(maxd, V[j * R + j]);
    const double thr = 1e-12 * maxd;
    std::fill(L, L + R * R, 0.0);
    for (int j = 0; j < R; ++j) {
        for (int k = 0; k < j; ++k) {
            double s = V[j * R + k];
            for (int m = 0; m < k; ++m) s -= L[j * R + m] * L[k * R + m];
            L[j * R + k] = s / L[k * R + k];
        }
        double d = V[j * R + j];
        for (int k = 0; k < j; ++k) d -= L[j * R + k] * L[j * R + k];
        if (!(d > thr)) return -1;
        L[j * R + j] = std::sqrt(d);
    }
    return 0;
}

/* Factor V (with one ridge retry: V + (1e-12 trace(V)/R) I), then per
 * row of M solve x V = m: forward with L, back with L^T.  X may alias M.          */
int oracle_cholesky_solve(int R, const double* V, uint64_t I, const double* M, double* X) {
    std::vector<double> L(R * R), W(V, V + R * R);
    if (cholesky(R, W.data(), L.data()) != 0) {
        double tr = 0.0;
        for (int j = 0; j < R; ++j) tr += V[j * R + j];
        const double ridge = 1e-12 * tr / R;
        for (int j = 0; j < R; ++j) W[j * R + j] += ridge;
        if (cholesky(R, W.data(), L.data()) != 0) return OR_SINGULAR;
    }
#pragma omp parallel
    {
        std::vector<double> y(R);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < (int64_t)I; ++i) {
            const double* m = M + (uint64_t)i * R;
            for (int j = 0; j < R; ++j) {            /* L y = m */
                double s = m[j];
                for (int k = 0; k < j; ++k) s -= L[j * R + k] * y[k];
                y[j] = s / L[j * R + j];
            }
            double* x = X + (uint64_t)i * R;
            for (int j = R - 1; j >= 0; --j) {       /* L^T x = y */
                double s = y[j];
                for (int k = j + 1; k < R; ++k) s -= L[k * R + j] * x[k];
                x[j] = s / L[j * R + j];
            }
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------ C-8 normalise */
/* which = 0: 2-norm (iteration 1): lambda_r = sqrt(sum_i A[i,r]^2); divide if > 0.
 * which = 1: max-norm (later):     lambda_r = max(1, max_i |A[i,r]|); divide.     */
void oracle_normalize(uint64_t I, int R, double* A, int which, double* lambda) {
    for (int r = 0; r < R; ++r) {
        double l;
        if (which == 0) {
            double s = 0.0;
            for (uint64_t i = 0; i < I; ++i) s += A[i * R + r] * A[i * R + r];
            l = std::sqrt(s);
        } else {
            double mx = 0.0;
            for (uint64_t i = 0; i < I; ++i) mx = std::max(mx, std::fabs(A[i * R + r]));
            l = std::max(1.0, mx);
        }
        lambda[r] = l;
        if (l > 0.0)
            for (uint64_t i = 0; i < I; ++i) A[i * R + r] /= l;
    }
}

/* ----------------------------------------------------------------- C-10 fit */
/* ||Z||^2 = sum_{r,s} lambda_r lambda_s prod_m G_m[r,s];
 * <X,Z>  = sum_r lambda_r sum_i M[i,r] A[i,r]  (M, A of the last mode);
 * fit = 1 - sqrt(max(0, ||X||^2 + ||Z||^2 - 2<X,Z>)) / sqrt(||X||^2).            */
double oracle_fit(int N, int R, const double* const* G, const double* lambda, uint64_t I_last,
                  const double* M_last, const double* A_last, double normx_sq) {
    double zz = 0.0;
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < R; ++s) {
            double h = lambda[r] * lambda[s];
            for (int m = 0; m < N; ++m) h *= G[m][r * R + s];
            zz += h;
        }
    double xz = 0.0;
    for (int r = 0; r < R; ++r) {
        double c = 0.0;
        for (uint64_t i = 0; i < I_last; ++i) c += M_last[i * R + r] * A_last[i * R + r];
        xz += lambda[r] * c;
    }
    const double res = std::max(0.0, normx_sq + zz - 2.0 * xz);
    return 1.0 - std::sqrt(res) / std::sqrt(normx_sq);
}

/* ------------------------------------------------------------ C-5 the loop */
/* timings (may be NULL), seconds: [0] MTTKRP, [1] Sort (grouping), [2] Mat A^TA,
 * [3] Mat norm, [4] CPD fit, [5] Inverse, [6] total loop  (Table III categories,
 * PAPER.md:404).                                                                  */
int oracle_cpd_als(int N, const uint64_t* dims, uint64_t nnz, const uint32_t* const* ind,
                   const double* vals, int R, int max_iters, double tol, uint64_t seed,
                   const double* const* init, double** A /* out, ld = R */, double* lambda,
                   double* fit_history, int* iters_out, double* fit_out, double* timings) {
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double>(b - a).count();
    };
    double tm[7] = {0, 0, 0, 0, 0, 0, 0};
    int st = oracle_validate(N, dims, nnz, ind);                       /* C-1 */
    if (st != OR_OK) return st;
    if (R < 1 || R > 128 || max_iters < 1 || !(tol >= 0.0)) return OR_BADINPUT;
    const double normx_sq = oracle_norm_sq(nnz, vals);                /* C-3 */
    if (!(normx_sq > 0.0)) return OR_EMPTY;

    if (init) {                                                        /* C-2 */
        for (int n = 0; n < N; ++n) std::memcpy(A[n], init[n], sizeof(double) * dims[n] * R);
    } else {
        oracle_init_factors(N, dims, R, seed, A);
    }
    auto t0 = clk::now();
    std::vector<std::vector<uint64_t>> row_ptr(N), order(N);           /* grouping ("Sort") */
    for (int n = 0; n < N; ++n) {
        row_ptr[n].resize(dims[n] + 1);
        order[n].resize(nnz);
        oracle_group_by_mode(nnz, ind[n], dims[n], row_ptr[n].data(), order[n].data());
    }
    tm[1] += secs(t0, clk::now());

    std::vector<std::vector<double>> G(N, std::vector<double>((size_t)R * R));
    std::vector<const double*> Gp(N);
    t0 = clk::now();
    for (int n = 0; n < N; ++n) { oracle_gram(dims[n], R, A[n], G[n].data()); Gp[n] = G[n].data(); }
    tm[2] += secs(t0, clk::now());

    uint64_t maxI = 0;
    for (int n = 0; n < N; ++n) maxI = std::max(maxI, dims[n]);
    std::vector<double> M(maxI * R), V((size_t)R * R);
    std::vector<const double*> Ac(N);
    for (int n = 0; n < N; ++n) Ac[n] = A[n];

    auto tl = clk::now();
    double fit = 0.0, prev = 0.0;
    int it = 0;
    for (it = 1; it <= max_iters; ++it) {
        for (int n = 0; n < N; ++n) {
            t0 = clk::now();
            oracle_hadamard_except(N, R, Gp.data(), n, V.data());         /* C-6: V */
            tm[2] += secs(t0, clk::now());
            t0 = clk::now();
            mttkrp_grouped(N, dims[n], ind, vals, n, R, Ac.data(), row_ptr[n].data(),
                           order[n].data(), M.data());                    /* C-6: MTTKRP */
            tm[0] += secs(t0, clk::now());
            t0 = clk::now();
            if (oracle_cholesky_solve(R, V.data(), dims[n], M.data(), A[n]) != OR_OK)
                return OR_SINGULAR;                                       /* C-7 */
            tm[5] += secs(t0, clk::now());
            t0 = clk::now();
            oracle_normalize(dims[n], R, A[n], it == 1 ? 0 : 1, lambda);  /* C-8 */
            tm[3] += secs(t0, clk::now());
            t0 = clk::now();
            oracle_gram(dims[n], R, A[n], G[n].data());                   /* C-9 */
            tm[2] += secs(t0, clk::now());
        }
        t0 = clk::now();
        fit = oracle_fit(N, R, Gp.data(), lambda, dims[N - 1], M.data(), A[N - 1], normx_sq);
        tm[4] += secs(t0, clk::now());                                    /* C-10 */
        if (fit_history) fit_history[it - 1] = fit;
        if (it >= 2 && std::fabs(fit - prev) < tol) break;                /* C-11 */
        prev = fit;
    }
    if (it > max_iters) it = max_iters;
    tm[6] = secs(tl, clk::now());

    for (int n = 0; n < N; ++n) {                                         /* C-12 */
        for (int r = 0; r < R; ++r) {
            double s = 0.0;
            for (uint64_t i = 0; i < dims[n]; ++i) s += A[n][i * R + r] * A[n][i * R + r];
            const double nu = std::sqrt(s);
            if (nu > 0.0) {
                for (uint64_t i = 0; i < dims[n]; ++i) A[n][i * R + r] /= nu;
                lambda[r] *= nu;
            }
        }
    }
    if (iters_out) *iters_out = it;
    if (fit_out) *fit_out = fit;
    if (timings) std::memcpy(timings, tm, sizeof(tm));
    return OR_OK;
}

/* ------------------------------------------------------------------ C-13 CSF */
/* CSF_n: perm p_0 = root, then the other modes by ascending length, ties to the
 * lower mode id.  std::stable_sort of positions by the coordinate
 * tuple; level-l nodes are maximal runs of equal prefixes (p_0..p_l).            */
struct OracleCsf {
    int N;
    uint64_t nnz;
    int perm[8];
    std::vector<uint32_t> ids[8];
    std::vector<uint32_t> ptr[8];
    std::vector<double> vals;
};

void oracle_csf_perm(int N, const uint64_t* dims, int root, int* perm) {
    perm[0] = root;
    int k = 1;
    std::vector<int> rest;
    for (int m = 0; m < N; ++m) if (m != root) rest.push_back(m);
    std::stable_sort(rest.begin(), rest.end(), [&](int a, int b) { return dims[a] < dims[b]; });
    for (int m : rest) perm[k++] = m;
}

void* oracle_csf_build(int N, const uint64_t* dims, uint64_t nnz, const uint32_t* const* ind,
                       const double* vals, int root) {
    OracleCsf* c = new OracleCsf();
    c->N = N;
    c->nnz = nnz;
    oracle_csf_perm(N, dims, root, c->perm);
    std::vector<uint64_t> pos(nnz);
    std::iota(pos.begin(), pos.end(), 0);
    const int* perm = c->perm;
    std::stable_sort(pos.begin(), pos.end(), [&](uint64_t a, uint64_t b) {
        for (int l = 0; l < N; ++l) {
            const uint32_t x = ind[perm[l]][a], y = ind[perm[l]][b];
            if (x != y) return x < y;
        }
        return false;
    });
    c->vals.resize(nnz);
    for (uint64_t j = 0; j < nnz; ++j) c->vals[j] = vals[pos[j]];
    /* leaf level: every nonzero is a node */
    c->ids[N - 1].resize(nnz);
    for (uint64_t j = 0; j < nnz; ++j) c->ids[N - 1][j] = ind[perm[N - 1]][pos[j]];
    /* internal levels: node starts where the prefix (p_0..p_l) changes */
    std::vector<uint64_t> node_at(nnz);         /* level-(l+1) node index of position j */
    for (uint64_t j = 0; j < nnz; ++j) node_at[j] = j;   /* level N-1: node = position */
    for (int l = N - 2; l >= 0; --l) {
        std::vector<uint64_t> this_node(nnz);
        uint64_t cnt = 0;
        for (uint64_t j = 0; j < nnz; ++j) {
            bool start = (j == 0);
            for (int q = 0; q <= l && !start; ++q)
                if (ind[perm[q]][pos[j]] != ind[perm[q]][pos[j - 1]]) start = true;
            if (start) {
                c->ids[l].push_back(ind[perm[l]][pos[j]]);
                c->ptr[l].push_back((uint32_t)node_at[j]);
                ++cnt;
            }
            this_node[j] = cnt - 1;
        }
        const uint64_t nchildren = (l == N - 2) ? nnz : c->ids[l + 1].size();
        c->ptr[l].push_back((uint32_t)nchildren);
        node_at.swap(this_node);
    }
    return c;
}
void oracle_csf_perm_of(void* h, int* perm) {
    OracleCsf* c = (OracleCsf*)h;
    for (int l = 0; l < c->N; ++l) perm[l] = c->perm[l];
}
uint64_t oracle_csf_nodes(void* h, int level) {
    OracleCsf* c = (OracleCsf*)h;
    return c->ids[level].size();
}
void oracle_csf_copy(void* h, int level, uint32_t* ids, uint32_t* ptr) {
    OracleCsf* c = (OracleCsf*)h;
    if (ids) std::memcpy(ids, c->ids[level].data(), 4 * c->ids[level].size());
    if (ptr && level < c->N - 1) std::memcpy(ptr, c->ptr[level].data(), 4 * c->ptr[level].size());
}
void oracle_csf_vals(void* h, double* v) {
    OracleCsf* c = (OracleCsf*)h;
    std::memcpy(v, c->vals.data(), 8 * c->vals.size());
}
void oracle_csf_free(void* h) { delete (OracleCsf*)h; }

/* ---------------------------------------------------- C-15 CSF allocation policy */
/* SPEC.md:128-136 (allocate_csfs), the paper's lock / no-lock dichotomy PAPER.md:469-470:
 *   ALL (0): one CSF rooted at every mode; every mode is a ROOT traversal (level 0).
 *   ONE (1): one CSF rooted at the shortest mode (ties -> lowest id), the other modes
 *            below it by ascending length (C-13's order); mode at level l uses level l.
 *   TWO (2): ONE's CSF plus a second rooted at the longest mode (the LAST mode of the
 *            ascending-length order); each root mode uses its own CSF at level 0, every
 *            other mode uses the first CSF at its level there.
 * Outputs: *ncsf, roots[ncsf], mode_csf[N] (which CSF), mode_level[N] (its level).  */
int oracle_csf_alloc(int N, const uint64_t* dims, int policy, int* ncsf, int* roots,
                     int* mode_csf, int* mode_level) {
    std::vector<int> asc(N);
    std::iota(asc.begin(), asc.end(), 0);
    std::stable_sort(asc.begin(), asc.end(), [&](int a, int b) { return dims[a] < dims[b]; });
    if (policy == 0) {
        *ncsf = N;
        for (int m = 0; m < N; ++m) { roots[m] = m; mode_csf[m] = m; mode_level[m] = 0; }
        return OR_OK;
    }
    if (policy != 1 && policy != 2) return OR_BADINPUT;
    *ncsf = policy;
    roots[0] = asc[0];
    for (int l = 0; l < N; ++l) { mode_csf[asc[l]] = 0; mode_level[asc[l]] = l; }
    if (policy == 2) {
        roots[1] = asc[N - 1];
        mode_csf[asc[N - 1]] = 1;
        mode_level[asc[N - 1]] = 0;
    }
    return OR_OK;
}

/* ------------------------------------------------------------ C-14 partition */
/* Cut S slices (weights w) into G contiguous ranges minimising the max weight.
 * The cap C* is the smallest feasible cap (binary search over integers); the
 * boundaries are leftmost-greedy under C*: each range takes as many slices as
 * fit.  bounds has G+1 entries.                                                  */
static bool fits(const uint64_t* w, uint64_t S, int G, uint64_t cap) {
    int parts = 1;
    uint64_t cur = 0;
    for (uint64_t s = 0; s < S; ++s) {
        if (w[s] > cap) return false;
        if (cur + w[s] > cap) { ++parts; cur = 0; }
        cur += w[s];
    }
    return parts <= G;
}
void oracle_partition(const uint64_t* w, uint64_t S, int G, uint64_t* bounds) {
    uint64_t lo = 0, hi = 0;
    for (uint64_t s = 0; s < S; ++s) { lo = std::max(lo, w[s]); hi += w[s]; }
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (fits(w, S, G, mid)) hi = mid; else lo = mid + 1;
    }
    const uint64_t cap = lo;
    uint64_t s = 0;
    bounds[0] = 0;
    for (int g = 0; g < G; ++g) {
        uint64_t cur = 0;
        while (s < S && cur + w[s] <= cap) { cur += w[s]; ++s; }
        bounds[g + 1] = s;
    }
    bounds[G] = S;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

}  /* extern "C" */
