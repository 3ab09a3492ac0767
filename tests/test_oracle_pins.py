"""Pins of the CPU oracle against things other than itself.

Every test here runs on CPU (no ``gpu`` marker).  Each pin is chosen so that a
plausible mistake in oracle/oracle.cpp — a dropped term, a wrong sign or index, a
transposed operand, a wrong norm or threshold — fails at least one of them:

  X-1  brute force (densify/unfold/explicit KRP/matmul, tests/brute.py)  -> MTTKRP, N=3,4
  X-2  closed form A((B^T B)*(C^T C)) on fully stored exact-rank tensors  -> MTTKRP
  X-3  exact integer arithmetic (bit-exact) + all-ones = slice sums        -> MTTKRP
  X-4  invariants: <M_n, A_n> equal over n, linearity, single nonzero      -> MTTKRP
  X-5  numpy.linalg.solve / lstsq of the dense normal equations           -> solve, update
  X-6  SPEC hand examples (tests/golden/spec_dense_examples.json)          -> Gram, Hadamard,
                                                                             normalise, solve
  X-7  dense reconstruction 1 - ||X - Z|| / ||X||                          -> fit
  X-8  planted exact-rank tensors (rank-1 after 1 iteration; rank-4)      -> ALS end to end
  X-9  ALS monotonicity (least-squares guarantee)                         -> ALS loop
  X-10 published splitmix64 outputs (tests/golden/splitmix64_vectors.json)-> init
  X-11 SPEC CSF examples + numpy lexsort + round trip                     -> CSF
  X-12 SPEC partition examples + brute-force optimality                   -> partition
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from tests import brute
from tests.conftest import golden


def rnd_factors(rng, dims, R, kind="normal"):
    if kind == "int":
        return [rng.integers(0, 3, (d, R)).astype(np.float64) for d in dims]
    return [rng.standard_normal((d, R)) for d in dims]


# ------------------------------------------------------------------ X-1
@pytest.mark.parametrize("N", [3, 4])
def test_x1_mttkrp_vs_dense_bruteforce(N):
    for seed in range(60):
        t = synth.random_tiny(seed, nmodes=N, max_dim=8 if N == 3 else 5, max_nnz=64,
                              dups=(seed % 3 == 0))
        rng = np.random.default_rng(1000 + seed)
        R = int(rng.integers(1, 6))
        A = rnd_factors(rng, t.dims, R)
        for n in range(N):
            M = oracle.mttkrp(t.dims, t.ind, t.vals, A, n)
            Md = brute.mttkrp_dense(t.dims, t.ind, t.vals, A, n)
            assert np.max(np.abs(M - Md)) <= 1e-12 * max(1.0, np.max(np.abs(Md)))


# ------------------------------------------------------------------ X-2
@pytest.mark.parametrize("N", [3, 4])
def test_x2_closed_form_exact_rank(N):
    rng = np.random.default_rng(7)
    dims = (5, 4, 6) if N == 3 else (4, 3, 5, 2)
    R = 3
    F = [rng.random((d, R)) for d in dims]
    t = synth.full_kruskal(F)
    for n in range(N):
        H = np.ones((R, R))
        for m in range(N):
            if m != n:
                H = H * (F[m].T @ F[m])
        expect = F[n] @ H
        M = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
        assert np.max(np.abs(M - expect)) <= 1e-12 * np.max(np.abs(expect))


# ------------------------------------------------------------------ X-3
def test_x3_integer_bit_exact():
    for seed in range(20):
        t = synth.random_tiny(seed, nmodes=3 + seed % 2, max_dim=7, max_nnz=60, int_values=True,
                              dups=True)
        rng = np.random.default_rng(seed)
        A = rnd_factors(rng, t.dims, 4, kind="int")
        for n in range(len(t.dims)):
            M = oracle.mttkrp(t.dims, t.ind, t.vals, A, n)
            Md = brute.mttkrp_dense(t.dims, t.ind, t.vals, A, n)
            assert np.array_equal(M, Md)


def test_x3_all_ones_is_slice_sum_and_spec_example():
    g = golden("spec_dense_examples.json")["mttkrp_ones"]
    dims = tuple(g["dims"])
    t = synth.full_kruskal([np.ones((d, 1)) for d in dims])  # all-ones tensor, every cell stored
    A = [np.ones((d, g["R"])) for d in dims]
    for n in range(3):
        M = oracle.mttkrp(dims, t.ind, t.vals, A, n)
        assert np.all(M == g["value"])
    t = synth.generate_config("c1")
    A = [np.ones((d, 3)) for d in t.dims]
    for n in range(3):
        M = oracle.mttkrp(t.dims, t.ind, t.vals, A, n)
        ss = np.bincount(t.ind[n], weights=t.vals, minlength=t.dims[n])
        assert np.allclose(M[:, 0], ss, rtol=1e-13, atol=0)


# ------------------------------------------------------------------ X-4
def test_x4_invariants():
    rng = np.random.default_rng(3)
    t = synth.generate((30, 20, 25), 2000, [("zipf", 1.1)] * 3, "u01", seed=11)
    A = rnd_factors(rng, t.dims, 5)
    ips = [np.sum(oracle.mttkrp(t.dims, t.ind, t.vals, A, n) * A[n]) for n in range(3)]
    assert max(ips) - min(ips) <= 1e-11 * max(abs(x) for x in ips)
    # linearity in one factor and in the values
    M = oracle.mttkrp(t.dims, t.ind, t.vals, A, 0)
    A2 = [A[0], 3.0 * A[1], A[2]]
    assert np.allclose(oracle.mttkrp(t.dims, t.ind, t.vals, A2, 0), 3.0 * M, rtol=1e-13, atol=1e-13)
    assert np.allclose(oracle.mttkrp(t.dims, t.ind, 2.0 * t.vals, A, 0), 2.0 * M, rtol=1e-13,
                       atol=1e-13)
    # a single nonzero gives exactly one nonzero row: v * (A1[j] * A2[k])
    ind = [np.array([2], np.uint32), np.array([1], np.uint32), np.array([4], np.uint32)]
    M1 = oracle.mttkrp((5, 3, 6), ind, np.array([2.5]), [rng.random((d, 4)) for d in (5, 3, 6)], 0)
    assert np.count_nonzero(np.any(M1 != 0, axis=1)) == 1 and np.any(M1[2] != 0)


# ------------------------------------------------------------------ X-5
def test_x5_solve_vs_numpy_and_residual():
    rng = np.random.default_rng(5)
    for R in (1, 2, 5, 17, 35):
        B = rng.standard_normal((R + 3, R))
        V = B.T @ B + np.eye(R)
        M = rng.standard_normal((40, R))
        X = oracle.cholesky_solve(V, M)
        assert np.max(np.abs(X - np.linalg.solve(V, M.T).T)) <= 1e-10 * max(1, np.max(np.abs(X)))
        assert np.max(np.abs(X @ V - M)) <= 1e-10 * np.max(np.abs(M))
    ex = golden("spec_dense_examples.json")["solve"][0]
    # sqrt(2) pivots: equal up to rounding (1 ulp), not bitwise
    assert np.allclose(oracle.cholesky_solve(np.array(ex["V"], float), np.array(ex["M"], float)),
                       np.array(ex["X"]), rtol=1e-15, atol=0)
    # V = I -> X = M
    M = rng.standard_normal((7, 4))
    assert np.allclose(oracle.cholesky_solve(np.eye(4), M), M, rtol=0, atol=0)


def test_x5_singular_and_ridge():
    with pytest.raises(oracle.OracleError) as e:
        oracle.cholesky_solve(np.zeros((3, 3)), np.ones((2, 3)))
    assert e.value.code == oracle.SINGULAR
    with pytest.raises(oracle.OracleError):
        oracle.cholesky_solve(-np.eye(3), np.ones((2, 3)))
    # rank-deficient but PSD: the 1e-12 trace/R ridge rescues it
    v = np.array([[1.0, 1.0], [1.0, 1.0]])
    X = oracle.cholesky_solve(v, np.array([[2.0, 2.0]]))
    assert np.all(np.isfinite(X))


def test_x5_ridge_magnitude_closed_form():
    """C-7 / Q-14 ridge size, pinned by closed forms: a PSD V whose first
    Cholesky attempt fails is retried as W = V + delta I with delta = 1e-12 trace(V) / R.
    With m along V's null vector u (V u = 0), x W = m has the closed-form solution
    x = m / delta, so x measures delta itself."""
    # V = [[1,1],[1,1]]: pivot 2 is exactly 0 -> ridge delta = 1e-12 * 2 / 2 = 1e-12;
    # u = [1,-1]: x = [1,-1] / 1e-12.
    X = oracle.cholesky_solve(np.array([[1.0, 1.0], [1.0, 1.0]]), np.array([[1.0, -1.0]]))
    assert np.allclose(X[0], [1e12, -1e12], rtol=1e-3, atol=0)
    # Unequal diagonal, so trace/R (= 2.5/3) differs from the max diagonal (1) and from the
    # trace (2.5): delta = 1e-12 * 2.5 / 3 -> x = [1,-1,0] / delta = [1.2e12, -1.2e12, 0].
    # (1e-12 * max diag would give 1e12, 1e-12 * trace 4e11.)
    V = np.array([[1.0, 1.0, 0.0], [1.0, 1.0, 0.0], [0.0, 0.0, 0.5]])
    X = oracle.cholesky_solve(V, np.array([[1.0, -1.0, 0.0]]))
    delta = 1e-12 * 2.5 / 3
    assert np.allclose(X[0], [1 / delta, -1 / delta, 0.0], rtol=1e-3, atol=1e-3)
    # A ridge too small to rescue: V = [[4,2],[2,1]] (null vector [1,-2]).  delta = 2.5e-12,
    # the retried pivot is delta + delta/(4+delta) = 1.25 delta = 3.1e-12 <= 1e-12 * (4 + delta)
    # -> SINGULAR.  A ridge of 1e-12 * trace (5e-12) or 1e-12 * max diag (4e-12) would pass.
    with pytest.raises(oracle.OracleError) as e:
        oracle.cholesky_solve(np.array([[4.0, 2.0], [2.0, 1.0]]), np.array([[1.0, 1.0]]))
    assert e.value.code == oracle.SINGULAR


def test_x5_pivot_threshold_closed_form():
    """Q-14 pivot threshold: a pivot d fails iff d <= 1e-12 * max_j V_jj.  V = [[1,1],[1,1+a]]
    has second pivot exactly a (1 + a - 1, Sterbenz), and for m = [0, 1]:
      no ridge:   x = m V^-1 = [-1, 1] / a
      with ridge: x = [-1, 1 + delta] / ((1+delta)(1+a+delta) - 1),  delta = 1e-12 (2+a)/2."""
    for a, ridged in ((1.1e-12, False), (2e-12, False), (0.9e-12, True), (0.5e-12, True)):
        V = np.array([[1.0, 1.0], [1.0, 1.0 + a]])
        a_eff = (1.0 + a) - 1.0  # the representable a
        X = oracle.cholesky_solve(V, np.array([[0.0, 1.0]]))[0]
        if ridged:
            d = 1e-12 * (2.0 + a_eff) / 2.0
            det = (1 + d) * (1 + a_eff + d) - 1
            ref = np.array([-1.0, 1.0 + d]) / det
        else:
            ref = np.array([-1.0, 1.0]) / a_eff
        assert np.allclose(X, ref, rtol=1e-3, atol=0), (a, X, ref)


def test_x5_one_mode_update_is_least_squares():
    """One ALS mode update = argmin_A ||X_(n) - A K^T||_F on the dense unfolding."""
    rng = np.random.default_rng(9)
    t = synth.random_tiny(4, nmodes=3, max_dim=7, max_nnz=80)
    R = 3
    A = rnd_factors(rng, t.dims, R)
    G = [oracle.gram(a) for a in A]
    for n in range(3):
        V = oracle.hadamard_except(G, n)
        M = oracle.mttkrp(t.dims, t.ind, t.vals, A, n)
        An = oracle.cholesky_solve(V, M)
        K = brute.khatri_rao_except(A, n)
        Xn = brute.unfold(brute.densify(t.dims, t.ind, t.vals), n)
        ref = np.linalg.lstsq(K, Xn.T, rcond=None)[0].T
        assert np.max(np.abs(An - ref)) <= 1e-9 * max(1.0, np.max(np.abs(ref)))


# ------------------------------------------------------------------ X-6
def test_x6_spec_dense_examples():
    g = golden("spec_dense_examples.json")
    for ex in g["gram"]:
        assert np.array_equal(oracle.gram(np.array(ex["A"], float)), np.array(ex["G"], float))
    for ex in g["hadamard"]:
        # hadamard_except over [V, G] leaving out a third (identity of ones) factor
        ones = np.ones_like(np.array(ex["V"], float))
        out = oracle.hadamard_except([np.array(ex["V"], float), np.array(ex["G"], float), ones], 2)
        assert np.array_equal(out, np.array(ex["out"], float))
    for ex in g["normalize"]:
        A = np.array(ex["col"], float)[:, None]
        An, lam = oracle.normalize(A, ex["which"])
        assert lam[0] == ex["lambda"]
        assert np.allclose(An[:, 0], ex["out"], rtol=0, atol=1e-15)


def test_x6_gram_random_and_symmetric():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((50, 7))
    G = oracle.gram(A)
    assert np.array_equal(G, G.T)
    assert np.allclose(G, A.T @ A, rtol=1e-13, atol=1e-13)
    # Hadamard order: ascending m, leaving n out
    Gs = [rng.random((4, 4)) for _ in range(4)]
    assert np.allclose(oracle.hadamard_except(Gs, 1), Gs[0] * Gs[2] * Gs[3], rtol=1e-15, atol=0)


def test_x6_normalize_properties():
    rng = np.random.default_rng(4)
    A = rng.standard_normal((30, 5)) * 3
    An, lam = oracle.normalize(A, 0)
    assert np.allclose(np.linalg.norm(An, axis=0), 1.0, atol=1e-12)
    assert np.allclose(An * lam, A, rtol=1e-12, atol=1e-12)
    An, lam = oracle.normalize(A, 1)
    assert np.allclose(lam, np.maximum(1.0, np.max(np.abs(A), axis=0)), rtol=0, atol=0)
    assert np.all(np.max(np.abs(An), axis=0) <= 1.0)


# ------------------------------------------------------------------ X-7
def test_x7_fit_vs_dense_reconstruction():
    for seed in range(30):
        rng = np.random.default_rng(seed)
        t = synth.random_tiny(100 + seed, nmodes=3 + seed % 2, max_dim=6, max_nnz=50)
        R = int(rng.integers(1, 4))
        F = rnd_factors(rng, t.dims, R)
        lam = rng.random(R) * 0.3
        X = brute.densify(t.dims, t.ind, t.vals)
        N = len(t.dims)
        M = brute.mttkrp_dense(t.dims, t.ind, t.vals, F, N - 1)
        G = [f.T @ f for f in F]
        f_or = oracle.fit(G, lam, M, F[N - 1], np.sum(t.vals ** 2))
        f_ref = brute.fit_dense(X, F, lam)
        assert abs(f_or - f_ref) <= 1e-9 * max(1.0, abs(f_ref))
    # zero model -> fit 0
    g = golden("spec_dense_examples.json")
    F = [np.ones((d, 2)) for d in t.dims]
    M = brute.mttkrp_dense(t.dims, t.ind, t.vals, F, len(t.dims) - 1)
    assert oracle.fit([f.T @ f for f in F], np.zeros(2), M, F[-1], np.sum(t.vals ** 2)) == \
        g["fit_zero_model"]


# ------------------------------------------------------------------ X-8
def _match_up_to_scale(A, B):
    a = A / np.linalg.norm(A, axis=0)
    b = B / np.linalg.norm(B, axis=0)
    return np.max(np.abs(a - b))


@pytest.mark.parametrize("N", [3, 4])
def test_x8_rank1_recovered_after_one_iteration(N):
    rng = np.random.default_rng(21)
    dims = (6, 5, 7) if N == 3 else (4, 5, 3, 6)
    F = [rng.random((d, 1)) + 0.1 for d in dims]
    t = synth.full_kruskal(F)
    out = oracle.cpd_als(t.dims, t.ind, t.vals, rank=1, max_iters=1, tol=0.0, seed=3)
    assert 0.0 <= 1.0 - out["fit"] <= 1e-7
    for n in range(N):
        assert _match_up_to_scale(out["factors"][n], F[n]) <= 1e-12
    # reconstruction of the returned model equals the tensor
    X = brute.densify(t.dims, t.ind, t.vals)
    Z = brute.kruskal_dense(out["factors"], out["lam"])
    assert np.max(np.abs(X - Z)) <= 1e-12 * np.max(np.abs(X))


def test_x8_planted_fixed_point():
    """Started at the exact planted factors, one iteration keeps fit = 1 (X-8 iii)."""
    rng = np.random.default_rng(8)
    F = [rng.random((d, 3)) for d in (7, 6, 5)]
    t = synth.full_kruskal(F)
    out = oracle.cpd_als(t.dims, t.ind, t.vals, rank=3, max_iters=1, init=F)
    assert 1.0 - out["fit"] <= 1e-7


def test_x8_rank4_recovery():
    """SPEC.md:519 reading (DESIGN.md §2.2 R-8): every cell of a planted rank-4
    50x40x30 tensor stored; fit >= 0.99 within 50 iterations for >= 9/10 seeds."""
    good = 0
    for seed in range(10):
        rng = np.random.default_rng(500 + seed)
        F = [rng.random((d, 4)) for d in (50, 40, 30)]
        t = synth.full_kruskal(F)
        out = oracle.cpd_als(t.dims, t.ind, t.vals, rank=4, max_iters=50, tol=0.0, seed=seed)
        good += out["fit"] >= 0.99
    assert good >= 9


# ------------------------------------------------------------------ X-9
def test_x9_monotone_fit():
    for seed in range(50):
        t = synth.random_tiny(300 + seed, nmodes=3, max_dim=9, max_nnz=150)
        if min(t.dims) < 2:
            continue
        try:
            out = oracle.cpd_als(t.dims, t.ind, t.vals, rank=3, max_iters=15, seed=seed)
        except oracle.OracleError as e:
            assert e.code == oracle.SINGULAR
            continue
        h = out["fit_history"]
        assert np.all(np.diff(h) >= -1e-9), (seed, h)


def test_x9_convergence_rule_and_iteration_count():
    t = synth.generate_config("c1")
    out = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=10, tol=0.0, seed=1)
    assert out["iters"] == 10 and len(out["fit_history"]) == 10
    out = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=200, tol=1e-3, seed=1)
    h = out["fit_history"]
    assert out["iters"] < 200 and abs(h[-1] - h[-2]) < 1e-3
    assert all(abs(h[k] - h[k - 1]) >= 1e-3 for k in range(1, len(h) - 1))
    # finalised factors: unit 2-norm columns, lambda >= 0
    for A in out["factors"]:
        assert np.allclose(np.linalg.norm(A, axis=0), 1.0, atol=1e-12)
    assert np.all(out["lam"] >= 0)


def test_x9_thread_count_independence():
    t = synth.generate((60, 50, 40), 6000, [("zipf", 1.1)] * 3, "ratings", seed=4)
    n0 = oracle.num_threads()
    try:
        oracle.set_threads(1)
        a = oracle.cpd_als(t.dims, t.ind, t.vals, rank=6, max_iters=4, seed=2)
        oracle.set_threads(max(2, n0))
        b = oracle.cpd_als(t.dims, t.ind, t.vals, rank=6, max_iters=4, seed=2)
    finally:
        oracle.set_threads(n0)
    assert a["fit"] == b["fit"]
    for x, y in zip(a["factors"], b["factors"]):
        assert np.array_equal(x, y)


def test_errors():
    t = synth.random_tiny(1)
    with pytest.raises(oracle.OracleError) as e:
        oracle.cpd_als(t.dims, t.ind, t.vals, rank=2, max_iters=0)
    assert e.value.code == oracle.BADINPUT
    with pytest.raises(oracle.OracleError) as e:
        oracle.cpd_als(t.dims, t.ind, np.zeros_like(t.vals), rank=2, max_iters=1)
    assert e.value.code == oracle.EMPTY
    bad = [a.copy() for a in t.ind]
    bad[0][0] = t.dims[0]
    assert oracle.validate(t.dims, bad) == oracle.BADINPUT


# ------------------------------------------------------------------ X-10
def test_x10_splitmix64_published_vectors():
    g = golden("splitmix64_vectors.json")
    for k, h in enumerate(g["raw_hex"]):
        assert oracle.splitmix64_raw(0, k) == int(h, 16)
    for seed, us in g["u01_survey"].items():
        for k, u in enumerate(us):
            assert oracle.u01(int(seed), k) == u


def test_x10_init_layout_and_determinism():
    dims = (3, 4, 2)
    A = oracle.init_factors(dims, 5, 42)
    B = oracle.init_factors(dims, 5, 42)
    assert all(np.array_equal(a, b) for a, b in zip(A, B))
    # counter k = sum_{m<n} I_m R + i R + r  (logical R)
    assert A[1][2, 3] == oracle.u01(42, 3 * 5 + 2 * 5 + 3)
    assert A[2][1, 4] == oracle.u01(42, (3 + 4) * 5 + 1 * 5 + 4)
    big = oracle.init_factors((200_000, 5), 5, 7)[0]
    assert abs(big.mean() - 0.5) < 0.01 and big.min() >= 0 and big.max() < 1


# ------------------------------------------------------------------ X-11
def _lexsort_csf(dims, ind, vals, perm):
    """Independent CSF from numpy lexsort (stable) + run detection."""
    N = len(dims)
    keys = [np.asarray(ind[perm[l]], dtype=np.int64) for l in range(N)]
    order = np.lexsort(tuple(reversed(keys)))  # last key in tuple is primary
    sk = [k[order] for k in keys]
    nnz = len(order)
    ids, ptr = [None] * N, [None] * (N - 1)
    ids[N - 1] = sk[N - 1].astype(np.uint32)
    child_node = np.arange(nnz)
    change = np.zeros(nnz, dtype=bool)
    change[0] = True
    starts_per_level = []
    for l in range(N - 1):
        ch = np.zeros(nnz, dtype=bool)
        ch[0] = True
        ch[1:] = sk[l][1:] != sk[l][:-1]
        change = change | ch
        starts_per_level.append(change.copy())
    for l in range(N - 2, -1, -1):
        st = starts_per_level[l]
        pos = np.flatnonzero(st)
        ids[l] = sk[l][pos].astype(np.uint32)
        nchild = nnz if l == N - 2 else len(ids[l + 1])
        ptr[l] = np.append(child_node[pos], nchild).astype(np.uint32)
        child_node = np.cumsum(st) - 1
    return ids, ptr, np.asarray(vals)[order]


def test_x11_spec_examples():
    for name in ("spec_csf_example.json", "spec_csf_singleton.json"):
        g = golden(name)
        c = np.array(g["coords"], dtype=np.uint32)
        ind = [c[:, m].copy() for m in range(3)]
        csf = oracle.csf_build(g["dims"], ind, np.array(g["vals"]), 0)
        for l in range(3):
            assert csf["ids"][l].tolist() == g["ids"][l]
        for l in range(2):
            assert csf["ptr"][l].tolist() == g["ptr"][l]
        assert csf["vals"].tolist() == g["csf_vals"]


def test_x11_spec_sort_example():
    g = golden("spec_sort_example.json")
    c = np.array(g["coords"], dtype=np.uint32)
    ind = [c[:, m].copy() for m in range(3)]
    vals = np.arange(len(c), dtype=np.float64)
    for case in g["cases"]:
        # realise SPEC's perm with dims forcing that below-root order
        perm = case["perm"]
        dims = [0, 0, 0]
        for rank_, m in enumerate(perm):
            dims[m] = 10 + rank_
        csf = oracle.csf_build(dims, ind, vals, perm[0])
        assert csf["perm"].tolist() == perm
        order = c[csf["vals"].astype(int)].tolist()
        assert order == case["order"]


def test_x11_perm_rule():
    assert oracle.csf_perm((4, 2, 8), 0).tolist() == [0, 1, 2]
    assert oracle.csf_perm((4, 2, 8), 2).tolist() == [2, 1, 0]
    assert oracle.csf_perm((5, 5, 5, 1), 1).tolist() == [1, 3, 0, 2]  # ties -> lower mode id


def test_x11_lexsort_agreement_and_round_trip():
    for seed in range(120):
        N = 3 + seed % 2
        t = synth.random_tiny(seed, nmodes=N, max_dim=6, max_nnz=60, dups=(seed % 2 == 0))
        vals = np.arange(t.nnz, dtype=np.float64)  # identity of each nonzero
        for root in range(N):
            csf = oracle.csf_build(t.dims, t.ind, vals, root)
            ids, ptr, v = _lexsort_csf(t.dims, t.ind, vals, csf["perm"])
            assert all(np.array_equal(a, b) for a, b in zip(csf["ids"], ids))
            assert all(np.array_equal(a, b) for a, b in zip(csf["ptr"], ptr))
            assert np.array_equal(csf["vals"], v)
            # round trip: expand the tree back to coordinates in sorted order
            rows = np.zeros((t.nnz, N), dtype=np.int64)
            rows[:, N - 1] = csf["ids"][N - 1]
            span = [np.arange(len(csf["ids"][N - 2]) + 0)]
            leaf_owner = np.repeat(np.arange(len(csf["ids"][N - 2])), np.diff(csf["ptr"][N - 2]))
            owner = leaf_owner
            for l in range(N - 2, -1, -1):
                rows[:, l] = csf["ids"][l][owner]
                if l > 0:
                    parent = np.repeat(np.arange(len(csf["ids"][l - 1])), np.diff(csf["ptr"][l - 1]))
                    owner = parent[owner]
            src = np.stack([t.ind[csf["perm"][l]] for l in range(N)], 1)[csf["vals"].astype(int)]
            assert np.array_equal(rows, src)
            del span


# ------------------------------------------------------------------ X-12
def test_x12_spec_partition_examples():
    for case in golden("spec_partition.json")["cases"]:
        assert oracle.partition(case["weights"], case["G"]).tolist() == case["bounds"]


def test_x12_partition_optimal_bruteforce():
    rng = np.random.default_rng(12)
    for _ in range(150):
        S = int(rng.integers(1, 11))
        G = int(rng.integers(1, 5))
        w = rng.integers(0, 20, S)
        b = oracle.partition(w, G)
        assert b[0] == 0 and b[-1] == S and np.all(np.diff(b) >= 0)
        got = max(int(w[b[g]:b[g + 1]].sum()) for g in range(G))
        best = math.inf
        for cuts in itertools.combinations_with_replacement(range(S + 1), G - 1):
            bb = (0,) + cuts + (S,)
            best = min(best, max(int(w[bb[g]:bb[g + 1]].sum()) for g in range(G)))
        assert got == best


# ------------------------------------------------------------------ X-13
def test_x13_spec_csf_alloc_examples():
    """C-15 against SPEC.md:128-136's allocate_csfs examples (tests/golden/spec_csf_alloc.json)."""
    g = golden("spec_csf_alloc.json")
    kind_of = {0: "ROOT"}
    for case in g["cases"]:
        a = oracle.csf_alloc(case["dims"], g["policies"][case["policy"]])
        assert a["roots"] == case["roots"]
        assert a["mode_csf"] == case["mode_csf"]
        assert a["mode_level"] == case["mode_level"]
        N = len(case["dims"])
        for m in range(N):
            lvl = a["mode_level"][m]
            kind = kind_of.get(lvl, "LEAF" if lvl == N - 1 else "INTERNAL")
            assert kind == case["kinds"][str(m)]
        for k, perm in enumerate(case.get("perms", [])):
            assert oracle.csf_perm(case["dims"], a["roots"][k]).tolist() == perm


def test_x13_csf_alloc_properties():
    """Every mode's level is its position in its CSF's level order; ALL is all-root; ONE's
    root is the shortest mode (ties -> lowest id); TWO adds the longest."""
    rng = np.random.default_rng(13)
    for _ in range(200):
        N = int(rng.integers(3, 9))
        dims = [int(x) for x in rng.integers(1, 6, N)]
        for pol in (0, 1, 2):
            a = oracle.csf_alloc(dims, pol)
            assert len(a["roots"]) == {0: N, 1: 1, 2: 2}[pol]
            for m in range(N):
                perm = oracle.csf_perm(dims, a["roots"][a["mode_csf"][m]]).tolist()
                assert perm[a["mode_level"][m]] == m
            if pol == 0:
                assert a["mode_level"] == [0] * N
            else:
                shortest = min(range(N), key=lambda m: (dims[m], m))
                assert a["roots"][0] == shortest
                if pol == 2:
                    longest = max(range(N), key=lambda m: (dims[m], m))
                    assert a["roots"][1] == longest
                    assert a["mode_level"][longest] == 0
    with pytest.raises(oracle.OracleError):
        oracle.csf_alloc([3, 4, 5], 7)
