"""CSF allocation policies ONE / TWO and the non-root MTTKRP kernels (
SPEC.md:128-136), through the C ABI, against the CPU oracle.

  * the policy's CSF set and mode dispatch equal the oracle's C-15 allocation, and every
    tree is bit-exact against the oracle's CSF (C-13) for its root;
  * MTTKRP through INTERNAL and LEAF kernels (fp64 atomics) <= 1e-10 against the
    definition (C-6), on every mode and config-shaped tensors, and bit-exact on integer
    inputs (every partial sum exact: the atomic order cannot matter);
  * the dispatch override (splatt_mttkrp_csf) runs every mode on every tree of the ALL set:
    each of ROOT / INTERNAL / LEAF on every level order, N = 3..8;
  * CP-ALS under ONE and TWO <= 1e-7 against the oracle (which has no policy: MTTKRP by
    definition), as under ALL.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALS_TOL, MTTKRP_TOL, dev_coo, dev_factors, rel_fro
from tests.test_gpu_parity import als_compare, tensors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb(cuda_ok):
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(sb):
    return sb.Context(0)


def check_policy_csf(sb, csf, t, policy):
    a = oracle.csf_alloc(t.dims, policy)
    assert csf.ncsf == len(a["roots"])
    for m in range(t.nmodes):
        assert csf.dispatch(m) == (a["mode_csf"][m], a["mode_level"][m])
    for k, root in enumerate(a["roots"]):
        g = csf.export(k)
        o = oracle.csf_build(t.dims, t.ind, t.vals, root)
        assert g["perm"] == o["perm"].tolist()
        for l in range(t.nmodes):
            assert np.array_equal(g["ids"][l], o["ids"][l]), (k, l)
        for l in range(t.nmodes - 1):
            assert np.array_equal(g["ptr"][l], o["ptr"][l]), (k, l)
        assert np.array_equal(g["vals"].view(np.uint64), o["vals"].view(np.uint64))


@pytest.mark.parametrize("policy", ["one", "two"])
def test_policy_csf_bit_exact_and_dispatch(sb, ctx, policy):
    pol = sb.POLICIES[policy]
    for seed in range(20):
        N = 3 + seed % 3
        t = synth.random_tiny(300 + seed, nmodes=N, max_dim=9, max_nnz=150, dups=(seed % 2 == 0))
        ind, vals = dev_coo(t)
        check_policy_csf(sb, sb.csf_build(ind, vals, t.dims, ctx=ctx, policy=pol), t, pol)
    for t in tensors():
        ind, vals = dev_coo(t)
        check_policy_csf(sb, sb.csf_build(ind, vals, t.dims, ctx=ctx, policy=pol), t, pol)


@pytest.mark.parametrize("policy", ["one", "two"])
@pytest.mark.parametrize("R", [1, 8, 16, 35, 64])
def test_policy_mttkrp_parity_config_shaped(sb, ctx, policy, R):
    rng = np.random.default_rng(100 + R)
    for t in tensors():
        F = [rng.standard_normal((d, R)) for d in t.dims]
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx, policy=policy)
        fd = dev_factors(F, ld=sb.padded_ld(R))
        for n in range(t.nmodes):
            M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()
            ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
            assert rel_fro(M[:, :R], ref) <= MTTKRP_TOL, (policy, t.dims, R, n, csf.dispatch(n))
            assert np.all(M[:, R:] == 0)


def test_every_kernel_kind_on_every_tree(sb, ctx):
    """splatt_mttkrp_csf: mode n on CSF k of the ALL set runs the level-of-n kernel of that
    tree, so every (level order, output level) pair is exercised, N = 3..8."""
    for seed in range(24):
        N = 3 + seed % 6
        t = synth.random_tiny(500 + seed, nmodes=N, max_dim=7 if N > 5 else 9,
                              max_nnz=400, dups=(seed % 4 == 0))
        rng = np.random.default_rng(seed)
        R = int(rng.integers(1, 70))
        F = [rng.standard_normal((d, R)) for d in t.dims]
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
        fd = dev_factors(F)
        for n in range(N):
            ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
            for k in range(N):
                M = sb.mttkrp(csf, n, fd, rank=R, which=k).cpu().numpy()
                assert rel_fro(M, ref) <= MTTKRP_TOL, (N, R, n, k)


def test_nonroot_kernels_span_chunks(sb, ctx):
    """Trees whose internal levels are much longer than a chunk (512 leaves) and whose
    nodes straddle chunk seams: the INTERNAL kernel's open-node flush and the LEAF/INTERNAL
    prefix rebuild at chunk starts."""
    rng = np.random.default_rng(8)
    for N, dims, nnz in ((3, (7, 3000, 40), 60_000), (4, (5, 9, 800, 30), 50_000)):
        t = synth.generate(dims, nnz, [("zipf", 1.3)] * N, "u01", seed=80 + N)
        F = [rng.standard_normal((d, 35)) for d in t.dims]
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
        fd = dev_factors(F, ld=36)
        for n in range(N):
            ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
            for k in range(N):
                M = sb.mttkrp(csf, n, fd, rank=35, which=k).cpu().numpy()[:, :35]
                assert rel_fro(M, ref) <= MTTKRP_TOL, (N, n, k)


def test_nonroot_integer_bit_exact(sb, ctx):
    """X-3 through the atomic kernels: integer values x factors in {0,1,2} are exact in any
    summation order, so INTERNAL/LEAF must agree with the oracle bit for bit."""
    rng = np.random.default_rng(12)
    for t in tensors()[1:3]:
        F = [rng.integers(0, 3, (d, 35)).astype(np.float64) for d in t.dims]
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx, policy="one")
        fd = dev_factors(F, ld=36)
        for n in range(t.nmodes):
            M = sb.mttkrp(csf, n, fd, rank=35).cpu().numpy()[:, :35]
            assert np.array_equal(M, oracle.mttkrp(t.dims, t.ind, t.vals, F, n)), n


def test_nonroot_heavy_rows(sb, ctx):
    """A leaf id shared by most fibers (atomic contention on one output row) and a long
    fiber, under ONE."""
    rng = np.random.default_rng(15)
    I0, I1, I2 = 20, 400, 5000
    n = 40_000
    c = np.stack([rng.integers(0, I0, n), rng.integers(0, I1, n),
                  np.where(rng.random(n) < 0.6, 17, rng.integers(0, I2, n))], 1)
    c = np.unique(c, axis=0)
    c = c[rng.permutation(len(c))].astype(np.uint32)
    t = synth.SparseTensor((I0, I1, I2), [c[:, m].copy() for m in range(3)], rng.random(len(c)))
    F = [rng.standard_normal((d, 16)) for d in t.dims]
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx, policy="one")
    fd = dev_factors(F)
    for m in range(3):
        M = sb.mttkrp(csf, m, fd, rank=16).cpu().numpy()
        assert rel_fro(M, oracle.mttkrp(t.dims, t.ind, t.vals, F, m)) <= MTTKRP_TOL, m


@pytest.mark.parametrize("policy", ["one", "two"])
def test_policy_cpd_als_c1(sb, ctx, policy):
    t = synth.generate_config("c1")
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=8, max_iters=10, seed=1, ctx=ctx, policy=policy)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=10, seed=1)
    als_compare(res, ref)


@pytest.mark.parametrize("policy", ["one", "two"])
@pytest.mark.parametrize("idx,R,iters", [(1, 35, 4), (2, 35, 4), (4, 16, 4)])
def test_policy_cpd_als_config_shaped(sb, ctx, policy, idx, R, iters):
    t = tensors()[idx]
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=iters, seed=idx, ctx=ctx,
                     policy=policy, stats=True)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=iters, seed=idx)
    als_compare(res, ref)
    assert res["stats"]["mttkrp_launches"] == iters * t.nmodes


def test_policy_errors(sb, ctx):
    t = synth.random_tiny(7)
    ind, vals = dev_coo(t)
    with pytest.raises(sb.BadInputError):
        sb.csf_build(ind, vals, t.dims, ctx=ctx, policy=5)
    with pytest.raises(sb.BadInputError):
        sb.cpd_als(ind, vals, t.dims, rank=2, max_iters=1, ctx=ctx, policy=9)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx, policy="one")
    F = dev_factors([np.ones((d, 2)) for d in t.dims])
    with pytest.raises(sb.BadInputError):
        sb.mttkrp(csf, 0, F, rank=2, which=1)  # ONE has a single tree
    ctx.sync()


def test_traffic_counters_policy_all(sb, ctx):
    """The bench's roofline inputs: per launch under ALL, B_alg (12 B per
    leaf, 8 B per internal node, 8R B per gathered non-root row) and the compulsory bytes
    (tree once + each referenced factor row once + output once), recomputed here from numpy
    distinct counts and the reported node counts."""
    t = tensors()[1]
    R, iters = 35, 2
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=iters, seed=1, ctx=ctx, stats=True)
    s, N = res["stats"], t.nmodes
    distinct = [np.unique(t.ind[m]).size for m in range(N)]
    alg = mn = 0.0
    for n in range(N):
        nodes = s["csf_nodes"][n]
        assert nodes[0] == distinct[n] and nodes[N - 1] == t.nnz
        internal = sum(nodes[:N - 1])
        alg += 12 * t.nnz + 8 * internal + 8 * R * sum(nodes[1:])
        mn += 12 * t.nnz + 8 * internal + 8 * R * (t.dims[n] + sum(
            distinct[m] for m in range(N) if m != n))
    assert s["mttkrp_launches"] == iters * N
    assert s["mttkrp_alg_bytes"] == pytest.approx(iters * alg, rel=1e-12)
    assert s["mttkrp_min_bytes"] == pytest.approx(iters * mn, rel=1e-12)
    assert s["mttkrp_min_bytes"] < s["mttkrp_alg_bytes"]
