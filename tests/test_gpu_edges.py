"""Edge cases through the C ABI against the oracle: a single nonzero, modes of length 1, the
maximum rank (128: 32-lane groups, 3 Gram block pairs per thread), chunk-size boundaries
(ragged tails), 8-mode tensors, every CSF policy on each."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALS_TOL, MTTKRP_TOL, dev_coo, dev_factors, rel_fro
from tests.test_gpu_parity import als_compare

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


def mttkrp_all(sb, ctx, t, R, policy, seed=0):
    rng = np.random.default_rng(seed)
    F = [rng.standard_normal((d, R)) for d in t.dims]
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx, policy=policy)
    fd = dev_factors(F, ld=sb.padded_ld(R))
    for n in range(t.nmodes):
        M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()[:, :R]
        ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
        assert rel_fro(M, ref) <= MTTKRP_TOL, (t.dims, R, policy, n)


@pytest.mark.parametrize("policy", ["all", "one", "two"])
def test_single_nonzero(sb, ctx, policy):
    t = synth.SparseTensor((5, 7, 3), [np.array([4], np.uint32), np.array([0], np.uint32),
                                      np.array([2], np.uint32)], np.array([2.5]))
    mttkrp_all(sb, ctx, t, 3, policy)
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=1, max_iters=3, seed=1, ctx=ctx, policy=policy)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=1, max_iters=3, seed=1)
    als_compare(res, ref)
    assert 0.0 <= 1.0 - res["fit"] <= 1e-7  # one nonzero is an exact rank-1 tensor


@pytest.mark.parametrize("policy", ["all", "one", "two"])
def test_modes_of_length_one(sb, ctx, policy):
    t = synth.generate((1, 300, 1, 40), 4000, [("uniform",), ("zipf", 1.1), ("uniform",),
                                               ("uniform",)], "u01", seed=7)
    mttkrp_all(sb, ctx, t, 5, policy)
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=4, max_iters=4, seed=2, ctx=ctx, policy=policy)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=4, max_iters=4, seed=2)
    als_compare(res, ref)


@pytest.mark.parametrize("policy", ["all", "one"])
def test_max_rank_128(sb, ctx, policy):
    t = synth.generate((900, 700, 1100), 60_000, [("zipf", 1.1)] * 3, "ratings", seed=12)
    mttkrp_all(sb, ctx, t, 128, policy, seed=3)
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=128, max_iters=2, seed=3, ctx=ctx, policy=policy)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=128, max_iters=2, seed=3)
    als_compare(res, ref)


@pytest.mark.parametrize("nnz", [255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 4095, 4096,
                                 4097])
def test_chunk_boundaries(sb, ctx, nnz):
    """nnz around the leaf-chunk sizes (256 for 3 modes, 1024 for 4+; 512 the non-root
    kernels' power-of-two groups see) and the 32-leaf batches:
    ragged last chunk, exactly full chunks, one leaf past."""
    for N in (3, 4):
        t = synth.generate((60, 50, 40, 30)[:N], nnz, [("zipf", 1.2)] * N, "u01", seed=nnz + N)
        assert t.nnz == nnz
        for R in (8, 35):
            mttkrp_all(sb, ctx, t, R, "all", seed=R)
        mttkrp_all(sb, ctx, t, 16, "one", seed=1)
    # long fibers (>= 4 leaves per fiber: the 512-leaf chunks of 3-mode trees)
    t = synth.generate((4, 3, 5000), nnz, [("uniform",)] * 3, "u01", seed=nnz)
    assert t.nnz == nnz
    mttkrp_all(sb, ctx, t, 35, "all", seed=2)


@pytest.mark.parametrize("policy", ["all", "one", "two"])
def test_eight_modes(sb, ctx, policy):
    t = synth.generate((6, 5, 7, 4, 6, 5, 3, 4), 3000, [("uniform",)] * 8, "u01", seed=88)
    mttkrp_all(sb, ctx, t, 6, policy, seed=8)
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=3, max_iters=3, seed=8, ctx=ctx, policy=policy)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=3, max_iters=3, seed=8)
    als_compare(res, ref)


def test_repeated_calls_reuse_arena(sb, ctx):
    """Repeated calls (arena reuse) and a smaller call after a larger one give the oracle's
    results every time."""
    big = synth.generate((4000, 1100, 7500), 200_000, [("zipf", 1.1)] * 3, "ratings", seed=5)
    small = synth.generate_config("c1")
    for t, R, seed in ((big, 16, 1), (small, 8, 2), (big, 16, 1), (small, 8, 2)):
        ind, vals = dev_coo(t)
        res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=3, seed=seed, ctx=ctx)
        ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=3, seed=seed)
        als_compare(res, ref)


@pytest.mark.parametrize("policy", ["all", "one", "two"])
def test_csf_maximum_dims(sb, ctx, policy):
    """Maximum mode lengths (I < 2^32: 32-bit coordinates, a 65-bit composite key -> two
    key groups; coordinates at 0 and I - 1 included) and duplicates: every tree bit-exact
    against the oracle.  (MTTKRP at these lengths would need 2^32-row factors.)"""
    rng = np.random.default_rng(71)
    dims = (2**32 - 1, 2**31 + 5, 7)
    n = 3000
    ind = [rng.integers(0, d, n, dtype=np.uint64).astype(np.uint32) for d in dims]
    ind[0][:3] = [0, dims[0] - 1, dims[0] - 1]
    ind[1][:3] = [dims[1] - 1, 0, 0]
    ind[2][:3] = [6, 0, 0]                       # positions 1 and 2: a duplicate pair
    t = synth.SparseTensor(dims, ind, rng.random(n))
    dind, dvals = dev_coo(t)
    csf = sb.csf_build(dind, dvals, t.dims, ctx=ctx, policy=policy)
    for k in range(csf.ncsf):
        g = csf.export(k)
        o = oracle.csf_build(t.dims, t.ind, t.vals, g["perm"][0])
        assert g["perm"] == o["perm"].tolist()
        for l in range(3):
            assert np.array_equal(g["ids"][l], o["ids"][l]), (k, l)
        for l in range(2):
            assert np.array_equal(g["ptr"][l], o["ptr"][l]), (k, l)
        assert np.array_equal(g["vals"].view(np.uint64), o["vals"].view(np.uint64))
    bad = [a.clone() for a in dind]
    with pytest.raises(sb.BadInputError):
        sb.csf_build(bad, dvals, (2**32, dims[1], dims[2]), ctx=ctx, policy=policy)
