"""Opt-in bitwise reproducibility (splatt_ctx_set_deterministic; SURVEY.md §8(b) Determinism):
the ROOT MTTKRP's chunk-seam rows are summed in fixed chunk order instead of with atomics, so
repeated runs — MTTKRP and the whole ALS under policy ALL — are bitwise identical, and equal
to the oracle within the usual bars."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import MTTKRP_TOL, dev_coo, dev_factors, rel_fro
from tests.test_gpu_parity import als_compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb(cuda_ok):
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as m
    return m


def heavy_tensor():
    """Slices spanning hundreds of 256-leaf chunks, plus many short ones."""
    rng = np.random.default_rng(17)
    I0, I1, I2 = 50, 40, 30_000
    a = np.stack([np.zeros(60_000, np.uint32), rng.integers(0, I1, 60_000).astype(np.uint32),
                  rng.integers(0, I2, 60_000).astype(np.uint32)], 1)
    b = np.stack([rng.integers(1, I0, 20_000), rng.integers(0, I1, 20_000),
                  rng.integers(0, I2, 20_000)], 1).astype(np.uint32)
    c = np.unique(np.concatenate([a, b]), axis=0)
    c = c[rng.permutation(len(c))]
    return synth.SparseTensor((I0, I1, I2), [c[:, m].copy() for m in range(3)], rng.random(len(c)))


@pytest.mark.parametrize("name", ["heavy", "c2shape"])
def test_deterministic_mttkrp_bitwise_repeatable(sb, name):
    t = heavy_tensor() if name == "heavy" else synth.generate(
        (40_000, 11_000, 75_000), 300_000, [("zipf", 1.1)] * 3, "ratings", seed=22)
    ctx = sb.Context(0)
    ctx.set_deterministic(True)
    rng = np.random.default_rng(3)
    R = 35
    F = [rng.standard_normal((d, R)) for d in t.dims]
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    fd = dev_factors(F, ld=36)
    for n in range(3):
        runs = [sb.mttkrp(csf, n, fd, rank=R).cpu().numpy() for _ in range(4)]
        for r in runs[1:]:
            assert np.array_equal(r.view(np.uint64), runs[0].view(np.uint64)), n
        assert rel_fro(runs[0][:, :R], oracle.mttkrp(t.dims, t.ind, t.vals, F, n)) <= MTTKRP_TOL
    # exact arithmetic (integer values and factors): equal to the oracle bit for bit
    vi = np.floor(t.vals * 5) + 1
    Fi = [rng.integers(0, 3, (d, R)).astype(np.float64) for d in t.dims]
    ind, vals = dev_coo(synth.SparseTensor(t.dims, t.ind, vi))
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    fdi = dev_factors(Fi, ld=36)
    for n in range(3):
        M = sb.mttkrp(csf, n, fdi, rank=R).cpu().numpy()[:, :R]
        assert np.array_equal(M, oracle.mttkrp(t.dims, t.ind, vi, Fi, n))


def test_deterministic_als_bitwise_repeatable(sb):
    t = synth.generate((4000, 1100, 7500), 150_000, [("zipf", 1.1)] * 3, "ratings", seed=22)
    ctx = sb.Context(0)
    ctx.set_deterministic(True)
    ind, vals = dev_coo(t)
    runs = [sb.cpd_als(ind, vals, t.dims, rank=16, max_iters=6, seed=5, ctx=ctx,
                       out_device=False) for _ in range(3)]
    for r in runs[1:]:
        for n in range(3):
            assert np.array_equal(r["factors"][n].view(np.uint64),
                                  runs[0]["factors"][n].view(np.uint64))
        assert np.array_equal(r["lam"].view(np.uint64), runs[0]["lam"].view(np.uint64))
        assert r["fit"] == runs[0]["fit"]
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=16, max_iters=6, seed=5)
    als_compare(runs[0], ref)


@pytest.mark.parametrize("N", [3, 4])
def test_gather_policy_tuning_changes_no_bits(sb, monkeypatch, N):
    """cpd_als times the ROOT gathers with L1-allocating loads (iteration 2) and
    L1::no_allocate (iteration 3) per tree (>= 2^20 nonzeros) and keeps the faster: the choice must not
    change a bit of the result (deterministic context), whichever way it goes."""
    dims = (40_000, 11_000, 75_000) if N == 3 else (20_000, 5_000, 1_000, 50)
    t = synth.generate(dims, 1_200_000, [("zipf", 1.1)] * N, "ratings", seed=23)
    ctx = sb.Context(0)
    ctx.set_deterministic(True)
    ind, vals = dev_coo(t)
    runs = []
    for force in (None, "0", "1"):
        if force is None:
            monkeypatch.delenv("SPLATT_L1_ALLOC", raising=False)
        else:
            monkeypatch.setenv("SPLATT_L1_ALLOC", force)
        runs.append(sb.cpd_als(ind, vals, t.dims, rank=35 if N == 3 else 16, max_iters=5, seed=5, ctx=ctx,
                               out_device=False, stats=True))
    for r in runs[1:]:
        for n in range(N):
            assert np.array_equal(r["factors"][n].view(np.uint64),
                                  runs[0]["factors"][n].view(np.uint64))
        assert np.array_equal(r["lam"].view(np.uint64), runs[0]["lam"].view(np.uint64))
    assert runs[0]["stats"]["host_syncs"] == runs[1]["stats"]["host_syncs"] + 1  # the tuning sync


def test_deterministic_with_leaf_tiles(sb):
    t = synth.generate((60, 50, 300_000), 1_500_000, [("zipf", 1.1), ("uniform",), ("zipf", 1.0)],
                       "ratings", seed=61)
    ctx = sb.Context(0)
    ctx.set_deterministic(True)
    ctx.set_leaf_tiling(0.5)
    rng = np.random.default_rng(4)
    R = 64
    F = [rng.standard_normal((d, R)) for d in t.dims]
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    fd = dev_factors(F)
    for n in range(3):
        a = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()
        b = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        assert rel_fro(a, oracle.mttkrp(t.dims, t.ind, t.vals, F, n)) <= MTTKRP_TOL


@pytest.mark.parametrize("policy", ["all", "one", "two"])
def test_cpd_als_on_prebuilt_csf(sb, policy):
    """splatt_cpd_als_csf: the same ALS as splatt_cpd_als on the trees of a prebuilt set,
    repeatedly (rank sweep, seeds) without rebuilding; deterministic mode makes the ALL-policy
    result bitwise equal to the COO entry point's."""
    t = synth.generate((4000, 1100, 7500), 150_000, [("zipf", 1.1)] * 3, "ratings", seed=22)
    ctx = sb.Context(0)
    ctx.set_deterministic(True)
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx, policy=policy)
    for R, seed in ((8, 1), (16, 5), (8, 1)):
        res = sb.cpd_als_csf(csf, rank=R, max_iters=4, seed=seed, out_device=False, stats=True)
        ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=4, seed=seed)
        als_compare(res, ref)
        assert res["stats"]["t_build"] < 0.05  # no CSF build inside the call
        if policy == "all":
            coo = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=4, seed=seed, ctx=ctx,
                             out_device=False)
            for n in range(3):
                assert np.array_equal(res["factors"][n], coo["factors"][n]) or \
                    rel_fro(res["factors"][n], coo["factors"][n]) <= 1e-12
