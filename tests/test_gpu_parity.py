"""GPU parity through the C ABI against the CPU oracle (gpu-marked).

Bars (BASELINE.json north star):
  CSF          bit-exact (ids, ptr, vals)                      — integer work
  MTTKRP       ||M_gpu - M_orc||_F / ||M_orc||_F <= 1e-10      — fp64, summation order only
               bit-exact on integer inputs (every partial sum is exact)
  CP-ALS       factors / lambda / fit <= 1e-7 relative after a fixed iteration count
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALS_TOL, MTTKRP_TOL, dev_coo, dev_factors, rel_fro

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


def check_csf_equal(csf, t):
    for n in range(t.nmodes):
        g = csf.export(n)
        o = oracle.csf_build(t.dims, t.ind, t.vals, n)
        assert g["perm"] == o["perm"].tolist()
        for l in range(t.nmodes):
            assert np.array_equal(g["ids"][l], o["ids"][l]), (n, l)
        for l in range(t.nmodes - 1):
            assert np.array_equal(g["ptr"][l], o["ptr"][l]), (n, l)
        assert np.array_equal(g["vals"].view(np.uint64), o["vals"].view(np.uint64))


def scaled_tensors():
    """Parity-size tensors with the configs' distributions, spanning many chunks."""
    out = [synth.generate_config("c1")]
    out.append(synth.generate((40_000, 11_000, 75_000), 300_000, [("zipf", 1.1)] * 3, "ratings",
                              seed=22))
    out.append(synth.generate((48_000, 1_800, 200), 250_000,
                              [("zipf", 1.0), ("zipf", 1.2), ("uniform",)], "ratings", seed=33))
    out.append(synth.generate((1_200, 900, 2_900), 200_000, [("uniform",)] * 3, "lognormal",
                              seed=44))
    out.append(synth.generate((20_000, 5_000, 1_000, 50), 300_000, [("zipf", 1.05)] * 4, "u01",
                              seed=55))
    return out


TENSORS = None


def tensors():
    global TENSORS
    if TENSORS is None:
        TENSORS = scaled_tensors()
    return TENSORS


# ------------------------------------------------------------------- CSF
def test_csf_bit_exact_random_small(sb, ctx):
    for seed in range(40):
        N = 3 + seed % 3
        t = synth.random_tiny(seed, nmodes=N, max_dim=9, max_nnz=120, dups=(seed % 2 == 0))
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
        check_csf_equal(csf, t)


def test_csf_bit_exact_config_shaped(sb, ctx):
    for t in tensors():
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
        check_csf_equal(csf, t)


def test_csf_host_input_and_wide_keys(sb, ctx):
    # host COO path + a key wider than 64 bits (8 modes x 2^9+ dims -> multi-group sort)
    rng = np.random.default_rng(3)
    dims = (700, 600, 900, 1000, 513, 800, 650, 1023)
    nnz = 3000
    ind = [rng.integers(0, d, nnz).astype(np.uint32) for d in dims]
    vals = rng.random(nnz)
    t = synth.SparseTensor(dims, ind, vals)
    csf = sb.csf_build(ind, vals, dims, ctx=ctx)
    check_csf_equal(csf, t)


def test_csf_bit_exact_mixed_radix_keys_and_sort_edges(sb, ctx):
    # Dims whose mixed-radix composite key needs fewer radix passes than the bit-packed one
    # (5x5x5: 9 -> 7 bits; 5^6: 18 -> 14 bits; the c5 dims: 57 -> 56 bits), so the builder
    # sorts and decodes mixed-radix keys; nonzero counts around the radix sort's tile (4096
    # pairs) and ragged ends (n % 4 != 0, n < 4: no bulk copy at all), and a c5-shaped tensor
    # of 1.5M nonzeros (several tiles per sort range).
    cases = [((5, 5, 5), n) for n in (1, 2, 3, 5, 100)]
    cases += [((5, 5, 5, 5, 5, 5), 3000), ((200_000, 50_000, 10_000, 500), 4096),
              ((200_000, 50_000, 10_000, 500), 4097), ((7, 300, 11), 8191)]
    for i, (dims, nnz) in enumerate(cases):
        rng = np.random.default_rng(100 + i)
        ind = [rng.integers(0, d, nnz).astype(np.uint32) for d in dims]
        vals = rng.random(nnz)
        t = synth.SparseTensor(dims, ind, vals)
        d_ind, d_vals = dev_coo(t)
        check_csf_equal(sb.csf_build(d_ind, d_vals, dims, ctx=ctx), t)
    t = synth.generate((200_000, 50_000, 10_000, 500), 1_500_000, [("zipf", 1.05)] * 4, "u01",
                       seed=56)
    d_ind, d_vals = dev_coo(t)
    check_csf_equal(sb.csf_build(d_ind, d_vals, t.dims, ctx=ctx), t)


def test_csf_bit_exact_adversarial_sort_inputs(sb, ctx):
    # The radix sort's corner cases through the builder: every nonzero at one coordinate (one
    # digit bucket takes all pairs in every pass, so the order is the input order alone), the
    # input already in CSF order and in reverse order, and a single hot slice holding half
    # the nonzeros across many sort tiles and ranges.
    rng = np.random.default_rng(7)
    n = 50_000
    dims = (300, 200, 100)
    cases = [[np.full(n, 7, np.uint32), np.full(n, 3, np.uint32), np.full(n, 99, np.uint32)]]
    ind = [rng.integers(0, d, n).astype(np.uint32) for d in dims]
    order = np.lexsort((ind[2], ind[1], ind[0]))
    cases.append([a[order] for a in ind])
    cases.append([a[order[::-1]] for a in ind])
    hot = [rng.integers(0, d, n).astype(np.uint32) for d in dims]
    hot[0][: n // 2] = 5
    cases.append(hot)
    for ind in cases:
        t = synth.SparseTensor(dims, ind, rng.random(n))
        d_ind, d_vals = dev_coo(t)
        check_csf_equal(sb.csf_build(d_ind, d_vals, dims, ctx=ctx), t)


# ---------------------------------------------------------------- MTTKRP
def run_mttkrp(sb, ctx, t, F, mode, ld=None, pad_value=0.0):
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    R = F[0].shape[1]
    fd = dev_factors(F, ld=ld, pad_value=pad_value)
    out = sb.mttkrp(csf, mode, fd, rank=R)
    ctx.sync()
    return out.cpu().numpy()[:, :R], out.cpu().numpy()


@pytest.mark.parametrize("R", [1, 3, 8, 16, 35, 64])
def test_mttkrp_parity_config_shaped(sb, ctx, R):
    rng = np.random.default_rng(R)
    for t in tensors():
        F = [rng.standard_normal((d, R)) for d in t.dims]
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
        ld = sb.padded_ld(R)
        fd = dev_factors(F, ld=ld)
        for n in range(t.nmodes):
            M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()
            ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
            assert rel_fro(M[:, :R], ref) <= MTTKRP_TOL, (t.dims, R, n)
            assert np.all(M[:, R:] == 0)


def test_leaf_tiling_auto_in_long_als_runs(sb):
    """Leaf tiling AUTO (the default): ALS runs of >= 10 iterations tile ROOT trees whose leaf
    factor exceeds half the L2 (300k x 36 doubles = 86 MB -> 2 tiles) — same result as the
    oracle; a second call on the context reuses arenas sized by the first."""
    t = synth.generate((60, 50, 300_000), 1_500_000, [("zipf", 1.1), ("uniform",), ("zipf", 1.0)],
                       "ratings", seed=62)
    ind, vals = dev_coo(t)
    ctx = sb.Context(0)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=35, max_iters=10, seed=4)
    for _ in range(2):
        res = sb.cpd_als(ind, vals, t.dims, rank=35, max_iters=10, seed=4, ctx=ctx, stats=True)
        als_compare(res, ref)
    off = sb.Context(0)
    off.set_leaf_tiling(0)
    res_off = sb.cpd_als(ind, vals, t.dims, rank=35, max_iters=10, seed=4, ctx=off, stats=True)
    als_compare(res_off, ref)
    # the tiled tree runs one ROOT launch per tile (and its split kernels) where off runs one
    assert res["stats"]["kernel_launches"] > res_off["stats"]["kernel_launches"]


@pytest.mark.parametrize("R", [8, 35, 64])
def test_mttkrp_l1_allocating_gathers(sb, ctx, monkeypatch, R):
    """The ROOT kernels' L1-allocating gather variant (chosen for leaf factors larger than
    half the L2; forced here with SPLATT_L1_ALLOC=1): same parity bar, N = 3 and 4, packed
    and power-of-two lane groups."""
    monkeypatch.setenv("SPLATT_L1_ALLOC", "1")
    rng = np.random.default_rng(100 + R)
    for t in (tensors()[1], tensors()[4]):
        F = [rng.standard_normal((d, R)) for d in t.dims]
        ind, vals = dev_coo(t)
        csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
        fd = dev_factors(F, ld=sb.padded_ld(R))
        for n in range(t.nmodes):
            M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()
            ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
            assert rel_fro(M[:, :R], ref) <= MTTKRP_TOL, (t.dims, R, n)


def test_mttkrp_integer_bit_exact(sb, ctx):
    """X-3: integer values x factors in {0,1,2}: exact in fp64 in any order."""
    rng = np.random.default_rng(11)
    for t in tensors()[1:3]:
        F = [rng.integers(0, 3, (d, 35)).astype(np.float64) for d in t.dims]
        for n in range(t.nmodes):
            M, _ = run_mttkrp(sb, ctx, t, F, n, ld=36)
            assert np.array_equal(M, oracle.mttkrp(t.dims, t.ind, t.vals, F, n))


def test_mttkrp_random_small_all_modes_and_ranks(sb, ctx):
    for seed in range(30):
        N = 3 + seed % 3
        t = synth.random_tiny(100 + seed, nmodes=N, max_dim=9, max_nnz=200, dups=(seed % 3 == 0))
        rng = np.random.default_rng(seed)
        R = int(rng.integers(1, 40))
        F = [rng.standard_normal((d, R)) for d in t.dims]
        for n in range(N):
            M, _ = run_mttkrp(sb, ctx, t, F, n)
            assert rel_fro(M, oracle.mttkrp(t.dims, t.ind, t.vals, F, n)) <= MTTKRP_TOL


def test_mttkrp_heavy_slice_and_long_fiber(sb, ctx):
    """One slice spanning hundreds of chunks (fp64 atomics at chunk seams) and a fiber
    longer than a chunk; plus many singleton slices."""
    rng = np.random.default_rng(5)
    I0, I1, I2 = 50, 40, 30_000
    a = [np.zeros(20_000, np.uint32), rng.integers(0, I1, 20_000).astype(np.uint32),
         rng.permutation(I2)[:20_000].astype(np.uint32)]
    a[1][:5000] = 7  # one long fiber (slice 0, j = 7)
    b = [rng.integers(1, I0, 3000).astype(np.uint32), rng.integers(0, I1, 3000).astype(np.uint32),
         rng.integers(0, I2, 3000).astype(np.uint32)]
    coords = np.unique(np.stack([np.concatenate([a[m], b[m]]) for m in range(3)], 1), axis=0)
    coords = coords[rng.permutation(len(coords))]
    t = synth.SparseTensor((I0, I1, I2), [coords[:, m].copy() for m in range(3)],
                           rng.random(len(coords)))
    F = [rng.standard_normal((d, 35)) for d in t.dims]
    for n in range(3):
        M, _ = run_mttkrp(sb, ctx, t, F, n)
        assert rel_fro(M, oracle.mttkrp(t.dims, t.ind, t.vals, F, n)) <= MTTKRP_TOL


def test_mttkrp_ld_variants_and_garbage_pads(sb, ctx):
    t = tensors()[1]
    rng = np.random.default_rng(2)
    R = 35
    F = [rng.standard_normal((d, R)) for d in t.dims]
    ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, 0)
    for ld, pad in ((35, 0.0), (36, np.nan), (40, 7.0), (37, 1e300)):
        M, full = run_mttkrp(sb, ctx, t, F, 0, ld=ld, pad_value=pad)
        assert rel_fro(M, ref) <= MTTKRP_TOL, ld
        assert np.all(full[:, R:] == 0), ld


def test_mttkrp_empty_rows_are_zero(sb, ctx):
    t = synth.generate((5000, 300, 200), 2000, [("zipf", 1.2)] * 3, "u01", seed=9)
    rng = np.random.default_rng(0)
    F = [rng.random((d, 8)) for d in t.dims]
    M, _ = run_mttkrp(sb, ctx, t, F, 0)
    empty = np.setdiff1d(np.arange(5000), t.ind[0])
    assert empty.size > 0 and np.all(M[empty] == 0)


# ----------------------------------------------------------------- CP-ALS
def als_compare(res, ref, tol=ALS_TOL):
    for n, (A, B) in enumerate(zip(res["factors"], ref["factors"])):
        A = A.cpu().numpy() if hasattr(A, "cpu") else A
        assert rel_fro(A, B) <= tol, ("factor", n, rel_fro(A, B))
    lam = res["lam"].cpu().numpy() if hasattr(res["lam"], "cpu") else res["lam"]
    assert rel_fro(lam, ref["lam"]) <= tol
    assert abs(res["fit"] - ref["fit"]) <= tol * abs(ref["fit"])
    assert res["iters"] == ref["iters"]
    assert np.allclose(res["fit_history"], ref["fit_history"], rtol=tol, atol=0)


def test_cpd_als_c1_full_parity(sb, ctx):
    t = synth.generate_config("c1")
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=8, max_iters=10, tol=0.0, seed=1, ctx=ctx)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=10, tol=0.0, seed=1)
    als_compare(res, ref)


@pytest.mark.parametrize("idx,R,iters", [(1, 35, 5), (2, 35, 5), (3, 64, 3), (4, 16, 5)])
def test_cpd_als_config_shaped_parity(sb, ctx, idx, R, iters):
    t = tensors()[idx]
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=iters, seed=idx, ctx=ctx)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=iters, seed=idx)
    als_compare(res, ref)


def test_cpd_als_one_step_from_oracle_state(sb, ctx):
    """Each GPU iteration started from the oracle's factors: isolates kernel error
    from the ALS amplification of rounding (last row)."""
    t = tensors()[1]
    R = 35
    A = oracle.init_factors(t.dims, R, 7)
    ind, vals = dev_coo(t)
    for step in range(3):
        ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=1, init=A)
        res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=1, init=A, ctx=ctx)
        als_compare(res, ref, tol=1e-9)
        A = [f * 1.0 for f in ref["factors"]]


@pytest.mark.parametrize("path", ["dmma", "simt"])
@pytest.mark.parametrize("R", [1, 5, 8, 13, 24, 35, 40, 57, 64, 65, 96])
def test_row_solve_paths_one_step(sb, ctx, monkeypatch, R, path):
    """Line 5's row solve + Gram/colmax/inner statistics on both kernels: the fp64
    tensor-core one (R <= 64: every 8-column tile count 1..8, ragged last tiles) and the SIMT
    one (forced with SPLATT_SOLVE_SIMT, and the only one beyond R = 64); one ALS step from
    the oracle's state, twice, at the one-step tolerance."""
    if path == "simt":
        monkeypatch.setenv("SPLATT_SOLVE_SIMT", "1")
    t = tensors()[2]
    A = oracle.init_factors(t.dims, R, 11)
    ind, vals = dev_coo(t)
    for _ in range(2):
        ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=1, init=A)
        res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=1, init=A, ctx=ctx)
        als_compare(res, ref, tol=1e-9)
        A = [f * 1.0 for f in ref["factors"]]


def test_cpd_als_rank1_planted_and_host_io(sb, ctx):
    rng = np.random.default_rng(4)
    F = [rng.random((d, 1)) + 0.1 for d in (9, 7, 8)]
    t = synth.full_kruskal(F)
    res = sb.cpd_als(t.ind, t.vals, t.dims, rank=1, max_iters=1, seed=3, ctx=ctx, out_device=False)
    assert 0.0 <= 1.0 - res["fit"] <= 1e-7
    for n in range(3):
        a = res["factors"][n][:, 0] / np.linalg.norm(res["factors"][n][:, 0])
        b = F[n][:, 0] / np.linalg.norm(F[n][:, 0])
        assert np.max(np.abs(a - b)) <= 1e-12


@pytest.mark.parametrize("tol", [1e-2, 1e-3, 1e-4, 2e-4, 1e-6])  # stops at 2, 3, 16, 14, 38
def test_cpd_als_tol_stops_like_oracle(sb, ctx, tol):
    """Q-6 on the device: the fit kernel marks the converged iteration and the host only looks
    every 8 iterations, so stopping points on and off that stride must both come out at the
    oracle's iteration with the oracle's factors (the up-to-7 enqueued extra iterations are
    no-ops)."""
    t = tensors()[0]
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=8, max_iters=100, tol=tol, seed=1, ctx=ctx)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=100, tol=tol, seed=1)
    assert res["iters"] == ref["iters"] < 100
    assert len(res["fit_history"]) == res["iters"]
    als_compare(res, ref)


def test_cpd_als_host_input_with_tol(sb, ctx):
    """Host-staged COO (values uploaded on the copy stream during the sort, ||X|| taken after
    the build) with the device-side convergence test: same stopping iteration and model as
    the oracle, host outputs."""
    t = tensors()[0]
    res = sb.cpd_als(t.ind, t.vals, t.dims, rank=8, max_iters=100, tol=1e-4, seed=1, ctx=ctx,
                     out_device=False)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=100, tol=1e-4, seed=1)
    assert res["iters"] == ref["iters"] < 100
    als_compare(res, ref)


def test_errors(sb, ctx):
    t = synth.random_tiny(3)
    ind, vals = dev_coo(t)
    with pytest.raises(ValueError):
        sb.cpd_als(ind, vals, t.dims, rank=0, max_iters=1, ctx=ctx)
    with pytest.raises(ValueError):
        sb.cpd_als(ind, vals, t.dims, rank=2, max_iters=0, ctx=ctx)
    with pytest.raises(sb.EmptyTensorError):
        sb.cpd_als(ind, vals * 0, t.dims, rank=2, max_iters=1, ctx=ctx)
    # host-staged values (uploaded while the sort runs; ||X|| checked at the end of the call)
    with pytest.raises(sb.EmptyTensorError):
        sb.cpd_als(t.ind, t.vals * 0, t.dims, rank=2, max_iters=3, ctx=ctx, out_device=False)
    bad_host = [a.copy() for a in t.ind]
    bad_host[2][-1] = t.dims[2]
    with pytest.raises(sb.BadInputError):
        sb.cpd_als(bad_host, t.vals, t.dims, rank=2, max_iters=1, ctx=ctx, out_device=False)
    bad = [a.clone() for a in ind]
    bad[1][0] = t.dims[1]
    with pytest.raises(sb.BadInputError):
        sb.cpd_als(bad, vals, t.dims, rank=2, max_iters=1, ctx=ctx)
    with pytest.raises(sb.BadInputError):
        sb.csf_build(bad, vals, t.dims, ctx=ctx)
    zero = [np.zeros((d, 3)) for d in t.dims]
    with pytest.raises(sb.SingularError):
        sb.cpd_als(ind, vals, t.dims, rank=3, max_iters=1, init=zero, ctx=ctx)
    ctx.sync()  # context still healthy after the errors


def test_mttkrp_leaf_tiling(sb, ctx):
    """NEXT-4: a leaf factor larger than half the L2 (300k rows x 64 doubles = 154 MB) makes the
    ROOT MTTKRP run on leaf-id tiles (later tiles add into the owned rows); every mode must
    still match the oracle, and integer inputs bit for bit."""
    t = synth.generate((60, 50, 300_000), 1_500_000, [("zipf", 1.1), ("uniform",), ("zipf", 1.0)],
                       "ratings", seed=61)
    rng = np.random.default_rng(61)
    R = 64
    F = [rng.standard_normal((d, R)) for d in t.dims]
    Fi = [rng.integers(0, 3, (d, R)).astype(np.float64) for d in t.dims]
    ind, vals = dev_coo(t)
    ctx = sb.Context(0)
    with pytest.raises(sb.BadInputError):
        ctx.set_leaf_tiling(-0.5)
    ctx.set_leaf_tiling("auto")
    ctx.set_leaf_tiling(0.5)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    fd, fdi = dev_factors(F), dev_factors(Fi)
    for n in range(3):
        M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()
        assert rel_fro(M, oracle.mttkrp(t.dims, t.ind, t.vals, F, n)) <= MTTKRP_TOL, n
        Mi = sb.mttkrp(csf, n, fdi, rank=R).cpu().numpy()
        assert np.array_equal(Mi, oracle.mttkrp(t.dims, t.ind, t.vals, Fi, n)), n
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=2, seed=3)
    # repeated calls on one context: the second call's trees, chunk tables and tiles come
    # from arenas sized by the first (a tree once recorded the build's scratch arena as its
    # allocator, so its tiles were released with the build temporaries: illegal access)
    for _ in range(3):
        res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=2, seed=3, ctx=ctx)
        als_compare(res, ref)
    res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=5, seed=3, ctx=ctx)  # + gather tuning
    als_compare(res, oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=5, seed=3))


@pytest.mark.parametrize("R", [3, 16, 35, 64])
def test_root_kernel_generations_agree(sb, ctx, monkeypatch, R):
    """The second-generation ROOT kernel (records + shared-memory hot rows, root2.cuh) and
    the first (mttkrp_kernel.cuh, SPLATT_ROOT2=0) against the oracle on power-law tensors
    (N = 3 and 4), where the hot-row table takes most gathers."""
    import torch
    for idx, (dims, nnz, dists) in enumerate([((3000, 800, 5000), 200_000, [("zipf", 1.1)] * 3),
                                              ((2000, 700, 300, 40), 150_000, [("zipf", 1.05)] * 4)]):
        t = synth.generate(dims, nnz, dists, "u01", seed=50 + idx)
        F = oracle.init_factors(t.dims, R, 7)
        ind, vals = dev_coo(t)
        fd = dev_factors(F, sb.padded_ld(R))
        for env in ("3", "0"):  # second generation (also on N = 3), first generation
            monkeypatch.setenv("SPLATT_ROOT2", env)
            csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
            for n in range(t.nmodes):
                M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()[:, :R]
                ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
                assert rel_fro(M, ref) <= MTTKRP_TOL, (env, n)
            del csf
        torch.cuda.synchronize()


@pytest.mark.parametrize("chunk", ["32", "96", "1024"])
def test_root2_four_mode_seams_and_tiles(sb, monkeypatch, chunk):
    """4-mode ROOT kernel v2 with tiny and default chunks (every kind of seam: slices,
    level-1 nodes and fibers cut by chunk ends, heavy slices over many chunks) and with forced
    leaf tiles (later tiles add into the owned rows), against the oracle."""
    monkeypatch.setenv("SPLATT_CHUNK", chunk)
    # >= 2^20 nonzeros: leaf tiling applies (the 90000-row leaf factor -> 8 tiles at 1e-4)
    t = synth.generate((60, 3000, 40, 90000), 1_100_000,
                       [("zipf", 1.3), ("zipf", 1.05), ("zipf", 1.2), ("uniform",)], "u01", seed=71)
    R = 16
    F = oracle.init_factors(t.dims, R, 3)
    ind, vals = dev_coo(t)
    fd = dev_factors(F, sb.padded_ld(R))
    for tiling in (0.0, 1e-4):
        c = sb.Context(0)
        c.set_leaf_tiling(tiling)
        csf = sb.csf_build(ind, vals, t.dims, ctx=c)
        for n in range(4):
            M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()[:, :R]
            ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
            assert rel_fro(M, ref) <= MTTKRP_TOL, (tiling, n)
        del csf
        c.close()


@pytest.mark.parametrize("R", [1, 5, 12, 16, 33, 40, 64, 100, 128])
def test_root2_four_mode_every_group_width(sb, ctx, R):
    """4-mode ROOT kernel v2 at every lane-group width (G = 2, 4, 8, 10 packed, 16, 32) and the
    batch sizes / hot-table capacities they imply, garbage in the factors' pad columns."""
    t = tensors()[4]  # c5-shaped (Zipf 1.05 x 4)
    F = oracle.init_factors(t.dims, R, 11)
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    fd = dev_factors(F, sb.padded_ld(R), pad_value=float("nan")) if sb.padded_ld(R) > R \
        else dev_factors(F, sb.padded_ld(R))
    for n in range(4):
        M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()
        assert np.all(M[:, R:] == 0.0)
        assert rel_fro(M[:, :R], oracle.mttkrp(t.dims, t.ind, t.vals, F, n)) <= MTTKRP_TOL, n


def test_root2_prebuilt_csf_and_hot_table_off(sb, monkeypatch):
    """cpd_als on a prebuilt 4-mode CSF (the plan is built lazily from the tree, not by the
    builder) and with the hot-row table disabled (SPLATT_ROOT2_HOT=0: every gather cold), both
    against the oracle."""
    t = tensors()[4]
    R = 16
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=3, seed=4)
    ind, vals = dev_coo(t)
    c = sb.Context(0)
    csf = sb.csf_build(ind, vals, t.dims, ctx=c)
    als_compare(sb.cpd_als_csf(csf, rank=R, max_iters=3, seed=4, out_device=False), ref)
    del csf
    monkeypatch.setenv("SPLATT_ROOT2_HOT", "0")
    als_compare(sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=3, seed=4, ctx=sb.Context(0),
                           out_device=False), ref)
