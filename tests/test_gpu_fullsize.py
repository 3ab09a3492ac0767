"""Full-size parity on BASELINE.json's configs, through the same C-ABI calls bench.py times.

c2 (8M nnz): CSF bit-exact against the oracle, MTTKRP <= 1e-10 for every mode, CP-ALS
20 iterations <= 1e-7.  c3 (100M), c4 (77M, R=35 and R=64) and c5 (150M, 4 modes): CSF
bit-exact against an independent library sort (stable torch.sort of the packed coordinate
key, which is the definition of the CSF order) for every tree, and against the oracle's
std::stable_sort CSF for c5's mode-0 tree; MTTKRP <= 1e-10 against the oracle for every
mode; CP-ALS against the oracle <= 1e-7 after the configs' 20 iterations on the metric's
configs c3 and c5 (BASELINE.json:9, :11), 2 on c4.  X-3:
on c2 and c3 at full scale, integer ratings x factors in {0, 1, 2} make every partial sum an
integer below 2^53, so the MTTKRP must equal the oracle's bit for bit.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALS_TOL, MTTKRP_TOL, dev_coo, rel_fro

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

_CACHE = {}


def tensor(name):
    if name not in _CACHE:
        _CACHE.clear()
        _CACHE[name] = synth.generate_config(name)
    return _CACHE[name]


@pytest.fixture(scope="module")
def sb(cuda_ok):
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(sb):
    return sb.Context(0)


def check_csf_by_library_sort(csf_export, t):
    """Expand the GPU CSF back to coordinates and compare with a stable sort of the COO by
    the packed (perm-ordered) key — positions break ties, so the order is unique."""
    import torch
    perm = csf_export["perm"]
    N = len(perm)
    # (torch's own CUDA sort: a library routine independent of the path under test, and
    # seconds faster per tree than the CPU sort at 150M keys)
    key = torch.zeros(t.nnz, dtype=torch.int64, device="cuda")
    for l in range(N):
        key = key * int(t.dims[perm[l]]) + torch.from_numpy(t.ind[perm[l]].astype(np.int64)).cuda()
    _, order = torch.sort(key, stable=True)
    order = order.cpu().numpy()
    del key
    ids, ptr = csf_export["ids"], csf_export["ptr"]
    # leaf level and values
    assert np.array_equal(ids[N - 1], t.ind[perm[N - 1]][order])
    assert np.array_equal(csf_export["vals"].view(np.uint64), t.vals[order].view(np.uint64))
    # internal levels: expand node ids to leaves through ptr
    owner = np.repeat(np.arange(len(ids[N - 2])), np.diff(ptr[N - 2].astype(np.int64)))
    for l in range(N - 2, -1, -1):
        assert np.array_equal(ids[l][owner], t.ind[perm[l]][order]), l
        if l > 0:
            parent = np.repeat(np.arange(len(ids[l - 1])), np.diff(ptr[l - 1].astype(np.int64)))
            owner = parent[owner]
        # nodes are maximal runs: consecutive nodes under one parent differ
    for l in range(N - 1):
        assert ptr[l][0] == 0 and np.all(np.diff(ptr[l].astype(np.int64)) > 0)


def mttkrp_all_modes(sb, ctx, t, R, seed):
    import torch
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    F = oracle.init_factors(t.dims, R, seed)
    ld = sb.padded_ld(R)
    fd = []
    for f in F:
        b = np.zeros((f.shape[0], ld))
        b[:, :R] = f
        fd.append(torch.from_numpy(b).cuda())
    for n in range(t.nmodes):
        M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()[:, :R]
        ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
        err = rel_fro(M, ref)
        assert err <= MTTKRP_TOL, (n, err)
    return csf


def x3_integer_bitexact(sb, ctx, t, R):
    """X-3 at full scale: factors with entries in {0, 1, 2} and integer values; every product
    and partial sum is an exact integer (< 2^53), so summation order cannot matter."""
    import torch
    assert np.array_equal(t.vals, np.round(t.vals))
    rng = np.random.default_rng(33)
    F = [rng.integers(0, 3, (int(d), R)).astype(np.float64) for d in t.dims]
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    ld = sb.padded_ld(R)
    fd = []
    for f in F:
        b = np.zeros((f.shape[0], ld))
        b[:, :R] = f
        fd.append(torch.from_numpy(b).cuda())
    for n in range(t.nmodes):
        M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()[:, :R]
        ref = oracle.mttkrp(t.dims, t.ind, t.vals, F, n)
        assert np.max(ref) < 2.0 ** 53
        assert np.array_equal(M, ref), (n, np.max(np.abs(M - ref)))


def als_check(sb, ctx, t, R, iters, seed):
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=iters, tol=0.0, seed=seed, ctx=ctx)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=iters, tol=0.0, seed=seed)
    for n in range(t.nmodes):
        e = rel_fro(res["factors"][n].cpu().numpy(), ref["factors"][n])
        assert e <= ALS_TOL, (n, e)
    assert rel_fro(res["lam"].cpu().numpy(), ref["lam"]) <= ALS_TOL
    assert abs(res["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


def test_c2_full(sb, ctx):
    t = tensor("c2")
    c = synth.config("c2")
    csf = mttkrp_all_modes(sb, ctx, t, c["rank"], c["seed"])
    for n in range(3):   # oracle CSF (std::stable_sort) at 8M nonzeros
        g = csf.export(n)
        o = oracle.csf_build(t.dims, t.ind, t.vals, n)
        assert g["perm"] == o["perm"].tolist()
        assert all(np.array_equal(a, b) for a, b in zip(g["ids"], o["ids"]))
        assert all(np.array_equal(a, b) for a, b in zip(g["ptr"], o["ptr"]))
        assert np.array_equal(g["vals"].view(np.uint64), o["vals"].view(np.uint64))
    als_check(sb, ctx, t, c["rank"], c["iters"], c["seed"])
    x3_integer_bitexact(sb, ctx, t, c["rank"])


@pytest.mark.parametrize("policy", ["one", "two"])
def test_c2_full_policies(sb, ctx, policy):
    """c2 under the ONE / TWO allocation policies, as `bench.py --policy` runs it: INTERNAL and
    LEAF traversals (bulk row reductions, hot rows, dynamic chunks over a persistent grid,
    256-leaf chunks on the shared tree) for 20 iterations against the oracle."""
    t = tensor("c2")
    c = synth.config("c2")
    ind, vals = dev_coo(t)
    res = sb.cpd_als(ind, vals, t.dims, rank=c["rank"], max_iters=c["iters"], tol=0.0,
                     seed=c["seed"], ctx=ctx, policy=policy)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=c["rank"], max_iters=c["iters"], tol=0.0,
                         seed=c["seed"])
    for n in range(t.nmodes):
        e = rel_fro(res["factors"][n].cpu().numpy(), ref["factors"][n])
        assert e <= ALS_TOL, (n, e)
    assert rel_fro(res["lam"].cpu().numpy(), ref["lam"]) <= ALS_TOL
    assert abs(res["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


@pytest.mark.parametrize("name", ["c3", "c4", "c4r64", "c5"])
def test_large_configs(sb, ctx, name):
    t = tensor(name.replace("r64", "") if name == "c4r64" else name)
    c = synth.config(name)
    csf = mttkrp_all_modes(sb, ctx, t, c["rank"], c["seed"])
    if name != "c4r64":
        for n in range(t.nmodes):
            check_csf_by_library_sort(csf.export(n), t)
    if name == "c5":  # the oracle's CSF (std::stable_sort, C-13) for the mode-0 tree
        g = csf.export(0)
        o = oracle.csf_build(t.dims, t.ind, t.vals, 0)
        assert g["perm"] == o["perm"].tolist()
        assert all(np.array_equal(a, b) for a, b in zip(g["ids"], o["ids"]))
        assert all(np.array_equal(a, b) for a, b in zip(g["ptr"], o["ptr"]))
        assert np.array_equal(g["vals"].view(np.uint64), o["vals"].view(np.uint64))
        del o
    del csf
    if name == "c3":
        x3_integer_bitexact(sb, ctx, t, c["rank"])
    # c3 and c5 (the metric's configs) run the configs' 20 iterations, the bench's code
    # path: leaf tiles of c3's 138 MB mode-0 factor, long-fiber chunks, the gather-policy
    # timing of iterations 2-3; c4 runs 2
    als_check(sb, ctx, t, c["rank"], c["iters"] if name in ("c3", "c5") else 2, c["seed"])


def test_c3_tiled_mttkrp(sb):
    """c3 with leaf tiles forced for single MTTKRPs (AUTO tiles only inside long ALS runs):
    the trees rooted at modes 1 and 2 run on half-L2 tiles of the mode-0 leaf factor."""
    import torch
    t = tensor("c3")
    c = synth.config("c3")
    ctx = sb.Context(0)
    ctx.set_leaf_tiling(0.5)
    ind, vals = dev_coo(t)
    csf = sb.csf_build(ind, vals, t.dims, ctx=ctx)
    R = c["rank"]
    F = oracle.init_factors(t.dims, R, 9)
    ld = sb.padded_ld(R)
    fd = []
    for f in F:
        b = np.zeros((f.shape[0], ld))
        b[:, :R] = f
        fd.append(torch.from_numpy(b).cuda())
    for n in (1, 2):
        M = sb.mttkrp(csf, n, fd, rank=R).cpu().numpy()[:, :R]
        assert rel_fro(M, oracle.mttkrp(t.dims, t.ind, t.vals, F, n)) <= MTTKRP_TOL, n
