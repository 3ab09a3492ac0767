"""The sharded (multi-rank) CP-ALS driver on one B200 through the loopback communicator.

G logical ranks (host threads, one context + stream each) run the same splatt_cpd_als as
the NCCL ranks of a multi-GPU job: per-mode C-14 partition, local CSFs of the owned
nonzeros, local MTTKRP + solves, all-reduce of the Gram/inner/colmax statistics and
all-gather of the owned rows.  Every rank must return the same model,
equal to the single-rank result up to summation order and to the oracle within 1e-7.
"""
import threading

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALS_TOL, rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb(cuda_ok):
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as m
    return m


def run_ranks(sb, t, G, R, iters, seed, tol=0.0, partition="slices", exchange="collective",
              calls=1, deterministic=False):
    import torch
    grp = sb.Loopback(G)
    results, errors = [None] * G, []

    def worker(r):
        try:
            stream = torch.cuda.Stream(0)
            ctx = sb.Context(0, stream=stream)
            ctx.set_comm_loopback(grp, r)
            ctx.set_partition(partition)
            ctx.set_exchange(exchange)
            ctx.set_deterministic(deterministic)
            with torch.cuda.stream(stream):
                ind = [torch.from_numpy(a.view(np.int32)).cuda() for a in t.ind]
                vals = torch.from_numpy(t.vals).cuda()
            stream.synchronize()
            for _ in range(calls):  # repeated calls reuse the context's arenas / factor slab
                res = sb.cpd_als(ind, vals, t.dims, rank=R, max_iters=iters, tol=tol, seed=seed,
                                 ctx=ctx, out_device=False, stats=True)
            results[r] = res
            ctx.close()
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    grp.close()
    assert not errors, errors
    return results


@pytest.mark.parametrize("partition", ["slices", "nnz", "auto"])
@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_sharded_als_matches_single_rank_and_oracle(sb, G, partition):
    t = synth.generate((4000, 1100, 7500), 150_000, [("zipf", 1.1)] * 3, "ratings", seed=22)
    R, iters = 16, 5
    single = run_ranks(sb, t, 1, R, iters, seed=5)[0]
    multi = run_ranks(sb, t, G, R, iters, seed=5, partition=partition)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=iters, seed=5)
    for r in range(G):
        assert multi[r]["stats"]["nranks"] == G
        for n in range(3):
            # every rank holds the identical model
            assert np.array_equal(multi[r]["factors"][n], multi[0]["factors"][n])
            assert rel_fro(multi[r]["factors"][n], single["factors"][n]) <= 1e-10
            assert rel_fro(multi[r]["factors"][n], ref["factors"][n]) <= ALS_TOL
        assert rel_fro(multi[r]["lam"], ref["lam"]) <= ALS_TOL
        assert abs(multi[r]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])
    # the ranks split the nonzeros of every mode (local CSF leaves sum to nnz); P2 shares
    # are equal to within one nonzero
    for n in range(3):
        loc = [multi[r]["stats"]["csf_nodes"][n][2] for r in range(G)]
        assert sum(loc) == t.nnz
        if partition == "nnz":
            assert max(loc) - min(loc) <= 1


def test_p2_slice_spanning_many_ranks(sb):
    """P2 with one slice holding ~40% of the nonzeros: it is split over 4+ of 8 ranks, whose
    partial rows must all reach its owner."""
    rng = np.random.default_rng(31)
    base = synth.generate((500, 300, 800), 30_000, [("uniform",)] * 3, "u01", seed=31)
    heavy = np.unique(np.stack([np.full(20_000, 7, np.uint32),
                                rng.integers(0, 300, 20_000).astype(np.uint32),
                                rng.integers(0, 800, 20_000).astype(np.uint32)], 1), axis=0)
    coords = np.concatenate([np.stack(base.ind, 1), heavy])
    coords = np.unique(coords, axis=0)
    coords = coords[rng.permutation(len(coords))]
    t = synth.SparseTensor((500, 300, 800), [coords[:, m].copy() for m in range(3)],
                           rng.random(len(coords)))
    multi = run_ranks(sb, t, 8, 8, 3, seed=4, partition="nnz")
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=3, seed=4)
    for r in range(8):
        for n in range(3):
            assert rel_fro(multi[r]["factors"][n], ref["factors"][n]) <= ALS_TOL
        assert abs(multi[r]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


@pytest.mark.parametrize("partition", ["slices", "nnz"])
def test_sharded_als_four_modes_with_empty_ranks(sb, partition):
    # 4-mode tensor whose last mode has fewer slices than ranks: some ranks own no rows
    t = synth.generate((300, 200, 100, 3), 20_000, [("zipf", 1.05)] * 4, "u01", seed=9)
    R = 8
    multi = run_ranks(sb, t, 4, R, 3, seed=2, partition=partition)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=3, seed=2)
    for r in range(4):
        for n in range(4):
            assert rel_fro(multi[r]["factors"][n], ref["factors"][n]) <= ALS_TOL
        assert abs(multi[r]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


def test_sharded_als_tol_stop(sb):
    t = synth.generate_config("c1")
    multi = run_ranks(sb, t, 2, 8, 100, seed=1, tol=1e-4)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=100, tol=1e-4, seed=1)
    for r in range(2):
        assert multi[r]["iters"] == ref["iters"]
        assert abs(multi[r]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


def test_nccl_single_rank_sharded_path(sb):
    """A one-rank NCCL communicator: the real NCCL calls (all-reduce sum/max, grouped
    broadcasts) and the sharded driver (bincount, C-14 cut, compaction, local CSFs) on
    this GPU; the model must equal the oracle's."""
    import torch
    t = synth.generate((4000, 1100, 7500), 150_000, [("zipf", 1.1)] * 3, "ratings", seed=22)
    stream = torch.cuda.Stream(0)
    ctx = sb.Context(0, stream=stream)
    ctx.set_comm(single=True)
    with torch.cuda.stream(stream):
        ind = [torch.from_numpy(a.view(np.int32)).cuda() for a in t.ind]
        vals = torch.from_numpy(t.vals).cuda()
    stream.synchronize()
    res = sb.cpd_als(ind, vals, t.dims, rank=16, max_iters=5, seed=5, ctx=ctx, out_device=False,
                     stats=True)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=16, max_iters=5, seed=5)
    assert res["stats"]["nranks"] == 1 and res["stats"]["t_comm"] > 0
    for n in range(3):
        assert rel_fro(res["factors"][n], ref["factors"][n]) <= ALS_TOL
    assert abs(res["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


def test_auto_partition_picks_p2_for_heavy_mode(sb):
    """AUTO: a mode whose heaviest slice holds 40% of 4M nonzeros gets the equal-nnz split
    (shares within one nonzero), the others stay whole-slice; the model still matches."""
    rng = np.random.default_rng(41)
    base = synth.generate((20_000, 3_000, 9_000), 2_400_000, [("uniform",)] * 3, "ratings", seed=41)
    heavy = np.stack([np.full(1_600_000, 123, np.uint32),
                      rng.integers(0, 3_000, 1_600_000).astype(np.uint32),
                      rng.integers(0, 9_000, 1_600_000).astype(np.uint32)], 1)
    coords = np.unique(np.concatenate([np.stack(base.ind, 1), heavy]), axis=0)
    coords = coords[rng.permutation(len(coords))]
    t = synth.SparseTensor((20_000, 3_000, 9_000), [coords[:, m].copy() for m in range(3)],
                           rng.integers(1, 6, len(coords)).astype(np.float64))
    multi = run_ranks(sb, t, 4, 8, 2, seed=6, partition="auto")
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=2, seed=6)
    for r in range(4):
        for n in range(3):
            assert rel_fro(multi[r]["factors"][n], ref["factors"][n]) <= ALS_TOL
        assert abs(multi[r]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])
    loc0 = [multi[r]["stats"]["csf_nodes"][0][2] for r in range(4)]
    assert sum(loc0) == t.nnz and max(loc0) - min(loc0) <= 1  # mode 0: P2


# ---- SPLATT_XCHG_PEER: the row solve stores its rows straight into the peers' factor
# matrices (splatt_b200.h, splatt_ctx_set_exchange); the all-gather never runs.  The model must
# be bit-identical to the collective exchange on every rank (the same values are stored) and
# match the oracle.

@pytest.mark.parametrize("partition", ["slices", "nnz"])
@pytest.mark.parametrize("G,R", [(2, 16), (3, 35), (8, 16), (4, 80)])  # R = 80: the FMA-pipe solve
def test_peer_exchange_bit_identical_to_collective(sb, G, R, partition):
    t = synth.generate((4000, 1100, 7500), 150_000, [("zipf", 1.1)] * 3, "ratings", seed=22)
    iters = 4
    # (deterministic ROOT seams: two runs of the same exchange are then bit-identical too)
    coll = run_ranks(sb, t, G, R, iters, seed=5, partition=partition, deterministic=True)
    peer = run_ranks(sb, t, G, R, iters, seed=5, partition=partition, exchange="peer", calls=2,
                     deterministic=True)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=iters, seed=5)
    for r in range(G):
        assert coll[r]["stats"]["exchange"] == 0 and peer[r]["stats"]["exchange"] == 1
        for n in range(3):
            assert np.array_equal(peer[r]["factors"][n], coll[r]["factors"][n])
            assert rel_fro(peer[r]["factors"][n], ref["factors"][n]) <= ALS_TOL
        assert np.array_equal(peer[r]["lam"], coll[r]["lam"])
        assert peer[r]["fit"] == coll[r]["fit"]
        assert abs(peer[r]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


def test_peer_exchange_four_modes_empty_ranks_and_growth(sb):
    """4-mode trees (second-generation ROOT kernel), ranks that own no rows of the last mode,
    and a context whose factor slab grows between calls (a small tensor first)."""
    import torch
    small = synth.generate((60, 50, 40, 3), 2_000, [("zipf", 1.05)] * 4, "u01", seed=8)
    t = synth.generate((300, 200, 100, 3), 20_000, [("zipf", 1.05)] * 4, "u01", seed=9)
    G, R = 4, 8
    grp = sb.Loopback(G)
    results, errors = [None] * G, []

    def worker(r):
        try:
            stream = torch.cuda.Stream(0)
            ctx = sb.Context(0, stream=stream)
            ctx.set_comm_loopback(grp, r)
            ctx.set_exchange("peer")
            out = []
            for x in (small, t):
                with torch.cuda.stream(stream):
                    ind = [torch.from_numpy(a.view(np.int32)).cuda() for a in x.ind]
                    vals = torch.from_numpy(x.vals).cuda()
                stream.synchronize()
                out.append(sb.cpd_als(ind, vals, x.dims, rank=R, max_iters=3, seed=2, ctx=ctx,
                                      out_device=False, stats=True))
            results[r] = out
            ctx.close()
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    grp.close()
    assert not errors, errors
    for k, x in enumerate((small, t)):
        ref = oracle.cpd_als(x.dims, x.ind, x.vals, rank=R, max_iters=3, seed=2)
        for r in range(G):
            assert results[r][k]["stats"]["exchange"] == 1
            for n in range(4):
                assert rel_fro(results[r][k]["factors"][n], ref["factors"][n]) <= ALS_TOL
            assert abs(results[r][k]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


def test_peer_exchange_tol_stop(sb):
    t = synth.generate_config("c1")
    multi = run_ranks(sb, t, 2, 8, 100, seed=1, tol=1e-4, exchange="peer")
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=100, tol=1e-4, seed=1)
    for r in range(2):
        assert multi[r]["iters"] == ref["iters"]
        assert abs(multi[r]["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])


def test_peer_exchange_one_rank_nccl(sb):
    """A one-rank NCCL communicator: no peer to store to, but the mapping exchange runs for
    real (cudaIpcGetMemHandle on the factor slab, ncclAllGather of the handle records, the
    failure-flag all-reduce); the model is the oracle's."""
    import torch
    t = synth.generate((400, 300, 200), 20_000, [("zipf", 1.1)] * 3, "ratings", seed=3)
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=3, seed=5)
    stream = torch.cuda.Stream(0)
    ctx = sb.Context(0, stream=stream)
    ctx.set_comm(single=True)
    ctx.set_exchange("peer")
    with torch.cuda.stream(stream):
        ind = [torch.from_numpy(a.view(np.int32)).cuda() for a in t.ind]
        vals = torch.from_numpy(t.vals).cuda()
    stream.synchronize()
    res = sb.cpd_als(ind, vals, t.dims, rank=8, max_iters=3, seed=5, ctx=ctx, out_device=False,
                     stats=True)
    assert res["stats"]["exchange"] == 1 and res["stats"]["nranks"] == 1
    for n in range(3):
        assert rel_fro(res["factors"][n], ref["factors"][n]) <= ALS_TOL
