"""Multi-rank path on CPU: world size 2 over gloo (no GPU).

The sharded ALS partitions each mode's root slices with
the library's host-only splatt_partition (C-14), lets every rank compute the MTTKRP and the
row solves of its own rows, all-reduces the Gram / inner-product partials (sum) and column
maxima (max), and all-gathers the owned rows.  Here each rank does its local arithmetic with
the oracle and the exchange with torch.distributed(gloo); the result must equal the
single-process mode update, and the ranks' local CSFs must concatenate to the global CSF.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tensor():
    import synth
    return synth.generate((300, 120, 200), 6000, [("zipf", 1.2), ("zipf", 1.0), ("uniform",)],
                          "ratings", seed=77)


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_1812_05961_b200 as sb
        t = _tensor()
        R = 5
        A = oracle.init_factors(t.dims, R, 3)
        G = [oracle.gram(a) for a in A]
        out = {}
        for n in range(3):
            w = np.bincount(t.ind[n], minlength=t.dims[n])
            b = sb.partition(w, world)                          # the library's C-14 cut
            lo, hi = int(b[rank]), int(b[rank + 1])
            own = (t.ind[n] >= lo) & (t.ind[n] < hi)
            lind = [a[own] for a in t.ind]
            lval = t.vals[own]
            # local CSF is a contiguous slice-range of the global one
            csf_local = oracle.csf_build(t.dims, lind, lval, n) if lval.size else None
            M = oracle.mttkrp(t.dims, lind, lval, A, n) if lval.size else np.zeros((t.dims[n], R))
            V = oracle.hadamard_except(G, n)
            An = np.zeros_like(A[n])
            An[lo:hi] = oracle.cholesky_solve(V, M[lo:hi]) if hi > lo else An[lo:hi]
            part = np.concatenate([(An[lo:hi].T @ An[lo:hi]).ravel(),
                                   [np.sum(M[lo:hi] * An[lo:hi])]])
            cmax = np.abs(An[lo:hi]).max(axis=0) if hi > lo else np.zeros(R)
            ts = torch.from_numpy(part.copy())
            tm = torch.from_numpy(cmax.copy())
            dist.all_reduce(ts, op=dist.ReduceOp.SUM)
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            # all-gather of uneven row blocks (pad to the largest block)
            maxrows = int(max(b[g + 1] - b[g] for g in range(world)))
            blk = torch.zeros((maxrows, R), dtype=torch.float64)
            blk[: hi - lo] = torch.from_numpy(An[lo:hi])
            gathered = [torch.zeros_like(blk) for _ in range(world)]
            dist.all_gather(gathered, blk)
            full = np.zeros_like(A[n])
            for g in range(world):
                full[b[g]:b[g + 1]] = gathered[g][: b[g + 1] - b[g]].numpy()
            out[n] = dict(bounds=b.tolist(), stats=ts.numpy(), cmax=tm.numpy(), A=full,
                          csf=csf_local)
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced in the parent
        q.put((rank, repr(e)))


@pytest.mark.timeout(300)
def test_two_rank_mode_update_equals_single_process():
    import oracle
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]

    t = _tensor()
    R = 5
    A = oracle.init_factors(t.dims, R, 3)
    G = [oracle.gram(a) for a in A]
    for n in range(3):
        # every rank computed the same cut and the same exchanged result
        assert res[0][n]["bounds"] == res[1][n]["bounds"]
        M = oracle.mttkrp(t.dims, t.ind, t.vals, A, n)
        An = oracle.cholesky_solve(oracle.hadamard_except(G, n), M)
        for r in range(world):
            assert np.allclose(res[r][n]["A"], An, rtol=1e-12, atol=1e-13)
            st = res[r][n]["stats"]
            assert np.allclose(st[:-1].reshape(R, R), An.T @ An, rtol=1e-11, atol=1e-12)
            assert np.isclose(st[-1], np.sum(M * An), rtol=1e-11)
            assert np.allclose(res[r][n]["cmax"], np.abs(An).max(axis=0), rtol=0, atol=0)
        # the ranks' local CSFs concatenate to the global CSF (slices are not split)
        g = oracle.csf_build(t.dims, t.ind, t.vals, n)
        parts = [res[r][n]["csf"] for r in range(world) if res[r][n]["csf"] is not None]
        assert np.array_equal(np.concatenate([p["ids"][0] for p in parts]), g["ids"][0])
        assert np.array_equal(np.concatenate([p["ids"][2] for p in parts]), g["ids"][2])
        assert np.array_equal(np.concatenate([p["vals"] for p in parts]), g["vals"])


def test_partition_balances_zipf_slices():
    import paper_1812_05961_b200 as sb
    t = _tensor()
    for n in range(3):
        w = np.bincount(t.ind[n], minlength=t.dims[n])
        for G in (2, 4, 8):
            b = sb.partition(w, G)
            loads = [int(w[b[g]:b[g + 1]].sum()) for g in range(G)]
            assert sum(loads) == t.nnz
            # optimal cut: max load <= ideal + heaviest slice
            assert max(loads) <= t.nnz / G + w.max()


# ------------------------------------------------------------------ P2 (NEXT-2)
def _p2_expected(w, G, g):
    """Definition: positions [k_g, k_{g+1}) of the slice-major order, k_g = floor(g nnz / G)."""
    P = np.concatenate([[0], np.cumsum(w)]).astype(np.int64)
    nnz = int(P[-1])
    k = [g2 * nnz // G for g2 in range(G + 1)]
    share = set()
    for s in range(len(w)):
        a = max(int(P[s]), k[g]) - int(P[s])
        b = min(int(P[s + 1]), k[g + 1]) - int(P[s])
        if b > a:
            share.add((s, a, b))
    rowb = [0] + [int(np.searchsorted(P[:-1], k[g2], side="left")) for g2 in range(1, G)] + [len(w)]
    split = sorted({int(np.searchsorted(P, k[g2], side="right")) - 1 for g2 in range(1, G)
                    if 0 < k[g2] < nnz and P[int(np.searchsorted(P, k[g2], side="right")) - 1] < k[g2]})
    return share, rowb, split


def test_partition_nnz_matches_definition():
    import paper_1812_05961_b200 as sb
    rng = np.random.default_rng(21)
    for trial in range(300):
        S = int(rng.integers(1, 25))
        w = rng.integers(0, 12, S) * (rng.random(S) < 0.8)
        if trial % 7 == 0:
            w[int(rng.integers(0, S))] += 200  # one slice spanning several cuts
        if w.sum() == 0:
            w[0] = 1
        G = int(rng.integers(1, 9))
        for g in range(G):
            got = sb.partition_nnz(w, G, g)
            share, rowb, split = _p2_expected(w, G, g)
            mine = {(s, 0, int(w[s])) for s in range(*got["full"]) if w[s] > 0}
            mine |= {p for p in got["parts"] if p[2] > p[1]}
            assert mine == share, (w.tolist(), G, g, got)
            assert got["row_bounds"] == rowb
            assert got["split"] == split
            assert len(got["parts"]) <= 2 and len(got["split"]) <= G - 1


def _p2_worker(rank, world, port, q):
    """One rank of the P2 mode update: equal nonzero ranges (slices split), local MTTKRP,
    all-reduce of the split slices' partial rows into their owners, solve of the owned rows,
    statistics all-reduce and row all-gather."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_1812_05961_b200 as sb
        t = _tensor()
        R = 5
        A = oracle.init_factors(t.dims, R, 3)
        G = [oracle.gram(a) for a in A]
        out = {}
        for n in range(3):
            w = np.bincount(t.ind[n], minlength=t.dims[n])
            p = sb.partition_nnz(w, world, rank)
            rb = p["row_bounds"]
            lo_full, hi_full = p["full"]
            sel = (t.ind[n] >= lo_full) & (t.ind[n] < hi_full)
            for s, a, b in p["parts"]:
                in_s = t.ind[n] == s
                rk = np.cumsum(in_s) - in_s  # rank within the slice, input order
                sel |= in_s & (rk >= a) & (rk < b)
            lind = [x[sel] for x in t.ind]
            lval = t.vals[sel]
            M = oracle.mttkrp(t.dims, lind, lval, A, n) if lval.size else np.zeros((t.dims[n], R))
            slots = torch.zeros((max(1, len(p["split"])), R), dtype=torch.float64)
            for k, s in enumerate(p["split"]):
                if any(pp[0] == s for pp in p["parts"]):
                    slots[k] = torch.from_numpy(M[s])
            dist.all_reduce(slots, op=dist.ReduceOp.SUM)
            for k, s in enumerate(p["split"]):
                if rb[rank] <= s < rb[rank + 1]:
                    M[s] = slots[k].numpy()
            lo, hi = rb[rank], rb[rank + 1]
            V = oracle.hadamard_except(G, n)
            An = np.zeros_like(A[n])
            if hi > lo:
                An[lo:hi] = oracle.cholesky_solve(V, M[lo:hi])
            maxrows = int(max(rb[g + 1] - rb[g] for g in range(world)))
            blk = torch.zeros((max(1, maxrows), R), dtype=torch.float64)
            blk[: hi - lo] = torch.from_numpy(An[lo:hi])
            gathered = [torch.zeros_like(blk) for _ in range(world)]
            dist.all_gather(gathered, blk)
            full = np.zeros_like(A[n])
            for g in range(world):
                full[rb[g]:rb[g + 1]] = gathered[g][: rb[g + 1] - rb[g]].numpy()
            out[n] = dict(A=full, local_nnz=int(lval.size))
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced in the parent
        q.put((rank, repr(e)))


@pytest.mark.timeout(300)
def test_two_rank_p2_mode_update_equals_single_process():
    import oracle
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_p2_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    t = _tensor()
    R = 5
    A = oracle.init_factors(t.dims, R, 3)
    G = [oracle.gram(a) for a in A]
    for n in range(3):
        M = oracle.mttkrp(t.dims, t.ind, t.vals, A, n)
        An = oracle.cholesky_solve(oracle.hadamard_except(G, n), M)
        # equal shares: |local_0 - local_1| <= 1
        assert abs(res[0][n]["local_nnz"] - res[1][n]["local_nnz"]) <= 1
        for r in range(world):
            assert np.allclose(res[r][n]["A"], An, rtol=1e-12, atol=1e-13)
