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
