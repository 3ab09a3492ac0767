"""Command line: `.tns` statistics and CP-ALS with Table III-style per-routine timings.

    python -m paper_1812_05961_b200 stats FILE.tns [--json]
    python -m paper_1812_05961_b200 cpd FILE.tns --rank R [--iters 50] [--tol 1e-5]
                                    [--seed 0] [--policy all|one|two] [--device 0]
                                    [--out factors.npz] [--json]

`stats` prints Table I's columns (dimensions, non-zeros, density) plus the
per-mode slice counts.  `cpd` runs splatt_cpd_als_ex on the GPU and prints the fit and the
per-routine times in the categories of Table III.  Parsing is the
library's multi-threaded .tns reader (splatt_tns_read); every arithmetic step runs in the
library's CUDA kernels.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

import paper_1812_05961_b200 as sb


def _stats(args) -> int:
    t0 = time.perf_counter()
    t = sb.read_tns(args.file)
    parse_s = time.perf_counter() - t0
    st = t.stats()
    st["parse_s"] = parse_s
    if args.json:
        print(json.dumps(st))
        return 0
    dims = " x ".join(str(d) for d in st["dims"])
    print(f"{args.file}: {st['nmodes']}-mode tensor {dims}, {st['nnz']} non-zeros, "
          f"density {st['density']:.3E} (parsed in {parse_s:.2f} s)")
    for m in range(st["nmodes"]):
        print(f"  mode {m}: {st['nonempty_slices'][m]} non-empty slices of {st['dims'][m]}, "
              f"largest slice {st['max_slice_nnz'][m]} non-zeros")
    return 0


def _cpd(args) -> int:
    t0 = time.perf_counter()
    t = sb.read_tns(args.file)
    parse_s = time.perf_counter() - t0
    if not 3 <= t.nmodes <= sb.MAX_NMODES:
        print(f"error: CP-ALS needs 3..8 modes, {args.file} has {t.nmodes}", file=sys.stderr)
        return 2
    ctx = sb.Context(args.device)
    try:
        res = sb.cpd_als(t.ind, t.vals, t.dims, rank=args.rank, max_iters=args.iters, tol=args.tol,
                         seed=args.seed, ctx=ctx, out_device=False, stats=True,
                         policy=args.policy)
    except (sb.BadInputError, sb.EmptyTensorError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except sb.SingularError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    s = res["stats"]
    # Table III categories.  Fused or overlapped steps are attributed to the
    # kernel that performs them: the Gram refresh runs inside the row solve ("Inverse"), the
    # Hadamard product of the Grams inside the side-stream inverse, the fit on the side stream.
    table = {
        "MTTKRP": s["t_mttkrp"],
        "Sort (CSF build)": s["t_build"],
        "Inverse (M V^-1 + Gram/norm statistics)": s["t_inverse"],
        "Mat A^TA (initial Grams)": s["t_ata"],
        "Mat norm": s["t_norm"],
        "COMM": s["t_comm"],
        "V^-1 and Hadamard (side stream, overlapped)": s["t_aux_inverse"],
        "CPD fit (side stream, overlapped)": s["t_aux_fit"],
        "ALS loop total": s["t_loop"],
    }
    out = dict(file=args.file, dims=list(t.dims), nnz=t.nnz, rank=args.rank, policy=args.policy,
               iters=res["iters"], fit=res["fit"], fit_history=res["fit_history"].tolist(),
               parse_s=parse_s, sec_per_iter=s["t_loop"] / max(1, res["iters"]),
               times_s=table)
    if args.out:
        np.savez(args.out, lam=res["lam"], **{f"A{m}": a for m, a in enumerate(res["factors"])})
        out["out"] = args.out
    if args.json:
        print(json.dumps(out))
        return 0
    dims = " x ".join(str(d) for d in t.dims)
    print(f"{args.file}: {dims}, {t.nnz} non-zeros (parsed in {parse_s:.2f} s)")
    print(f"CP-ALS rank {args.rank}, policy {args.policy}: {res['iters']} iterations, "
          f"fit {res['fit']:.10f}, {out['sec_per_iter'] * 1e3:.3f} ms/iteration")
    print("per-routine times (s):")
    for k, v in table.items():
        print(f"  {k:<46s} {v:10.6f}")
    if args.out:
        print(f"factors and lambda written to {args.out}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1812_05961_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("stats", help="Table I statistics of a .tns file")
    a.add_argument("file")
    a.add_argument("--json", action="store_true")
    b = sub.add_parser("cpd", help="CP-ALS of a .tns file on the GPU")
    b.add_argument("file")
    b.add_argument("--rank", type=int, required=True)
    b.add_argument("--iters", type=int, default=50)
    b.add_argument("--tol", type=float, default=1e-5)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--policy", default="all", choices=["all", "one", "two"])
    b.add_argument("--device", type=int, default=0)
    b.add_argument("--out", default=None, help="write factors + lambda (.npz)")
    b.add_argument("--json", action="store_true")
    args = ap.parse_args(argv)
    return _stats(args) if args.cmd == "stats" else _cpd(args)


if __name__ == "__main__":
    sys.exit(main())
