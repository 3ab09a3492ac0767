"""Dense brute-force references used to PIN the oracle (tests only).

Each function is the textbook definition written with numpy primitives, independent
of oracle/oracle.cpp: densify the COO tensor, unfold it along a mode, build the
Khatri-Rao product explicitly, multiply (Kolda & Bader unfolding; the ordering of
the KRP columns matches the C-order flattening of the remaining modes, ascending m,
so the product is convention-free — SURVEY.md Q-12).
"""
import numpy as np


def densify(dims, ind, vals):
    X = np.zeros(tuple(int(d) for d in dims))
    np.add.at(X, tuple(np.asarray(a, dtype=np.int64) for a in ind), np.asarray(vals))
    return X


def unfold(X, n):
    return np.moveaxis(X, n, 0).reshape(X.shape[n], -1)


def khatri_rao_except(factors, n):
    K = None
    for m, A in enumerate(factors):
        if m == n:
            continue
        K = A.copy() if K is None else (K[:, None, :] * A[None, :, :]).reshape(-1, A.shape[1])
    return K


def mttkrp_dense(dims, ind, vals, factors, n):
    X = densify(dims, ind, vals)
    return unfold(X, n) @ khatri_rao_except(factors, n)


def kruskal_dense(factors, lam=None):
    R = factors[0].shape[1]
    lam = np.ones(R) if lam is None else lam
    letters = "abcdefgh"[: len(factors)]
    spec = ",".join(f"{c}r" for c in letters) + ",r->" + letters
    return np.einsum(spec, *factors, lam)


def fit_dense(X, factors, lam):
    Z = kruskal_dense(factors, lam)
    return 1.0 - np.linalg.norm((X - Z).ravel()) / np.linalg.norm(X.ravel())
