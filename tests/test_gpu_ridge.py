"""C-7's ridge branch on the GPU against the oracle (PAPER.md:194 V-dagger, realised as
potrf/potrs at PAPER.md:387; reading Q-14: pivot test 1e-12 * max diag, one retry with
V + 1e-12 trace(V)/R I, else SINGULAR).

The initial factors are built so that iteration 1's first mode update takes the retry and is
rescued, on both sides, with a well-defined answer:
  * A_2's column r is supported on rows where its other columns are zero, so G_2[r, s] = 0
    for s != r and V_0 = G_1 * G_2 has row/column r zero off the diagonal: V's r-th pivot
    is exactly V_rr for Cholesky (oracle) and Gauss-Jordan (GPU) alike;
  * A_1's column r is scaled by kappa so that V_rr = 0.6e-12 * max diag: the first attempt
    fails (0.6e-12 max <= 1e-12 max) and the retried pivot V_rr + 1e-12 tr/R passes.
The rescued solve along the decoupled axis is a plain division x_r = m_r / (V_rr + delta),
so the two sides agree to rounding; later modes see well-conditioned V.  The same input with
kappa = 0 (V_rr = 0: the retried pivot delta < 1e-12 max diag) is SINGULAR on both sides.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALS_TOL, rel_fro

pytestmark = pytest.mark.gpu

R, r = 4, 3


def _init(t, kappa):
    rng = np.random.default_rng(77)
    A = [rng.random((int(d), R)) for d in t.dims]
    I2 = int(t.dims[2])
    h = I2 // 2
    A[2][:h, r] = 0.0       # column r lives on rows h.. only
    A[2][h:, :r] = 0.0      # the other columns on rows ..h only
    # V_0 = G_1 * G_2 (Hadamard): scale A_1[:, r] so that V_rr = 0.6e-12 * max_{j<r} V_jj
    G1, G2 = A[1].T @ A[1], A[2].T @ A[2]
    V = G1 * G2
    mx = max(V[j, j] for j in range(r))
    if kappa is None:
        kappa = np.sqrt(0.6e-12 * mx / V[r, r])
    A[1][:, r] *= kappa
    return A, kappa


def _branch(A):
    """(first attempt fails, retry passes) for V_0 from these factors, in closed form."""
    G1, G2 = A[1].T @ A[1], A[2].T @ A[2]
    V = G1 * G2
    assert np.all(V[r, :r] == 0.0) and np.all(V[:r, r] == 0.0)
    mx = np.max(np.diag(V))
    delta = 1e-12 * np.trace(V) / R
    return V[r, r] <= 1e-12 * mx, V[r, r] + delta > 1e-12 * (mx + delta)


@pytest.fixture(scope="module")
def sb(cuda_ok):
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as m
    return m


@pytest.mark.parametrize("iters", [1, 4])
def test_ridge_rescue_matches_oracle(sb, iters):
    t = synth.generate_config("c1")
    A, _ = _init(t, None)
    fails_first, rescued = _branch(A)
    assert fails_first and rescued  # the input does exercise the retry branch
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=iters, tol=0.0, init=A)
    res = sb.cpd_als(t.ind, t.vals, t.dims, rank=R, max_iters=iters, tol=0.0, init=A,
                     out_device=False)
    for n in range(3):
        assert np.all(np.isfinite(res["factors"][n]))
        e = rel_fro(res["factors"][n], ref["factors"][n])
        assert e <= ALS_TOL, (n, e)
    assert rel_fro(res["lam"], ref["lam"]) <= ALS_TOL
    assert abs(res["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])
    assert np.allclose(res["fit_history"], ref["fit_history"], rtol=ALS_TOL, atol=0)


def test_ridge_too_small_is_singular_on_both(sb):
    t = synth.generate_config("c1")
    A, _ = _init(t, 0.0)
    fails_first, rescued = _branch(A)
    assert fails_first and not rescued
    with pytest.raises(oracle.OracleError) as e:
        oracle.cpd_als(t.dims, t.ind, t.vals, rank=R, max_iters=2, tol=0.0, init=A)
    assert e.value.code == oracle.SINGULAR
    with pytest.raises(sb.SingularError):
        sb.cpd_als(t.ind, t.vals, t.dims, rank=R, max_iters=2, tol=0.0, init=A, out_device=False)
