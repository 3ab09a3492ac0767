"""NEXT-3 on the GPU: `python -m paper_1812_05961_b200 cpd FILE.tns` equals the API call on the
same tensor, and both equal the oracle (1e-7, as the other CP-ALS parity tests)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth
from tests.conftest import ROOT
from tests.gpu_util import ALS_TOL, rel_fro

pytestmark = pytest.mark.gpu


def test_cli_cpd_matches_api_and_oracle(cuda_ok, tmp_path):
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as sb
    t = synth.generate_config("c1")
    p = os.path.join(str(tmp_path), "c1.tns")
    sb.write_tns(p, t.ind, t.vals, t.dims)
    out = os.path.join(str(tmp_path), "f.npz")
    r = subprocess.run([sys.executable, "-m", "paper_1812_05961_b200", "cpd", p, "--rank", "8",
                        "--iters", "10", "--tol", "0", "--seed", "1", "--out", out, "--json"],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr
    res = json.loads(r.stdout)
    assert res["iters"] == 10 and res["nnz"] == t.nnz
    ref = oracle.cpd_als(t.dims, t.ind, t.vals, rank=8, max_iters=10, tol=0.0, seed=1)
    assert abs(res["fit"] - ref["fit"]) <= ALS_TOL * abs(ref["fit"])
    f = np.load(out)
    for m in range(3):
        assert rel_fro(f[f"A{m}"], ref["factors"][m]) <= ALS_TOL
    assert rel_fro(f["lam"], ref["lam"]) <= ALS_TOL
    assert set(res["times_s"]) >= {"MTTKRP", "Sort (CSF build)", "ALS loop total"}


def test_cli_cpd_errors(cuda_ok, tmp_path):
    p = os.path.join(str(tmp_path), "two.tns")
    with open(p, "w") as f:
        f.write("1 1 1.0\n2 2 2.0\n")
    r = subprocess.run([sys.executable, "-m", "paper_1812_05961_b200", "cpd", p, "--rank", "2"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 2 and "3..8 modes" in r.stderr
