"""NEXT-3: the library's .tns reader/writer, tensor statistics and the CLI (host-only, CPU).

Pinned to SPEC.md's parse/stats examples (tests/golden/spec_tns_examples.json) and to an
independent pure-Python reader/writer (synth.read_tns / synth.write_tns)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from tests.conftest import ROOT, golden


@pytest.fixture(scope="module")
def sb():
    from paper_1812_05961_b200 import build
    build.build()
    import paper_1812_05961_b200 as m
    return m


def write(tmp_path, name, text):
    p = os.path.join(str(tmp_path), name)
    with open(p, "w") as f:
        f.write(text)
    return p


def test_spec_parse_examples(sb, tmp_path):
    g = golden("spec_tns_examples.json")
    for k, case in enumerate(g["parse_ok"]):
        t = sb.read_tns(write(tmp_path, f"ok{k}.tns", case["text"]))
        assert list(t.dims) == case["dims"] and t.nnz == case["nnz"]
        assert t.vals.tolist() == case["vals"]
        assert [a.tolist() for a in t.ind] == case["ind"]


def test_spec_parse_errors(sb, tmp_path):
    g = golden("spec_tns_examples.json")
    for k, case in enumerate(g["parse_err"]):
        p = write(tmp_path, f"err{k}.tns", case["text"])
        if case["line"] == 1 and "3-mode" in case.get("why", ""):
            # a lone "1 1 2.0" is a valid 2-mode line; inside a 3-mode file it is an error
            p = write(tmp_path, f"err{k}b.tns", "1 1 1 1.0\n" + case["text"])
            with pytest.raises(sb.BadInputError, match="line 2"):
                sb.read_tns(p)
            continue
        with pytest.raises(sb.BadInputError) as e:
            sb.read_tns(p)
        if case["line"]:
            assert f"line {case['line']}:" in str(e.value)
        else:
            assert "no nonzeros" in str(e.value)
    with pytest.raises(sb.BadInputError):
        sb.read_tns(os.path.join(str(tmp_path), "missing.tns"))


def test_spec_stats_examples(sb):
    for case in golden("spec_tns_examples.json")["stats"]:
        c = np.array(case["coords"], dtype=np.uint32)
        st = sb.coo_stats([c[:, m] for m in range(3)], np.ones(len(c)), case["dims"])
        assert st["density"] == case["density"]
        assert st["nnz"] == len(c) and st["dims"] == case["dims"]


def test_stats_against_numpy(sb):
    t = synth.generate((300, 40, 900), 5000, [("zipf", 1.2), ("uniform",), ("zipf", 1.0)], "u01",
                       seed=4)
    st = sb.coo_stats(t.ind, t.vals, t.dims)
    for m in range(3):
        cnt = np.bincount(t.ind[m], minlength=t.dims[m])
        assert st["nonempty_slices"][m] == int((cnt > 0).sum())
        assert st["max_slice_nnz"][m] == int(cnt.max())
    assert st["density"] == 5000 / (300.0 * 40.0 * 900.0)


@pytest.mark.parametrize("N", [3, 4, 5])
def test_round_trip_against_python_reader_writer(sb, tmp_path, N):
    t = synth.random_tiny(40 + N, nmodes=N, max_dim=9, max_nnz=300, dups=True)
    vals = np.random.default_rng(N).standard_normal(t.nnz) * 1e3  # arbitrary doubles
    a = os.path.join(str(tmp_path), "lib.tns")
    sb.write_tns(a, t.ind, vals, t.dims)
    ref = synth.read_tns(a)                      # independent reader of the library's output
    for m in range(N):
        assert np.array_equal(ref.ind[m], t.ind[m])
    assert np.array_equal(ref.vals.view(np.uint64), vals.view(np.uint64))  # shortest round trip
    b = os.path.join(str(tmp_path), "py.tns")
    synth.write_tns(synth.SparseTensor(t.dims, t.ind, vals), b)
    got = sb.read_tns(b)                         # library reader of the independent writer
    for m in range(N):
        assert np.array_equal(got.ind[m], t.ind[m])
    assert np.array_equal(got.vals.view(np.uint64), vals.view(np.uint64))
    assert tuple(got.dims) == tuple(int(x.max()) + 1 for x in t.ind)


def test_multichunk_parse_and_error_line(sb, tmp_path):
    """A multi-megabyte file is parsed by several threads: order, dims and the global line
    number of an error must not depend on the chunking."""
    t = synth.generate((5000, 700, 3000), 150_000, [("zipf", 1.1)] * 3, "ratings", seed=9)
    p = os.path.join(str(tmp_path), "big.tns")
    synth.write_tns(t, p)
    assert os.path.getsize(p) > 2 << 20
    got = sb.read_tns(p)
    assert got.nnz == t.nnz
    for m in range(3):
        assert np.array_equal(got.ind[m], t.ind[m])
    assert np.array_equal(got.vals, t.vals)
    lines = open(p).read().splitlines()
    bad = len(lines) - 17
    lines[bad - 1] = "1 2 x 3.0"
    q = os.path.join(str(tmp_path), "bad.tns")
    with open(q, "w") as f:
        f.write("\n".join(lines) + "\n")
    with pytest.raises(sb.BadInputError, match=f"line {bad}:"):
        sb.read_tns(q)


def test_cli_stats(sb, tmp_path):
    p = write(tmp_path, "s.tns", "1 1 1 2.0\n2 2 2 3.0\n2 1 2 1.0\n")
    r = subprocess.run([sys.executable, "-m", "paper_1812_05961_b200", "stats", p, "--json"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    st = json.loads(r.stdout)
    assert st["dims"] == [2, 2, 2] and st["nnz"] == 3 and st["density"] == 3 / 8
    assert st["nonempty_slices"] == [2, 2, 2] and st["max_slice_nnz"] == [2, 2, 2]
