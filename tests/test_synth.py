"""The seeded input recipe (synth/): determinism, exact nnz, shapes."""
import os

import numpy as np

import synth
from tests.conftest import golden


def test_generate_deterministic_and_distinct():
    a = synth.generate((300, 200, 100), 20_000, [("zipf", 1.1), ("zipf", 1.0), ("uniform",)],
                       "ratings", seed=9)
    b = synth.generate((300, 200, 100), 20_000, [("zipf", 1.1), ("zipf", 1.0), ("uniform",)],
                       "ratings", seed=9)
    assert all(np.array_equal(x, y) for x, y in zip(a.ind, b.ind))
    assert np.array_equal(a.vals, b.vals)
    key = (a.ind[0].astype(np.int64) * 200 + a.ind[1]) * 100 + a.ind[2]
    assert np.unique(key).shape[0] == 20_000
    for m, d in enumerate(a.dims):
        assert a.ind[m].dtype == np.uint32 and a.ind[m].max() < d
    assert set(np.unique(a.vals).tolist()) <= {1.0, 2.0, 3.0, 4.0, 5.0}
    # Zipf: the heaviest slice of the s=1.1 mode holds far more than the uniform one's
    h0 = np.bincount(a.ind[0], minlength=300).max()
    h2 = np.bincount(a.ind[2], minlength=100).max()
    assert h0 > 3 * (20_000 / 300) and h2 < 3 * (20_000 / 100)


def test_c1_config_shape():
    t = synth.generate_config("c1")
    assert t.dims == (100, 80, 60) and t.nnz == 5000
    assert np.all((t.vals >= 0) & (t.vals < 1))
    assert t.meta["rank"] == 8 and t.meta["iters"] == 10


def test_c4_density_matches_table1():
    g = golden("table1_density.json")
    c = synth.config("c4")
    assert list(c["dims"]) == g["dims"] and c["nnz"] == g["nnz"]
    dens = c["nnz"] / np.prod(np.array(c["dims"], dtype=np.float64))
    assert abs(dens - g["density_printed"]) <= g["rel_tol"] * g["density_printed"]


def test_four_mode_and_tns_roundtrip(tmp_path):
    t = synth.generate((20, 10, 8, 5), 500, [("zipf", 1.05)] * 4, "u01", seed=3)
    p = os.path.join(tmp_path, "x.tns")
    synth.write_tns(t, p)
    u = synth.read_tns(p)
    assert all(np.array_equal(x, y) for x, y in zip(t.ind, u.ind))
    assert np.array_equal(t.vals, u.vals)


def test_config_cache_round_trip(tmp_path, monkeypatch):
    """The on-disk cache (manifest + SHA-256) returns the generated tensor bit for bit, and a
    corrupted payload is regenerated, not used."""
    import os
    import synth
    monkeypatch.setenv("SPLATT_SYNTH_CACHE", str(tmp_path))
    monkeypatch.setattr(synth, "_cache_dir", lambda: str(tmp_path))
    ref = synth.generate_config("c2", nnz=200_000, cache=False)
    spec_nnz = 200_000
    # force caching for this small size through the helpers
    spec = dict(dims=list(synth.CONFIGS["c2"]["dims"]), nnz=spec_nnz,
                dists=[list(d) for d in synth.CONFIGS["c2"]["dists"]], values="ratings", seed=2)
    synth._cache_store("c2", spec, ref)
    got = synth._cache_load("c2", spec)
    assert got is not None
    for a, b in zip(got.ind, ref.ind):
        assert np.array_equal(a, b)
    assert np.array_equal(got.vals.view(np.uint64), ref.vals.view(np.uint64))
    binp, _ = synth._cache_paths("c2", spec)
    with open(binp, "r+b") as f:
        f.seek(100)
        f.write(b"\xff\xff")
    assert synth._cache_load("c2", spec) is None
    assert os.path.exists(binp)
