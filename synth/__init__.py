"""Seeded synthetic sparse-tensor generators — shared input recipe, NO method arithmetic.

This module is the only code shared by the oracle side (``oracle/``) and the CUDA
side (``paper_1812_05961_b200``).  It draws coordinates and values; it never sorts
into CSF, never computes an MTTKRP, a Gram, a solve or a fit.  Random numbers the
*method* draws (factor initialisation) are NOT produced here:
both sides implement the same counter-based splitmix64 generator independently.

Recipe (SURVEY.md §8(d) "Generator spec"; DESIGN.md §3 restates it):
  1. rng = numpy PCG64(seed), seed = config index (c1..c5 -> 1..5).
  2. perm[n] = rng.permutation(I_n) for every mode, in mode order (labels of Zipf
     ranks are scattered).
  3. per-mode draw of b indices: uniform -> perm[n][rng.integers(0, I_n, b)];
     Zipf(s) -> perm[n][searchsorted(cdf_n, rng.random(b), 'right')] with
     cdf_n = cumsum(k^-s, k=1..I_n)/sum (truncated Zipf).
  4. batches: b = nnz first, then b = ceil(nnz/4); within a batch modes are drawn
     0..N-1 in order; duplicates are removed keeping the first occurrence in draw
     order; stop once >= nnz distinct coordinates exist and keep the first nnz
     distinct ones in draw order (the configs state an exact nnz).
  5. values drawn after all coordinates, in kept order: U[0,1) (c1, c5), integer
     ratings 1..5 (c2, c3), lognormal(0, 1) (c4).

The paper's datasets (YELP, NELL-2, NETFLIX-shaped; Table I)
are not available; these seeded tensors stand in for them (BASELINE.json configs).
torch CPU ops are used only as faster, bit-identical library primitives
(searchsorted, stable sort) for steps 3-4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["SparseTensor", "CONFIGS", "config", "generate", "generate_config",
           "random_tiny", "planted", "full_kruskal", "write_tns", "read_tns"]


@dataclass
class SparseTensor:
    """COO tensor: ``ind[m]`` is a uint32 array of 0-based mode-m indices."""
    dims: tuple
    ind: list
    vals: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def nmodes(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def coords(self) -> np.ndarray:
        return np.stack([np.asarray(a, dtype=np.int64) for a in self.ind], axis=1)


# BASELINE.json "configs" (BJ:7-11).  'dists' per mode: ('uniform',) or ('zipf', s).
CONFIGS = {
    "c1": dict(dims=(100, 80, 60), nnz=5_000, dists=[("uniform",)] * 3, values="u01",
               rank=8, iters=10, seed=1),
    "c2": dict(dims=(40_000, 11_000, 75_000), nnz=8_000_000, dists=[("zipf", 1.1)] * 3,
               values="ratings", rank=35, iters=20, seed=2),
    "c3": dict(dims=(480_000, 18_000, 2_000), nnz=100_000_000,
               dists=[("zipf", 1.0), ("zipf", 1.2), ("uniform",)], values="ratings",
               rank=35, iters=20, seed=3),
    "c4": dict(dims=(12_000, 9_000, 29_000), nnz=77_000_000, dists=[("uniform",)] * 3,
               values="lognormal", rank=35, iters=20, seed=4),
    "c4r64": dict(dims=(12_000, 9_000, 29_000), nnz=77_000_000, dists=[("uniform",)] * 3,
                  values="lognormal", rank=64, iters=20, seed=4),
    "c5": dict(dims=(200_000, 50_000, 10_000, 500), nnz=150_000_000,
               dists=[("zipf", 1.05)] * 4, values="u01", rank=16, iters=20, seed=5),
}


def config(name: str) -> dict:
    return dict(CONFIGS[name])


def _searchsorted_right(cdf: np.ndarray, u: np.ndarray) -> np.ndarray:
    try:
        import torch
        return torch.searchsorted(torch.from_numpy(cdf), torch.from_numpy(u), right=True).numpy()
    except Exception:  # pragma: no cover - torch is always present in this image
        return np.searchsorted(cdf, u, "right")


def _first_occurrences(keys: np.ndarray) -> np.ndarray:
    """Positions of the first occurrence of each distinct key, ascending."""
    try:
        import torch
        tk = torch.from_numpy(keys.view(np.int64))
        sk, order = torch.sort(tk, stable=True)
        sk = sk.numpy(); order = order.numpy()
    except Exception:  # pragma: no cover
        order = np.argsort(keys, kind="stable"); sk = keys[order]
    start = np.empty(sk.shape[0], dtype=bool)
    if sk.shape[0]:
        start[0] = True
        np.not_equal(sk[1:], sk[:-1], out=start[1:])
    mask = np.zeros(keys.shape[0], dtype=bool)
    mask[order[start]] = True
    return np.flatnonzero(mask)


def _draw_mode(rng, dist, I, perm, b, cdf_cache, n):
    if dist[0] == "uniform":
        r = rng.integers(0, I, b)
    elif dist[0] == "zipf":
        cdf = cdf_cache.get(n)
        if cdf is None:
            w = np.arange(1, I + 1, dtype=np.float64) ** (-float(dist[1]))
            cdf = np.cumsum(w)
            cdf /= cdf[-1]
            cdf_cache[n] = cdf
        r = _searchsorted_right(cdf, rng.random(b))
        np.minimum(r, I - 1, out=r)
    else:
        raise ValueError(f"unknown distribution {dist}")
    return perm[r].astype(np.uint32)


def generate(dims, nnz, dists, values="u01", seed=0) -> SparseTensor:
    """Draw a COO tensor with exactly ``nnz`` distinct coordinates (recipe above)."""
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    cap = 1
    for d in dims:
        cap *= d
    if nnz > cap:
        raise ValueError("nnz exceeds the number of cells")
    if math.prod(dims) >= 2 ** 63:
        raise ValueError("dims too large for the 63-bit dedup key")
    rng = np.random.Generator(np.random.PCG64(seed))
    perms = [rng.permutation(I) for I in dims]
    cdf_cache: dict = {}
    inds = [[] for _ in range(N)]
    keys = []
    total = 0
    b = nnz
    kept = None
    while True:
        batch = [_draw_mode(rng, dists[n], dims[n], perms[n], b, cdf_cache, n) for n in range(N)]
        key = np.zeros(b, dtype=np.uint64)
        for n in range(N):
            key *= np.uint64(dims[n])
            key += batch[n].astype(np.uint64)
        for n in range(N):
            inds[n].append(batch[n])
        keys.append(key)
        total += b
        allk = keys[0] if len(keys) == 1 else np.concatenate(keys)
        first = _first_occurrences(allk)
        if first.shape[0] >= nnz:
            kept = first[:nnz]
            break
        b = (nnz + 3) // 4
    ind = []
    for n in range(N):
        a = inds[n][0] if len(inds[n]) == 1 else np.concatenate(inds[n])
        ind.append(np.ascontiguousarray(a[kept]))
    if values == "u01":
        vals = rng.random(nnz)
    elif values == "ratings":
        vals = rng.integers(1, 6, nnz).astype(np.float64)
    elif values == "lognormal":
        vals = rng.lognormal(0.0, 1.0, nnz)
    else:
        raise ValueError(f"unknown value distribution {values}")
    meta = dict(seed=seed, dists=[list(d) for d in dists], values=values, draws=total)
    return SparseTensor(dims, ind, np.ascontiguousarray(vals, dtype=np.float64), meta)


def _cache_dir():
    import os
    return os.environ.get("SPLATT_SYNTH_CACHE",
                          os.path.join(os.path.expanduser("~"), ".cache", "splatt_b200_synth"))


def _cache_paths(name, spec):
    import hashlib
    import json
    import os
    key = hashlib.sha256(json.dumps(spec, sort_keys=True).encode()).hexdigest()[:16]
    base = os.path.join(_cache_dir(), f"{name}-{key}")
    return base + ".bin", base + ".json"


def _cache_load(name, spec):
    """The cached tensor if its manifest matches `spec` and the payload's SHA-256 checks."""
    import hashlib
    import json
    import os
    binp, manp = _cache_paths(name, spec)
    try:
        with open(manp) as f:
            man = json.load(f)
        if man.get("spec") != spec or os.path.getsize(binp) != man["bytes"]:
            return None
        raw = np.fromfile(binp, dtype=np.uint8)
        if hashlib.sha256(raw.tobytes()).hexdigest() != man["sha256"]:
            return None
    except (OSError, ValueError, KeyError):
        return None
    nnz, N = spec["nnz"], len(spec["dims"])
    ind = [np.frombuffer(raw, dtype="<u4", count=nnz, offset=4 * nnz * m).copy() for m in range(N)]
    vals = np.frombuffer(raw, dtype="<f8", count=nnz, offset=4 * nnz * N).copy()
    return SparseTensor(tuple(spec["dims"]), ind, vals, dict(man.get("meta", {})))


def _cache_store(name, spec, t):
    """Little-endian uint32 indices then float64 values, plus a JSON manifest with the
    recipe and the payload's SHA-256 (SURVEY.md §8(d) generator step 6).  Best effort."""
    import hashlib
    import json
    import os
    binp, manp = _cache_paths(name, spec)
    try:
        os.makedirs(os.path.dirname(binp), exist_ok=True)
        payload = b"".join([np.ascontiguousarray(a, dtype="<u4").tobytes() for a in t.ind] +
                           [np.ascontiguousarray(t.vals, dtype="<f8").tobytes()])
        tmp = binp + f".tmp{os.getpid()}"
        with open(tmp, "wb") as f:
            f.write(payload)
        os.replace(tmp, binp)
        man = dict(spec=spec, bytes=len(payload), sha256=hashlib.sha256(payload).hexdigest(),
                   meta={k: v for k, v in t.meta.items() if isinstance(v, (int, float, str, list))})
        with open(manp + f".tmp{os.getpid()}", "w") as f:
            json.dump(man, f)
        os.replace(manp + f".tmp{os.getpid()}", manp)
    except OSError:
        pass


def generate_config(name: str, seed=None, nnz=None, dims=None, cache=True) -> SparseTensor:
    """A BASELINE.json config (optionally re-seeded or shrunk for parity tests).  Large
    tensors are cached on disk (manifest + SHA-256; SPLATT_SYNTH_CACHE, default
    ~/.cache/splatt_b200_synth) and re-generated whenever the cache does not verify: the
    result is the same either way."""
    c = CONFIGS[name]
    spec = dict(dims=list(dims or c["dims"]), nnz=int(nnz or c["nnz"]),
                dists=[list(d) for d in c["dists"]], values=c["values"],
                seed=int(c["seed"] if seed is None else seed))
    use_cache = cache and spec["nnz"] >= 10_000_000
    t = _cache_load(name, spec) if use_cache else None
    if t is None:
        t = generate(spec["dims"], spec["nnz"], c["dists"], c["values"], spec["seed"])
        if use_cache:
            _cache_store(name, spec, t)
    t.meta.update(config=name, rank=c["rank"], iters=c["iters"])
    return t


def random_tiny(seed, nmodes=3, max_dim=8, max_nnz=64, dups=False, int_values=False) -> SparseTensor:
    """Small random tensors for property tests (SPEC.md:514-516 style)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    dims = tuple(int(x) for x in rng.integers(1, max_dim + 1, nmodes))
    cells = math.prod(dims)
    nnz = int(rng.integers(1, min(max_nnz, cells) + 1))
    if dups:
        coords = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    else:
        flat = rng.choice(cells, size=nnz, replace=False)
        coords = np.stack(np.unravel_index(flat, dims), axis=1)
    vals = (rng.integers(-4, 5, nnz).astype(np.float64) if int_values
            else rng.standard_normal(nnz))
    ind = [np.ascontiguousarray(coords[:, m].astype(np.uint32)) for m in range(nmodes)]
    return SparseTensor(dims, ind, vals, dict(seed=seed))


def full_kruskal(factors, lam=None) -> SparseTensor:
    """Every cell of [[lam; A_0, ..., A_{N-1}]] stored as a nonzero (exact-rank tensor).

    This is the *definition* of a Kruskal tensor (SURVEY.md X-2/X-8 pins), used only
    to build inputs; the resulting values are inputs, not expected outputs.
    """
    dims = tuple(a.shape[0] for a in factors)
    R = factors[0].shape[1]
    lam = np.ones(R) if lam is None else np.asarray(lam, dtype=np.float64)
    grids = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    coords = [g.reshape(-1) for g in grids]
    vals = np.zeros(coords[0].shape[0])
    for r in range(R):
        term = np.full(coords[0].shape[0], lam[r])
        for m, a in enumerate(factors):
            term = term * a[coords[m], r]
        vals += term
    ind = [np.ascontiguousarray(c.astype(np.uint32)) for c in coords]
    return SparseTensor(dims, ind, vals, dict(kind="full_kruskal"))


def planted(dims, nnz, rank, seed) -> SparseTensor:
    """SPEC.md:475 ``cmd_gen --rank``: sampled distinct coordinates, model-valued entries."""
    rng = np.random.Generator(np.random.PCG64(seed))
    facs = [rng.random((d, rank)) for d in dims]
    cells = math.prod(dims)
    flat = rng.choice(cells, size=nnz, replace=False)
    coords = np.unravel_index(flat, dims)
    vals = np.zeros(nnz)
    for r in range(rank):
        term = np.ones(nnz)
        for m, f in enumerate(facs):
            term = term * f[coords[m], r]
        vals += term
    ind = [np.ascontiguousarray(c.astype(np.uint32)) for c in coords]
    return SparseTensor(tuple(dims), ind, vals, dict(seed=seed, planted_rank=rank, factors=facs))


def write_tns(t: SparseTensor, path: str) -> None:
    """FROSTT ``.tns`` writer: 1-based indices, one nonzero per line."""
    with open(path, "w") as f:
        for p in range(t.nnz):
            f.write(" ".join(str(int(t.ind[m][p]) + 1) for m in range(t.nmodes)))
            f.write(" %r\n" % float(t.vals[p]))


def read_tns(path: str) -> SparseTensor:
    """FROSTT ``.tns`` reader: '#' comments and blank lines skipped."""
    rows = []
    vals = []
    width = None
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            parts = s.split()
            if width is None:
                width = len(parts)
            if len(parts) != width or width < 2:
                raise ValueError(f"line {ln}: wrong field count")
            try:
                idx = [int(x) for x in parts[:-1]]
                v = float(parts[-1])
            except ValueError as e:
                raise ValueError(f"line {ln}: {e}") from None
            if min(idx) < 1:
                raise ValueError(f"line {ln}: index < 1")
            rows.append(idx)
            vals.append(v)
    if not rows:
        raise ValueError("no nonzeros")
    c = np.asarray(rows, dtype=np.int64) - 1
    dims = tuple(int(x) + 1 for x in c.max(axis=0))
    ind = [np.ascontiguousarray(c[:, m].astype(np.uint32)) for m in range(c.shape[1])]
    return SparseTensor(dims, ind, np.asarray(vals, dtype=np.float64), {})
