"""Seeded generators for fully symmetric sparse tensors in canonical-triangle COO.

What is drawn follows BASELINE.json ``configs`` and SURVEY.md §8(d) (the
survey's reading X18 of the generator details):

* numpy ``default_rng(seed)`` (PCG64); the seed of config ``cK`` is K.
* raw tuples are sorted within the tuple (canonical coordinates,
  PAPER.md:162-167 Def. Canonical) and de-duplicated keeping the first
  occurrence in draw order until ``nnz`` distinct tuples exist;
* "strict" entries: iid uniform tuples with any repeated index rejected
  (uniform over c_0 < ... < c_{n-1});
* "forced-diagonal" entries: pattern quotas split equally over the
  2^(n-1)-1 non-trivial equality patterns (remainder to the lowest codes),
  each pattern capped at its pool size, the shortfall handed round-robin to
  the uncapped patterns; a pattern draws k = #runs distinct sorted values and
  expands them by run length;
* the stored tensor is lexicographically sorted; then
  ``vals = uniform(-1,1,nnz)`` and ``B = uniform(-1,1,(dim,R))``, both fp32.

Nothing here computes any part of the MTTKRP: the equality-pattern "code"
below only describes which diagonal a forced entry is drawn on.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

GEN_VERSION = "v1"


@dataclass
class Workload:
    name: str
    order: int
    dim: int
    R: int
    idx: np.ndarray    # int32 [nnz][order], canonical (ascending in row), lexicographically sorted
    vals: np.ndarray   # float32 [nnz]
    B: np.ndarray      # float32 [dim][R]
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.idx.shape[0])


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    order: int
    dim: int
    nnz: int
    R: int
    mode: str          # "strict" (strict + forced diagonals), "uniform", "zipf"
    n_forced: int
    seed: int
    zipf_s: float = 0.0
    describe: str = ""


# BASELINE.json "configs", in order.
CONFIGS = {
    "c1": ConfigSpec("c1", 3, 64, 2_000, 8, "strict", 200, 1,
                     describe="order-3, dim 64, 2k nnz (10% forced diagonal), R 8"),
    "c2": ConfigSpec("c2", 3, 100_000, 10_000_000, 32, "uniform", 0, 2,
                     describe="order-3, dim 1e5, 10M nnz uniform, R 32"),
    "c3": ConfigSpec("c3", 3, 1_000_000, 50_000_000, 32, "zipf", 0, 3, zipf_s=1.1,
                     describe="order-3, dim 1e6, 50M nnz Zipf(1.1), R 32"),
    "c4": ConfigSpec("c4", 4, 10_000, 20_000_000, 16, "strict", 1_000_000, 4,
                     describe="order-4, dim 1e4, 20M nnz (5% forced diagonal), R 16"),
    "c5": ConfigSpec("c5", 5, 1_000, 10_000_000, 16, "strict", 500_000, 5,
                     describe="order-5, dim 1e3, 10M nnz (5% forced diagonal, all patterns), R 16"),
}


def key_bits(dim: int) -> int:
    """Bits per index in a packed lexicographic key: ceil(log2 dim), at least 1."""
    return max(1, int(math.ceil(math.log2(dim)))) if dim > 1 else 1


def _pack(c: np.ndarray, bits: int) -> np.ndarray:
    n = c.shape[1]
    k = np.zeros(c.shape[0], dtype=np.uint64)
    for t in range(n):
        k = (k << np.uint64(bits)) | c[:, t].astype(np.uint64)
    return k


def _distinct_first(draw, target: int, bits: int, batch: int) -> np.ndarray:
    """Draw sorted tuples with ``draw(m)`` until ``target`` distinct ones exist;
    keep first occurrences in draw order."""
    parts = []
    rounds = 0
    while True:
        rounds += 1
        if rounds > 1000:
            raise RuntimeError("generator could not reach the requested distinct count")
        parts.append(draw(batch))
        allc = np.concatenate(parts, axis=0) if len(parts) > 1 else parts[0]
        keys = _pack(allc, bits)
        _, first = np.unique(keys, return_index=True)
        if first.size >= target:
            first.sort()
            return allc[first[:target]]
        have = first.size
        # next batch: enough to cover the shortfall at the observed yield
        yield_ = max(have / max(allc.shape[0], 1), 1e-3)
        batch = int((target - have) / yield_ * 1.2) + 64


def _strict_draw(rng, n, dim):
    def draw(m):
        c = np.sort(rng.integers(0, dim, size=(m, n), dtype=np.int64), axis=1)
        ok = np.all(c[:, 1:] != c[:, :-1], axis=1)
        return c[ok]
    return draw


def _uniform_draw(rng, n, dim):
    def draw(m):
        return np.sort(rng.integers(0, dim, size=(m, n), dtype=np.int64), axis=1)
    return draw


def _zipf_draw(rng, n, dim, s):
    w = np.arange(1, dim + 1, dtype=np.float64) ** (-s)   # P(k) ∝ (k+1)^-s, hub = index 0
    cdf = np.cumsum(w)
    cdf /= cdf[-1]

    def draw(m):
        u = rng.random((m, n))
        c = np.searchsorted(cdf, u, side="right").astype(np.int64)
        np.minimum(c, dim - 1, out=c)
        return np.sort(c, axis=1)
    return draw


def run_lengths(order: int, code: int) -> list[int]:
    """Run lengths of an equality pattern: bit t of ``code`` says c_t == c_{t+1}."""
    runs = [1]
    for t in range(order - 1):
        if (code >> t) & 1:
            runs[-1] += 1
        else:
            runs.append(1)
    return runs


def _pattern_quotas(order: int, dim: int, total: int) -> dict[int, int]:
    codes = list(range(1, 1 << (order - 1)))
    P = len(codes)
    quota = {c: total // P + (1 if i < total % P else 0) for i, c in enumerate(codes)}
    pool = {c: math.comb(dim, len(run_lengths(order, c))) for c in codes}
    capped = set()
    while True:
        short = 0
        for c in codes:
            if c not in capped and quota[c] >= pool[c]:
                short += quota[c] - pool[c]
                quota[c] = pool[c]
                capped.add(c)
        if short == 0:
            return quota
        open_ = [c for c in codes if c not in capped]
        if not open_:
            raise ValueError("not enough diagonal coordinates for the forced quota")
        for i, c in enumerate(open_):
            quota[c] += short // len(open_) + (1 if i < short % len(open_) else 0)


def _forced_draw(rng, order, dim, code):
    runs = run_lengths(order, code)
    k = len(runs)
    rep = np.array(runs)

    def draw(m):
        v = np.sort(rng.integers(0, dim, size=(m, k), dtype=np.int64), axis=1)
        if k > 1:
            v = v[np.all(v[:, 1:] != v[:, :-1], axis=1)]
        return np.repeat(v, rep, axis=1)
    return draw


def _forced(rng, order, dim, total, bits):
    out = []
    for code, q in _pattern_quotas(order, dim, total).items():
        if q == 0:
            continue
        runs = run_lengths(order, code)
        if len(runs) == 1:
            v = rng.permutation(dim)[:q].astype(np.int64)
            out.append(np.repeat(v[:, None], order, axis=1))
        else:
            out.append(_distinct_first(_forced_draw(rng, order, dim, code), q, bits,
                                       batch=int(q * 1.3) + 16))
    return np.concatenate(out, axis=0) if out else np.zeros((0, order), np.int64)


def _banded_draw(rng, dim, band):
    """Order 2: pairs (i, i + d), i uniform, d uniform in [0, band] (rows near
    the diagonal only, the profile of FEM / structural matrices)."""
    def draw(m):
        i = rng.integers(0, dim, size=m, dtype=np.int64)
        j = i + rng.integers(0, band + 1, size=m, dtype=np.int64)
        ok = j < dim
        return np.stack([i[ok], j[ok]], axis=1)
    return draw


def make(name: str, order: int, dim: int, nnz: int, R: int, seed: int,
         mode: str = "strict", n_forced: int = 0, zipf_s: float = 1.1, band: int = 0) -> Workload:
    """Draw one workload (see module docstring).  mode "banded" (order 2 only):
    entries (i, j) with 0 <= j - i <= band."""
    if order < 1 or dim < 1 or nnz < 0 or R < 1:
        raise ValueError("bad workload shape")
    if nnz > math.comb(dim + order - 1, order):
        raise ValueError("nnz exceeds the number of canonical coordinates")
    rng = np.random.default_rng(seed)
    bits = key_bits(dim)
    if nnz == 0:
        c = np.zeros((0, order), np.int64)
    elif mode == "uniform":
        c = _distinct_first(_uniform_draw(rng, order, dim), nnz, bits, batch=int(nnz * 1.05) + 64)
    elif mode == "zipf":
        c = _distinct_first(_zipf_draw(rng, order, dim, zipf_s), nnz, bits, batch=int(nnz * 1.6) + 64)
    elif mode == "banded":
        if order != 2 or band < 0 or nnz > dim * (band + 1):
            raise ValueError("banded: order 2 and nnz <= dim * (band + 1)")
        c = _distinct_first(_banded_draw(rng, dim, band), nnz, bits, batch=int(nnz * 1.3) + 64)
    elif mode == "strict":
        n_strict = nnz - n_forced
        parts = []
        if n_strict > 0:
            if n_strict > math.comb(dim, order):
                raise ValueError("not enough strict coordinates")
            parts.append(_distinct_first(_strict_draw(rng, order, dim), n_strict, bits,
                                         batch=int(n_strict * 1.1) + 64))
        if n_forced > 0:
            parts.append(_forced(rng, order, dim, n_forced, bits))
        c = np.concatenate(parts, axis=0)
    else:
        raise ValueError(mode)
    order_ix = np.argsort(_pack(c, bits), kind="stable")
    c = np.ascontiguousarray(c[order_ix]).astype(np.int32)
    vals = rng.uniform(-1.0, 1.0, nnz).astype(np.float32)
    B = rng.uniform(-1.0, 1.0, (dim, R)).astype(np.float32)
    return Workload(name, order, dim, R, c, vals, B,
                    meta={"seed": seed, "mode": mode, "n_forced": n_forced, "band": band, "gen": GEN_VERSION})


def _cache_dir() -> str:
    return os.environ.get("SYSTEC_CACHE", "/tmp/systec_workloads")


def _digest(w_idx, w_vals, w_B) -> dict:
    import hashlib
    return {k: hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()
            for k, a in (("idx", w_idx), ("vals", w_vals), ("B", w_B))}


def generate(name: str, cache: bool = True, seed: int | None = None) -> Workload:
    """The BASELINE.json config ``name`` (c1..c5), optionally cached on disk
    (the cache only saves time; it is regenerated when absent or when its
    SHA-256 manifest does not match the arrays).  ``seed`` overrides the
    config's seed (a different draw of the same shape)."""
    s = CONFIGS[name]
    sd = s.seed if seed is None else int(seed)
    tag = f"{name}_{GEN_VERSION}" + ("" if seed is None else f"_s{sd}")
    path = os.path.join(_cache_dir(), f"{tag}.npz")
    manifest = path[:-4] + ".sha256.json"
    if cache and os.path.exists(path) and os.path.exists(manifest):
        try:
            import json
            z = np.load(path)
            idx, vals, B = z["idx"], z["vals"], z["B"]
            with open(manifest) as f:
                want = json.load(f)
            if _digest(idx, vals, B) == want:
                return Workload(name, s.order, s.dim, s.R, idx, vals, B,
                                meta={"seed": sd, "mode": s.mode, "gen": GEN_VERSION, "cached": True})
        except Exception:
            pass
    w = make(name, s.order, s.dim, s.nnz, s.R, sd, s.mode, s.n_forced, s.zipf_s)
    if cache:
        try:
            import json
            os.makedirs(_cache_dir(), exist_ok=True)
            tmp = path + f".{os.getpid()}.tmp.npz"
            np.savez(tmp, idx=w.idx, vals=w.vals, B=w.B)
            with open(manifest + f".{os.getpid()}.tmp", "w") as f:
                json.dump(_digest(w.idx, w.vals, w.B), f)
            os.replace(tmp, path)
            os.replace(manifest + f".{os.getpid()}.tmp", manifest)
        except OSError:
            pass
    return w

def small_random(order: int, dim: int, nnz: int, R: int, seed: int,
                 diag_frac: float = 0.2, mode: str = "strict") -> Workload:
    """A small workload with the same recipe, for parity tests."""
    if mode != "strict":
        return make(f"rand{order}_{dim}_{nnz}", order, dim, nnz, R, seed, mode)
    n_forced = int(round(nnz * diag_frac))
    diag_pool = sum(math.comb(dim, len(run_lengths(order, c))) for c in range(1, 1 << (order - 1)))
    n_forced = min(n_forced, nnz, diag_pool)
    # not enough strict coordinates on tiny cubes: move the rest to the diagonals
    n_forced = max(n_forced, nnz - math.comb(dim, order))
    return make(f"rand{order}_{dim}_{nnz}", order, dim, nnz, R, seed, "strict", n_forced)


def integer_workload(w: Workload, seed: int, lo: int = -2, hi: int = 2) -> Workload:
    """Same coordinates, integer values and factor entries in [lo, hi] (as fp32)."""
    rng = np.random.default_rng(seed)
    vals = rng.integers(lo, hi + 1, w.nnz).astype(np.float32)
    B = rng.integers(lo, hi + 1, w.B.shape).astype(np.float32)
    return Workload(w.name + "_int", w.order, w.dim, w.R, w.idx, vals, B, dict(w.meta, integer=True))


def scramble(idx: np.ndarray, vals: np.ndarray, seed: int):
    """Shuffle the entry order and permute the indices inside every tuple
    (a non-canonical spelling of the same symmetric tensor)."""
    rng = np.random.default_rng(seed)
    p = rng.permutation(idx.shape[0])
    idx2 = idx[p]
    perm = np.argsort(rng.random(idx2.shape), axis=1)
    idx2 = np.take_along_axis(idx2, perm, axis=1)
    return np.ascontiguousarray(idx2.astype(np.int32)), np.ascontiguousarray(vals[p])
