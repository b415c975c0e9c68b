"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and
compare it with the CPU oracle element by element."""
import math

import numpy as np

# BASELINE.json north_star: max |C_gpu - C_ref| / S <= 1e-4, S = oracle's sum of
# absolute terms (per element; reading X15)
TOL = 1e-4


def to_dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def parity(Cg, Cref, S, tol=TOL):
    """Returns the max normalised error; asserts the north_star bar and that
    elements with no terms are exactly zero."""
    Cg = np.asarray(Cg, dtype=np.float64)
    zero = S == 0
    assert np.all(Cg[zero] == 0.0), "element with no terms is not exactly zero"
    den = np.where(zero, 1.0, S)
    err = float(np.max(np.abs(Cg - Cref) / den)) if Cg.size else 0.0
    assert err <= tol, f"max normalised error {err:.3e} > {tol}"
    return err


def orbit_sizes(c_sorted):
    """n!/prod m! per sorted tuple (numpy, for the P7 invariant)."""
    n = c_sorted.shape[1]
    first = np.ones(c_sorted.shape, bool)
    first[:, 1:] = c_sorted[:, 1:] != c_sorted[:, :-1]
    den = np.ones(c_sorted.shape[0], np.int64)
    fact = np.array([math.factorial(k) for k in range(n + 1)])
    for t in range(n):
        m = np.sum(c_sorted == c_sorted[:, t:t + 1], axis=1)
        den *= np.where(first[:, t], fact[m], 1)
    return math.factorial(n) // den


def contraction_invariant(w, Cg, chunk=1 << 21):
    """P7 at any size: Σ_i C[i,r] B[i,r] = Σ_e v_e orbit_e prod_t B[c_t,r]; returns
    the error normalised by Σ_e |v_e| orbit_e prod_t |B[c_t,r]|."""
    B64 = w.B.astype(np.float64)
    lhs = np.sum(np.asarray(Cg, np.float64) * B64, axis=0)
    rhs = np.zeros(w.R)
    scale = np.zeros(w.R)
    for lo in range(0, w.nnz, chunk):
        c = w.idx[lo:lo + chunk].astype(np.int64)
        c.sort(axis=1)
        v = w.vals[lo:lo + chunk].astype(np.float64) * orbit_sizes(c)
        p = np.ones((c.shape[0], w.R))
        for t in range(w.order):
            p *= B64[c[:, t]]
        rhs += v @ p
        scale += np.abs(v) @ np.abs(p)
    return float(np.max(np.abs(lhs - rhs) / np.where(scale > 0, scale, 1.0)))


def sample_rows(w, k=48, seed=0):
    """Rows to check one by one at full size: the hub (most frequent leading
    index), both ends, and a random sample."""
    rng = np.random.default_rng(seed)
    lead = w.idx[:, 0]
    counts = np.bincount(lead, minlength=w.dim)
    hubs = np.argsort(counts)[-4:]
    rows = set(int(x) for x in hubs) | {0, w.dim - 1, int(w.idx[-1, -1]), int(w.idx[0, 0])}
    rows |= set(int(x) for x in rng.choice(w.dim, size=min(k, w.dim), replace=False))
    return np.array(sorted(rows), dtype=np.int64)
