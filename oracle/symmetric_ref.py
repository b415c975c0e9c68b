"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The symmetric method written out in fp64 numpy, independently of the CUDA
path: one read per stored canonical entry and one update per DISTINCT index
position, weighted by the number of distinct permutations that put that index
first.  This is pin P4 of SURVEY.md §8(c): it must equal the expansion oracle
(``oracle.mttkrp``) to rounding, on inputs that cover every equality pattern.

Derivation, in the paper's terms:
* the stored entry is a canonical coordinate read once
  ("reusing canonical reads");
* its equivalence group E is the partition of positions
  into runs of equal indices, with run sizes m_1..m_k;
* the unique symmetry group S_P|E has n!/prod m_w!
  members (read as a multinomial);
* the members that put the value of run u in the output position are the
  distinct permutations of the remaining multiset:
      coef_u = (n-1)! / ((m_u - 1)! prod_{w != u} m_w!) = (n-1)! m_u / prod_w m_w!
  and they all contribute the same product (the distributive grouping of
  PAPER.md:577-591, visible in Listing 6 PAPER.md:689-705 and the factors of
  Listing 7).
"""
from __future__ import annotations

import math

import numpy as np


def run_multiplicities(c_sorted: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """For sorted tuples [nnz][n]: (first, m) where first[e,t] says position t
    starts a run and m[e,t] is the size of the run containing t."""
    n = c_sorted.shape[1]
    first = np.ones(c_sorted.shape, dtype=bool)
    first[:, 1:] = c_sorted[:, 1:] != c_sorted[:, :-1]
    m = np.zeros(c_sorted.shape, dtype=np.int64)
    for t in range(n):
        m[:, t] = np.sum(c_sorted == c_sorted[:, t:t + 1], axis=1)
    return first, m


def position_coefficients(c_sorted: np.ndarray) -> np.ndarray:
    """coef[e,t] = (n-1)! m_t / prod_w m_w! at run-first t, else 0 (int64)."""
    n = c_sorted.shape[1]
    first, m = run_multiplicities(c_sorted)
    fact = np.array([math.factorial(k) for k in range(n + 1)], dtype=np.int64)
    denom = np.ones(c_sorted.shape[0], dtype=np.int64)
    for t in range(n):
        denom *= np.where(first[:, t], fact[m[:, t]], 1)
    num = math.factorial(n - 1) * m
    assert np.all((num % denom[:, None]) == 0)
    return np.where(first, num // denom[:, None], 0)


def mttkrp(order: int, dim: int, idx, vals, B, chunk: int = 1 << 18) -> np.ndarray:
    """Symmetric MTTKRP by per-position coefficients, fp64.  Returns C [dim][R]."""
    idx = np.asarray(idx).reshape(-1, order)
    B64 = np.asarray(B, dtype=np.float64)
    R = B64.shape[1]
    C = np.zeros((dim, R), np.float64)
    for lo in range(0, idx.shape[0], chunk):
        c = np.sort(idx[lo:lo + chunk].astype(np.int64), axis=1)
        v = np.asarray(vals[lo:lo + chunk], dtype=np.float64)
        coef = position_coefficients(c)
        rows = B64[c]                                   # [m][n][R]
        for t in range(order):
            w = coef[:, t] * v
            keep = w != 0
            if not np.any(keep):
                continue
            others = np.ones((int(keep.sum()), R))
            for s in range(order):
                if s != t:
                    others *= rows[keep, s, :]
            upd = w[keep, None] * others
            tgt = c[keep, t]
            for r in range(R):
                C[:, r] += np.bincount(tgt, weights=upd[:, r], minlength=dim)
    return C
