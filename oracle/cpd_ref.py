"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Symmetric CP-ALS written out in fp64 numpy on top of the expansion oracle
(SURVEY.md §8(f) NEXT-2).  The paper states only that symmetric CPD uses one
factor matrix for every mode so the update is identical in all modes
(PAPER.md:853-857); the update itself is the one-factor form of CP-ALS
(reading X22):

    M = MTTKRP(X, B)                  (oracle.mttkrp, fp64)
    B = M ((B^T B)^{.(n-1)})^{-1}
    lambda = column 2-norms of B;  B = B / lambda

and the fit of an iterate is 1 - ||X - Xhat|| / ||X|| with
||X||^2 = sum_e v_e^2 orbit_e, <X, Xhat> = sum_r lambda_r (M^T B)_rr,
||Xhat||^2 = lambda^T (B^T B)^{.n} lambda.
"""
from __future__ import annotations

import math

import numpy as np

from . import mttkrp as oracle_mttkrp
from .symmetric_ref import run_multiplicities


def tensor_norm2(order: int, idx, vals) -> float:
    c = np.sort(np.asarray(idx).reshape(-1, order), axis=1)
    first = np.ones(c.shape, bool)
    first[:, 1:] = c[:, 1:] != c[:, :-1]
    _, m = run_multiplicities(c)
    den = np.ones(c.shape[0])
    for t in range(order):
        den *= np.where(first[:, t], [math.factorial(k) for k in m[:, t]], 1)
    orbit = math.factorial(order) / den
    v = np.asarray(vals, np.float64)
    return float(np.sum(v * v * orbit))


def fit_of(order, x2, M, B, lam):
    inner = float(np.sum(lam * np.sum(M * B, axis=0)))
    G = B.T @ B
    xhat2 = float(lam @ (G ** order) @ lam)
    return 1.0 - math.sqrt(max(0.0, x2 - 2 * inner + xhat2)) / math.sqrt(x2)


def cp_als_sym(order: int, dim: int, idx, vals, B0, iters: int):
    """Runs `iters` updates from B0.  Returns (B, lam, fits) where fits[k] is the
    fit of the iterate after update k+1 evaluated with the next MTTKRP
    (len(fits) == iters, the last one needs one more MTTKRP — computed here)."""
    B = np.asarray(B0, np.float64).copy()
    lam = None
    x2 = tensor_norm2(order, idx, vals)
    fits = []
    for it in range(iters + 1):
        M, _ = oracle_mttkrp(order, dim, idx, vals, B_as_f32(B))
        if lam is not None:
            fits.append(fit_of(order, x2, M, B, lam))
        if it == iters:
            break
        H = (B.T @ B) ** (order - 1)
        Bn = np.linalg.solve(H.T, M.T).T          # M H^{-1}
        lam = np.linalg.norm(Bn, axis=0)
        B = Bn / np.where(lam > 0, lam, 1.0)
    return B, lam, np.array(fits)


def B_as_f32(B):
    """The expansion oracle takes B in fp32 (as the ABI does); the ALS state is
    kept in fp64 and rounded to fp32 at each MTTKRP input."""
    return np.asarray(B, np.float32)
