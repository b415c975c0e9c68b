"""CPU pin of the one-pass CP-ALS scheme the GPU path runs (DESIGN.md reading
X25, csrc/cpd.cu cp_small_kernel): the stored factor F = B diag(t) carries a
column scale, one dense pass writes F_new = M W with
W = diag(t)^{-(n-1)} H^{-1} diag(1/lt), and lambda, t, the next B^T B and the
fit come from the R x R algebra (P = W^T M^T M W).  In exact (fp64)
arithmetic this must reproduce the plain symmetric ALS step
B_new = M(B) H^{-1}, lambda = column norms, B = B_new / lambda — iterates,
weights and fits — for any column scaling of the caller's factor.

The scheme is written here from its description (not from the CUDA code),
and the plain step is oracle/cpd_ref.py's, on a dense fp64 MTTKRP (tiny
sizes: the orbit expansion of every stored entry, then einsum)."""
import itertools
import math

import numpy as np
import pytest


def dense_sym(order, dim, idx, vals):
    X = np.zeros((dim,) * order)
    for c, v in zip(idx, vals):
        for p in set(itertools.permutations(c)):
            X[p] += float(v)
    return X


def mttkrp_dense(X, B):
    """M[i, r] = sum_{j..} X[i, j..] prod_t B[j_t, r]: contract the trailing
    modes one by one (the first contraction creates the rank axis)."""
    M = np.einsum("...j,jr->...r", X, B)
    for _ in range(X.ndim - 2):
        M = np.einsum("...jr,jr->...r", M, B)
    return M


def plain_als(X, B0, iters):
    """oracle/cpd_ref.py's step in fp64 (no fp32 rounding of B)."""
    n = X.ndim
    x2 = float(np.sum(X * X))
    B, lam, fits = np.array(B0, np.float64), None, []
    for it in range(iters + 1):
        M = mttkrp_dense(X, B)
        if lam is not None:
            inner = float(np.sum(lam * np.sum(M * B, axis=0)))
            xhat2 = float(lam @ ((B.T @ B) ** n) @ lam)
            fits.append(1 - math.sqrt(max(0.0, x2 - 2 * inner + xhat2)) / math.sqrt(x2))
        if it == iters:
            break
        Bn = M @ np.linalg.inv((B.T @ B) ** (n - 1))
        lam = np.linalg.norm(Bn, axis=0)
        B = Bn / lam
    return B, lam, np.array(fits)


def one_pass_scheme(X, B0, iters):
    """The GPU path's iteration, in fp64: F stored with scale t, one pass per
    iteration (iteration 0: Gram first, B_1 written normalised, the lambda
    prediction corrected by the caller's column norms c^{n-1})."""
    n = X.ndim
    x2 = float(np.sum(X * X))
    R = B0.shape[1]
    F = np.array(B0, np.float64)
    GB = F.T @ F                          # Gram of the current iterate (t = 1: F is the iterate)
    lam, t, lt, pf = np.ones(R), np.ones(R), np.ones(R), np.ones(R)

    def solve():                          # W = diag(t)^{-(n-1)} H^{-1} diag(1/lt), lt = pf lambda
        nonlocal lt, pf
        H = GB ** (n - 1)
        e = 1 / np.sqrt(np.diag(H))
        Hinv = e[:, None] * np.linalg.inv(e[:, None] * H * e[None, :]) * e[None, :]
        lt = lam * pf
        pf = np.ones(R)
        return (t ** -(n - 1))[:, None] * Hinv / lt[None, :]

    W = solve()
    fits = []
    for it in range(iters + 1):
        M = mttkrp_dense(X, F)
        if it > 0:                        # fit of the current iterate from the pass's dots
            dots = np.sum(M * F, axis=0)
            inner = float(np.sum(lam * dots / t ** n))
            xhat2 = float(lam @ (GB ** n) @ lam)
            fits.append(1 - math.sqrt(max(0.0, x2 - 2 * inner + xhat2)) / math.sqrt(x2))
        if it == iters:
            break
        GM = M.T @ M
        P = W.T @ GM @ W                  # = F_new^T F_new
        tn = np.sqrt(np.diag(P))
        lam = tn * lt
        if it == 0:                       # two passes: B_1 written normalised
            pf = np.diag(GB) ** ((n - 1) / 2)
            W = W / tn[None, :]
            GB = P / np.outer(tn, tn)
            t = np.ones(R)
        else:
            t = tn
            GB = P / np.outer(t, t)
        F = M @ W
        W = solve()
    return F / t[None, :], lam, np.array(fits)


@pytest.mark.parametrize("order,dim,R,span", [(3, 8, 3, 0), (3, 9, 4, 3), (4, 6, 2, 2), (5, 5, 2, 1)])
def test_one_pass_scheme_equals_plain_als(order, dim, R, span):
    rng = np.random.default_rng(order * 10 + R)
    canon = np.array(list(itertools.combinations_with_replacement(range(dim), order)), np.int32)
    keep = rng.random(len(canon)) < 0.6
    idx, vals = canon[keep], rng.standard_normal(int(keep.sum()))
    X = dense_sym(order, dim, idx, vals)
    B0 = rng.standard_normal((dim, R)) * np.logspace(-span, span, R)[None, :]   # arbitrary column scales
    iters = 6
    Bp, lp, fp = plain_als(X, B0, iters)
    Bs, ls, fs = one_pass_scheme(X, B0, iters)
    assert np.max(np.abs(Bs - Bp)) < 1e-9, np.max(np.abs(Bs - Bp))
    np.testing.assert_allclose(ls, lp, rtol=1e-9)
    np.testing.assert_allclose(fs, fp, rtol=0, atol=1e-9)


def test_plain_als_here_is_cpd_ref():
    """The fp64 plain step above is oracle/cpd_ref.py's (which rounds B to
    fp32 at each MTTKRP): they agree to fp32 rounding."""
    from oracle import cpd_ref
    rng = np.random.default_rng(4)
    order, dim, R = 3, 10, 3
    canon = np.array(list(itertools.combinations_with_replacement(range(dim), order)), np.int32)
    keep = rng.random(len(canon)) < 0.5
    idx, vals = canon[keep], rng.standard_normal(int(keep.sum())).astype(np.float32)
    B0 = rng.standard_normal((dim, R)).astype(np.float32)
    Bp, lp, fp = plain_als(dense_sym(order, dim, idx, vals), B0, 3)
    Br, lr, fr = cpd_ref.cp_als_sym(order, dim, idx, vals, B0, iters=3)
    assert np.max(np.abs(Bp - Br)) < 1e-4
    np.testing.assert_allclose(lp, lr, rtol=1e-4)
    np.testing.assert_allclose(fp, fr, atol=1e-5)
