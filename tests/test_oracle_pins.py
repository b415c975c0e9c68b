"""Pins of the CPU oracle against things other than itself (SURVEY.md §8(c)
P1-P10, P12).  No GPU is needed; nothing here touches the CUDA path."""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
from oracle import symmetric_ref
from synth import small_random, scramble
from synth.workloads import run_lengths

RNG = np.random.default_rng(1234)


def read_rows(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


def rel_err(C, ref, S):
    den = np.where(S > 0, S, 1.0)
    return float(np.max(np.abs(C - ref) / den)) if C.size else 0.0


# ---------------------------------------------------------------- P2/P3 helpers
def dense_from_entries(order, dim, idx, vals):
    """Abar[x] = sum of v_e with sort(idx_e) == sort(x), by scanning every
    coordinate of the cube (Def. Symmetry) — does not use
    any permutation enumeration."""
    table = {}
    for c, v in zip(np.sort(idx, axis=1), vals):
        k = tuple(int(x) for x in c)
        table[k] = table.get(k, 0.0) + float(v)
    A = np.zeros((dim,) * order)
    for x in itertools.product(range(dim), repeat=order):
        A[x] = table.get(tuple(sorted(x)), 0.0)
    return A


def dense_mttkrp(A, B):
    """C[i,r] = sum A[i,j1..] prod B[jt,r] by numpy.einsum."""
    n = A.ndim
    letters = "abcdefgh"[:n]
    spec = letters + "," + ",".join(f"{letters[t]}z" for t in range(1, n)) + "->az"
    return np.einsum(spec, A, *([B.astype(np.float64)] * (n - 1)))


# ---------------------------------------------------------------- P1
def brute_coef(c):
    """Count distinct permutations of c that start with each value (set of
    itertools.permutations — independent of the oracle's walk)."""
    perms = set(itertools.permutations(c))
    out = []
    for t in range(len(c)):
        first = t == 0 or c[t] != c[t - 1]
        out.append(sum(1 for p in perms if p[0] == c[t]) if first else 0)
    return out, len(perms)


def pattern_tuple(n, code):
    runs = run_lengths(n, code)
    vals = []
    for u, m in enumerate(runs):
        vals += [u] * m
    return vals


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_p1_coefficients_vs_bruteforce(n):
    for code in range(1 << (n - 1)):
        c = pattern_tuple(n, code)
        want, orbit = brute_coef(c)
        got = symmetric_ref.position_coefficients(np.array([c]))[0].tolist()
        assert got == want, (n, code)
        assert sum(got) == orbit
        ms = run_lengths(n, code)
        assert orbit == math.factorial(n) // math.prod(math.factorial(m) for m in ms)


def test_p1_n3_matches_listing6(golden_dir):
    rel = {"<<": 0, "=<": 1, "<=": 2, "==": 3}
    for row in read_rows(os.path.join(golden_dir, "listing6_mttkrp3_updates.txt")):
        code = rel[row[0]]
        want = [0 if x == "-" else int(x) for x in row[1:4]]
        c = pattern_tuple(3, code)
        assert symmetric_ref.position_coefficients(np.array([c]))[0].tolist() == want
        assert brute_coef(c)[1] == int(row[4])
        # the same counts through the expansion oracle: B = 1, v = 1 gives
        # C[x] = number of orbit members with leading index x
        C, _ = oracle.mttkrp(3, 3, np.array([c]), np.ones(1, np.float32),
                             np.ones((3, 1), np.float32), threads=1)
        for t in range(3):
            if want[t]:
                assert C[c[t], 0] == want[t]


def test_p1_lookup_factors(golden_dir):
    """PAPER.md:545 values: per-update factor f(E) = coef / m."""
    rel = {"<<": 0, "=<": 1, "<=": 2, "==": 3}
    for row in read_rows(os.path.join(golden_dir, "lookup_table_n3.txt")):
        c = pattern_tuple(3, rel[row[0]])
        coef = symmetric_ref.position_coefficients(np.array([c]))[0]
        _, m = symmetric_ref.run_multiplicities(np.array([c]))
        f = coef[0] / m[0, 0]
        assert abs(f - int(row[1]) / int(row[2])) < 1e-15


# ---------------------------------------------------------------- P2
@pytest.mark.parametrize("n,dim", [(2, 6), (3, 5), (4, 4), (5, 4), (3, 1), (5, 2)])
def test_p2_orbit_coverage(n, dim):
    canon = np.array(list(itertools.combinations_with_replacement(range(dim), n)), np.int32)
    assert canon.shape[0] == math.comb(dim + n - 1, n)
    # Σ orbit sizes = dim^n: every coordinate produced
    assert oracle.count_expanded(n, canon) == dim ** n
    # Abar == 1 everywhere  =>  C[i,r] = (Σ_j B[j,r])^(n-1): a duplicated or
    # missing permutation changes the left side
    B = RNG.uniform(-1, 1, (dim, 3)).astype(np.float32)
    C, _ = oracle.mttkrp(n, dim, canon, np.ones(canon.shape[0], np.float32), B, threads=2)
    want = np.tile(B.astype(np.float64).sum(0) ** (n - 1), (dim, 1))
    np.testing.assert_allclose(C, want, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- P3
@pytest.mark.parametrize("n,dim,nnz", [(3, 12, 150), (3, 7, 60), (4, 8, 200), (5, 6, 120), (2, 9, 30)])
def test_p3_dense_bruteforce(n, dim, nnz):
    w = small_random(n, dim, nnz, 5, seed=n * 100 + dim, diag_frac=0.3)
    idx, vals = scramble(w.idx, w.vals, seed=7)
    # add duplicates of some coordinates (additive, reading X11)
    idx = np.concatenate([idx, idx[:7]])
    vals = np.concatenate([vals, vals[:7] * 0.5])
    A = dense_from_entries(n, dim, idx, vals)
    want = dense_mttkrp(A, w.B)
    C, S = oracle.mttkrp(n, dim, idx, vals, w.B, threads=3)
    assert rel_err(C, want, S) < 1e-12
    # S is the sum of |terms| of the same einsum with |A| and |B|
    Sw = dense_mttkrp(np.abs(A), np.abs(w.B))
    # with duplicates |v1|+|v2| >= |v1+v2|, so S >= that bound
    assert np.all(S >= Sw * (1 - 1e-12))


# ---------------------------------------------------------------- P4
@pytest.mark.parametrize("n,dim,nnz", [(3, 40, 3000), (4, 20, 3000), (5, 12, 3000), (2, 50, 500)])
def test_p4_symmetric_formula_equals_expansion(n, dim, nnz):
    w = small_random(n, dim, nnz, 7, seed=11 * n, diag_frac=0.4)
    c = np.sort(w.idx, axis=1)
    codes = np.zeros(nnz, np.int64)
    for t in range(n - 1):
        codes |= (c[:, t] == c[:, t + 1]).astype(np.int64) << t
    assert set(codes.tolist()) == set(range(1 << (n - 1))), "every equality pattern covered"
    C, S = oracle.mttkrp(n, dim, w.idx, w.vals, w.B)
    Csym = symmetric_ref.mttkrp(n, dim, w.idx, w.vals, w.B)
    assert rel_err(Csym, C, S) < 1e-12
    # the same method in plain C (oracle_mttkrp_symmetric: the one-core CPU
    # analogue bench.py times), written separately from the numpy one
    Cc = oracle.mttkrp_symmetric(n, dim, w.idx, w.vals, w.B)
    assert rel_err(Cc, C, S) < 1e-12


# ---------------------------------------------------------------- P5
def load_worked(golden_dir):
    d = {"B": [], "entry": [], "C": [], "alt": []}
    for row in read_rows(os.path.join(golden_dir, "worked_example_n3.txt")):
        if row[0] in ("order", "dim", "R"):
            d[row[0]] = int(row[1])
        else:
            d[row[0]].append([float(x) for x in row[1:]])
    return d


def test_p5_hand_worked_example(golden_dir):
    d = load_worked(golden_dir)
    ent = np.array(d["entry"])
    idx, vals = ent[:, :3].astype(np.int32), ent[:, 3].astype(np.float32)
    B = np.array(d["B"], np.float32)
    C, S = oracle.mttkrp(3, d["dim"], idx, vals, B, threads=1)
    assert np.array_equal(C, np.array(d["C"]))
    alt = np.array(d["alt"])
    C2, _ = oracle.mttkrp(3, d["dim"], alt[:, :3].astype(np.int32), alt[:, 3].astype(np.float32), B)
    assert np.array_equal(C2, np.array(d["C"]))
    # and the dense einsum agrees
    A = dense_from_entries(3, 3, idx, vals)
    assert np.array_equal(dense_mttkrp(A, B), np.array(d["C"]))
    assert np.array_equal(symmetric_ref.mttkrp(3, 3, idx, vals, B), np.array(d["C"]))
    assert np.array_equal(oracle.mttkrp_symmetric(3, 3, idx, vals, B), np.array(d["C"]))


# ---------------------------------------------------------------- P6
@pytest.mark.parametrize("n,dim", [(3, 9), (4, 6), (5, 5)])
def test_p6_rank_one_closed_form(n, dim):
    lam = 0.7
    x = RNG.uniform(0.5, 1.5, dim)
    canon = np.array(list(itertools.combinations_with_replacement(range(dim), n)), np.int32)
    vals = (lam * np.prod(x[canon], axis=1)).astype(np.float32)
    B = RNG.uniform(-1, 1, (dim, 4)).astype(np.float32)
    C, S = oracle.mttkrp(n, dim, canon, vals, B)
    # value stored per canonical coordinate is fp32-rounded: compare with the
    # closed form on those rounded values through the dense tensor, and with
    # the exact closed form at fp32 rounding level
    want = lam * x[:, None] * (x @ B.astype(np.float64))[None, :] ** (n - 1)
    assert rel_err(C, want, S) < 1e-6


# ---------------------------------------------------------------- P7 / P8
def orbit_sizes(c):
    _, m = symmetric_ref.run_multiplicities(c)
    first = np.ones(c.shape, bool)
    first[:, 1:] = c[:, 1:] != c[:, :-1]
    n = c.shape[1]
    den = np.ones(c.shape[0], np.int64)
    for t in range(n):
        den *= np.where(first[:, t], [math.factorial(k) for k in m[:, t]], 1)
    return math.factorial(n) // den


@pytest.mark.parametrize("n,dim,nnz", [(3, 30, 2000), (4, 15, 2000), (5, 10, 1500)])
def test_p7_p8_invariants(n, dim, nnz):
    w = small_random(n, dim, nnz, 3, seed=5 + n, diag_frac=0.3)
    c = np.sort(w.idx, axis=1).astype(np.int64)
    orb = orbit_sizes(c)
    B64 = w.B.astype(np.float64)
    C, S = oracle.mttkrp(n, dim, w.idx, w.vals, w.B)
    # P7: Σ_i C[i,r] B[i,r] = Σ_e v_e orbit_e prod_t B[c_t,r]   (full contraction)
    lhs = np.sum(C * B64, axis=0)
    rhs = np.sum((w.vals.astype(np.float64) * orb)[:, None] * np.prod(B64[c], axis=1), axis=0)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-10, atol=1e-10)
    # P8: B = 1  =>  Σ_i C[i,r] = Σ_e v_e orbit_e
    C1, _ = oracle.mttkrp(n, dim, w.idx, w.vals, np.ones((dim, 2), np.float32))
    np.testing.assert_allclose(C1.sum(0), np.sum(w.vals.astype(np.float64) * orb), rtol=1e-10)


# ---------------------------------------------------------------- P9
def test_p9_order2_is_symmetric_spmm():
    dim, nnz = 40, 300
    w = small_random(2, dim, nnz, 6, seed=9, diag_frac=0.1)
    A = np.zeros((dim, dim))
    for (i, j), v in zip(w.idx, w.vals):
        A[i, j] += v
        if i != j:
            A[j, i] += v
    C, S = oracle.mttkrp(2, dim, w.idx, w.vals, w.B)
    assert rel_err(C, A @ w.B.astype(np.float64), S) < 1e-13


# ---------------------------------------------------------------- P10
def test_p10_homogeneity_linearity_shuffle():
    n, dim, nnz = 4, 14, 1200
    w = small_random(n, dim, nnz, 5, seed=3, diag_frac=0.25)
    C, S = oracle.mttkrp(n, dim, w.idx, w.vals, w.B)
    C2, _ = oracle.mttkrp(n, dim, w.idx, w.vals, (2.0 * w.B).astype(np.float32))
    np.testing.assert_allclose(C2, 8.0 * C, rtol=1e-12, atol=1e-12)
    si, sv = scramble(w.idx, w.vals, seed=4)
    C3, _ = oracle.mttkrp(n, dim, si, sv, w.B)
    assert rel_err(C3, C, S) < 1e-13
    # linearity: splitting every value into two stored duplicates
    half = (w.vals * 0.5).astype(np.float32)
    C4, _ = oracle.mttkrp(n, dim, np.concatenate([w.idx, w.idx]), np.concatenate([half, w.vals - half]), w.B)
    assert rel_err(C4, C, S) < 1e-12


# ---------------------------------------------------------------- P12
def test_p12_counters_match_paper_ratios(golden_dir):
    for row in read_rows(os.path.join(golden_dir, "reduction_ratios.txt")):
        n = int(row[0])
        w = small_random(n, 30, 500, 1, seed=n, diag_frac=0.0)
        expanded = oracle.count_expanded(n, w.idx)
        reads_ratio = w.nnz / expanded
        updates_ratio = (n * w.nnz) / expanded       # one update per distinct position
        assert reads_ratio == int(row[1]) / int(row[2])
        assert updates_ratio == int(row[3]) / int(row[4])


# ---------------------------------------------------------------- host logic
def test_oracle_threading_modes_agree():
    w = small_random(3, 50, 4000, 6, seed=21, diag_frac=0.2)
    C1, S1 = oracle.mttkrp(3, 50, w.idx, w.vals, w.B, threads=1)
    C4, S4 = oracle.mttkrp(3, 50, w.idx, w.vals, w.B, threads=4)
    Cr, Sr = oracle.mttkrp(3, 50, w.idx, w.vals, w.B, threads=4, mem_budget_bytes=1)
    assert rel_err(C4, C1, S1) < 1e-13 and rel_err(Cr, C1, S1) < 1e-13
    np.testing.assert_allclose(S4, S1, rtol=1e-13)
    rows = np.array([0, 7, 49, 3])
    Cq, Sq = oracle.mttkrp_rows(3, 50, w.idx, w.vals, w.B, rows, threads=3)
    assert rel_err(Cq, C1[rows], S1[rows]) < 1e-13


def test_oracle_errors():
    with pytest.raises(IndexError):
        oracle.mttkrp(3, 4, np.array([[0, 1, 4]], np.int32), np.ones(1, np.float32), np.ones((4, 2), np.float32))
    C, S = oracle.mttkrp(3, 4, np.zeros((0, 3), np.int32), np.zeros(0, np.float32), np.ones((4, 2), np.float32))
    assert not C.any() and not S.any()


# ---------------------------------------------------------------- general (non-symmetric) oracle
@pytest.mark.parametrize("n,dim,nnz", [(3, 9, 200), (4, 6, 300), (5, 5, 400), (2, 12, 50)])
def test_general_oracle_vs_dense_einsum(n, dim, nnz):
    rng = np.random.default_rng(n * 7 + dim)
    idx = rng.integers(0, dim, (nnz, n)).astype(np.int32)          # arbitrary tuples, repeats allowed
    vals = rng.uniform(-1, 1, nnz).astype(np.float32)
    B = rng.uniform(-1, 1, (dim, 3)).astype(np.float32)
    A = np.zeros((dim,) * n)
    np.add.at(A, tuple(idx.T), vals.astype(np.float64))
    C, S = oracle.mttkrp_general(n, dim, idx, vals, B)
    assert rel_err(C, dense_mttkrp(A, B), S) < 1e-12


@pytest.mark.parametrize("n,dim,nnz", [(3, 10, 150), (4, 7, 200), (5, 6, 150)])
def test_general_oracle_on_expanded_equals_symmetric(n, dim, nnz):
    """The naive kernel over the expanded tensor (every distinct permutation
    listed, via itertools) equals the symmetric oracle: the paper's premise."""
    w = small_random(n, dim, nnz, 4, seed=n, diag_frac=0.3)
    ex_i, ex_v = [], []
    for c, v in zip(w.idx, w.vals):
        for p in sorted(set(itertools.permutations(c.tolist()))):
            ex_i.append(p)
            ex_v.append(v)
    C1, S1 = oracle.mttkrp(n, dim, w.idx, w.vals, w.B)
    C2, _ = oracle.mttkrp_general(n, dim, np.array(ex_i, np.int32), np.array(ex_v, np.float32), w.B)
    assert rel_err(C2, C1, S1) < 1e-13


# ---------------------------------------------------------------- (min,+) relaxation oracle (NEXT-3)
def test_minplus_oracle_vs_dense():
    rng = np.random.default_rng(3)
    dim, nnz = 40, 300
    w = small_random(2, dim, nnz, 1, seed=3, diag_frac=0.1)
    vals = rng.uniform(-1, 3, nnz).astype(np.float32)
    d = rng.uniform(0, 10, dim).astype(np.float32)
    A = np.full((dim, dim), np.inf, np.float32)
    for (a, b), v in zip(w.idx, vals):
        A[a, b] = min(A[a, b], v)
        A[b, a] = min(A[b, a], v)
    want = np.minimum(d, np.min(A + d[None, :], axis=1))        # fp32 adds, exact min
    si, sv = scramble(w.idx, vals, seed=1)                       # either orientation
    assert np.array_equal(oracle.minplus_sym2(dim, si, sv, d), want)


# ---------------------------------------------------------------- symmetric CP-ALS oracle (NEXT-2)
def planted(order, dim, R, seed, noise=0.0):
    """All canonical coordinates of X = sum_r lam_r b_r^{(x)n} (+ noise)."""
    rng = np.random.default_rng(seed)
    Bt = rng.standard_normal((dim, R))
    Bt /= np.linalg.norm(Bt, axis=0)
    lam = np.linspace(2.0, 1.0, R)
    canon = np.array(list(itertools.combinations_with_replacement(range(dim), order)), np.int32)
    vals = np.zeros(len(canon))
    for r in range(R):
        vals += lam[r] * np.prod(Bt[canon, r], axis=1)
    vals += noise * rng.standard_normal(len(canon))
    return canon, vals.astype(np.float32), Bt, lam


def test_cpd_oracle_fit_formula_vs_dense():
    from oracle import cpd_ref
    order, dim, R = 3, 7, 2
    idx, vals, Bt, lam = planted(order, dim, R, seed=1, noise=0.05)
    rng = np.random.default_rng(2)
    B = rng.standard_normal((dim, R))
    B /= np.linalg.norm(B, axis=0)
    lam_e = np.array([1.3, 0.7])
    M, _ = oracle.mttkrp(order, dim, idx, vals, B.astype(np.float32))
    A = dense_from_entries(order, dim, idx, vals)
    Xhat = sum(lam_e[r] * np.einsum("i,j,k->ijk", B[:, r], B[:, r], B[:, r]) for r in range(R))
    want = 1 - np.linalg.norm(A - Xhat) / np.linalg.norm(A)
    x2 = cpd_ref.tensor_norm2(order, idx, vals)
    assert abs(x2 - np.sum(A * A)) < 1e-9 * x2
    # M was computed from fp32-rounded B: compare at that precision
    assert abs(cpd_ref.fit_of(order, x2, M, B, lam_e) - want) < 1e-6


@pytest.mark.parametrize("order,dim,R", [(3, 12, 3), (4, 8, 2), (3, 10, 1)])
def test_cpd_oracle_recovers_planted(order, dim, R):
    from oracle import cpd_ref
    idx, vals, Bt, lam = planted(order, dim, R, seed=order + R)
    rng = np.random.default_rng(5)
    B0 = Bt + 0.1 * rng.standard_normal(Bt.shape)
    B, lam_got, fits = cpd_ref.cp_als_sym(order, dim, idx, vals, B0, iters=40)
    assert fits[-1] > 0.999          # the fit formula cancels: ~1e-4 floor from fp32 MTTKRP input
    # columns match the planted factors up to order and sign
    match = np.abs(B.T @ Bt)
    assert np.all(match.max(axis=1) > 0.999)
    assert np.allclose(np.sort(lam_got), np.sort(lam), rtol=1e-3)


# ---------------------------------------------------------------- TTM oracle (NEXT-4)
def test_ttm_oracle_vs_einsum():
    w = small_random(3, 9, 120, 4, seed=31, diag_frac=0.3)
    si, sv = scramble(w.idx, w.vals, seed=3)
    A = dense_from_entries(3, 9, si, sv)
    want = np.einsum("kjl,ki->jli", A, w.B.astype(np.float64))     # C[j][l][i]
    got = oracle.ttm_sym3(9, si, sv, w.B)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    assert np.allclose(got, got.transpose(1, 0, 2))                   # visible output symmetry


def oracle_sssp(dim, idx, vals, source, max_iters=None):
    """Bellman-Ford by iterating the (min,+) relaxation oracle until no change."""
    d = np.full(dim, np.inf, np.float32)
    d[source] = 0
    it = 0
    for it in range(1, (max_iters or dim) + 1):
        y = oracle.minplus_sym2(dim, idx, vals, d)
        if np.array_equal(y, d):
            return y, it
        d = y
    return d, it


def test_sssp_oracle_vs_scipy_shortest_path():
    """Pin of the iterated relaxation against scipy's Dijkstra on the same
    undirected graph (fp32 sums vs fp64: 1e-5 relative)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import shortest_path
    w = small_random(2, 300, 2000, 1, seed=4, diag_frac=0.0)
    vals = np.random.default_rng(2).uniform(0.1, 5.0, w.nnz).astype(np.float32)
    A = coo_matrix((vals.astype(np.float64), (w.idx[:, 0], w.idx[:, 1])), shape=(300, 300)).tocsr()
    want = shortest_path(A, method="D", directed=False, indices=7)
    got, iters = oracle_sssp(300, w.idx, vals, 7)
    finite = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), finite)
    np.testing.assert_allclose(got[finite], want[finite], rtol=1e-5)
    assert iters > 1
