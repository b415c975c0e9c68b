"""The pins catch plausible oracle mistakes: each deliberately broken variant
of mttkrp_oracle.c must fail at least one pin that the real oracle passes.
The variants are made here, by a textual patch of a temporary copy of the
oracle source (the oracle itself carries no mutation hooks).  CPU only."""
import itertools
import os
import subprocess

import numpy as np
import pytest

import oracle
from synth import scramble, small_random
from test_oracle_pins import dense_from_entries, dense_mttkrp, load_worked, rel_err

# k: (what the bug is, the exact source text it replaces, its replacement)
MUTATIONS = {
    1: ("tuple not sorted before the permutation walk",
        "sort_small(p, n);                                   /* step 2 */", ""),
    2: ("last factor of the product dropped",
        "for (int t = 1; t < n; t++) {", "for (int t = 1; t < n - 1; t++) {"),
    3: ("product indexes p[t-1] instead of p[t]",
        "J->B + (int64_t)p[t] * R;", "J->B + (int64_t)p[t - 1] * R;"),
    4: ("update lands on the last index instead of the first",
        "double *c = J->C + out * R, *s = J->S + out * R;",
        "out = J->rowslot ? out : p[n - 1] - J->row_lo;\n            double *c = J->C + out * R, *s = J->S + out * R;"),
    5: ("sign flipped on the update",
        "c[r] += J->term[r]; s[r] += fabs(J->term[r]);", "c[r] -= J->term[r]; s[r] += fabs(J->term[r]);"),
    6: ("only the first permutation of each entry",
        "} while (next_perm(p, n));\n    }\n    return NULL;", "} while (0);\n    }\n    return NULL;"),
    7: ("off-diagonal permutations counted twice (a wrong multiplicity)",
        "c[r] += J->term[r]; s[r] += fabs(J->term[r]);",
        "c[r] += (p[0] == p[n - 1] ? 1.0 : 2.0) * J->term[r]; s[r] += fabs(J->term[r]);"),
}


def pins_fail(lib, golden_dir):
    """Runs P2 (orbit coverage), P3 (dense brute force) and P5 (hand example)
    with the given oracle library; returns the names of the pins that fail."""
    failed = []
    n, dim = 3, 5
    canon = np.array(list(itertools.combinations_with_replacement(range(dim), n)), np.int32)
    if oracle.count_expanded(n, canon, lib=lib) != dim ** n:
        failed.append("P2-count")
    B = np.random.default_rng(0).uniform(-1, 1, (dim, 3)).astype(np.float32)
    C, _ = oracle.mttkrp(n, dim, canon, np.ones(len(canon), np.float32), B, threads=1, lib=lib)
    if not np.allclose(C, np.tile(B.astype(np.float64).sum(0) ** (n - 1), (dim, 1)), rtol=1e-12, atol=1e-12):
        failed.append("P2-ones")
    for n, dim, nnz in ((3, 8, 80), (4, 6, 100)):
        w = small_random(n, dim, nnz, 4, seed=n, diag_frac=0.3)
        si, sv = scramble(w.idx, w.vals, seed=2)
        want = dense_mttkrp(dense_from_entries(n, dim, si, sv), w.B)
        C, S = oracle.mttkrp(n, dim, si, sv, w.B, threads=1, lib=lib)
        if not rel_err(C, want, S) < 1e-12:
            failed.append(f"P3-n{n}")
    d = load_worked(golden_dir)
    ent = np.array(d["entry"])
    C, _ = oracle.mttkrp(3, 3, ent[:, :3].astype(np.int32), ent[:, 3].astype(np.float32),
                         np.array(d["B"], np.float32), threads=1, lib=lib)
    if not np.array_equal(C, np.array(d["C"])):
        failed.append("P5")
    return failed


def build_variant(k, tmp):
    """k = 0: the oracle source as committed; k >= 1: a patched copy."""
    with open(os.path.join(os.path.dirname(oracle.__file__), "mttkrp_oracle.c")) as f:
        text = f.read()
    if k:
        _, old, new = MUTATIONS[k]
        assert text.count(old) == 1, f"mutation {k}: the patched text must occur exactly once"
        text = text.replace(old, new)
    src = os.path.join(tmp, f"oracle_m{k}.c")
    with open(src, "w") as f:
        f.write(text)
    out = os.path.join(tmp, f"liboracle_m{k}.so")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", out, src, "-lm"])
    return oracle.load_variant(out)


def test_real_oracle_passes_the_pin_subset(golden_dir, tmp_path):
    assert pins_fail(build_variant(0, str(tmp_path)), golden_dir) == []


@pytest.mark.timeout(120)
@pytest.mark.parametrize("k", sorted(MUTATIONS))
def test_each_mutation_is_caught(k, golden_dir, tmp_path):
    failed = pins_fail(build_variant(k, str(tmp_path)), golden_dir)
    assert failed, f"mutation {k} ({MUTATIONS[k][0]}) passed every pin"
