"""The seeded input generators (synth/): deterministic, canonical, distinct,
and with the structure BASELINE.json asks for.  CPU only."""
import hashlib

import numpy as np

from synth import CONFIGS, generate, scramble, small_random
from synth.workloads import make, run_lengths


def digest(w):
    h = hashlib.sha256()
    for a in (w.idx, w.vals, w.B):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def codes_of(idx):
    c = np.sort(idx, axis=1)
    code = np.zeros(c.shape[0], np.int64)
    for t in range(c.shape[1] - 1):
        code |= (c[:, t] == c[:, t + 1]).astype(np.int64) << t
    return code


def check_canonical_sorted_distinct(w):
    c = w.idx.astype(np.int64)
    assert np.all(c[:, 1:] >= c[:, :-1])
    assert c.min() >= 0 and c.max() < w.dim
    # lexicographic strict increase between consecutive rows => sorted and distinct
    diff = c[1:] - c[:-1]
    first_nz = np.argmax(diff != 0, axis=1)
    lead = diff[np.arange(len(diff)), first_nz]
    assert np.all(lead > 0)


def test_c1_structure_and_determinism():
    w1 = generate("c1", cache=False)
    w2 = generate("c1", cache=False)
    assert digest(w1) == digest(w2)
    assert (w1.order, w1.dim, w1.nnz, w1.R) == (3, 64, 2000, 8)
    check_canonical_sorted_distinct(w1)
    code = codes_of(w1.idx)
    assert np.sum(code != 0) == 200                 # 10% forced diagonal
    assert np.sum(code == 3) == 64                  # all-equal pool capped at dim
    assert np.sum(code == 1) == 68 and np.sum(code == 2) == 68
    assert w1.vals.dtype == np.float32 and np.all(np.abs(w1.vals) <= 1)
    assert w1.B.shape == (64, 8)


def test_small_random_covers_patterns_and_shapes():
    for n in (2, 3, 4, 5):
        w = small_random(n, {2: 40, 3: 20, 4: 14, 5: 12}[n], 600, 4, seed=n, diag_frac=0.3)
        check_canonical_sorted_distinct(w)
        assert set(codes_of(w.idx).tolist()) == set(range(1 << (n - 1)))


def test_uniform_and_zipf_modes_small():
    w = make("u", 3, 1000, 20000, 4, seed=2, mode="uniform")
    check_canonical_sorted_distinct(w)
    z = make("z", 3, 10000, 20000, 4, seed=3, mode="zipf", zipf_s=1.1)
    check_canonical_sorted_distinct(z)
    # hub row 0 leads a long run in the skewed mode
    assert np.mean(z.idx[:, 0] == 0) > 0.1
    assert np.mean(w.idx[:, 0] == 0) < 0.01


def test_scramble_is_same_multiset():
    w = small_random(4, 10, 300, 2, seed=1)
    si, sv = scramble(w.idx, w.vals, seed=3)
    a = sorted(zip(map(tuple, np.sort(si, axis=1).tolist()), sv.tolist()))
    b = sorted(zip(map(tuple, w.idx.tolist()), w.vals.tolist()))
    assert a == b
    assert not np.all(np.diff(si, axis=1) >= 0)     # really non-canonical


def test_config_table_matches_baseline():
    assert [CONFIGS[k].order for k in ("c1", "c2", "c3", "c4", "c5")] == [3, 3, 3, 4, 5]
    assert [CONFIGS[k].nnz for k in ("c1", "c2", "c3", "c4", "c5")] == [2000, 10**7, 5 * 10**7, 2 * 10**7, 10**7]
    assert [CONFIGS[k].R for k in ("c1", "c2", "c3", "c4", "c5")] == [8, 32, 32, 16, 16]
    assert run_lengths(5, 0b1010) == [1, 2, 2]


def test_banded_order2_generator():
    """mode "banded" (order-2 stand-in for the paper's FEM-like SSYMV matrices):
    canonical, sorted, distinct, within the band, deterministic."""
    import numpy as np

    from synth.workloads import make
    w = make("b", 2, 5000, 60000, 4, seed=3, mode="banded", band=40)
    w2 = make("b", 2, 5000, 60000, 4, seed=3, mode="banded", band=40)
    assert np.array_equal(w.idx, w2.idx) and np.array_equal(w.vals, w2.vals)
    d = w.idx[:, 1] - w.idx[:, 0]
    assert d.min() >= 0 and d.max() <= 40
    keys = w.idx[:, 0].astype(np.int64) * 5000 + w.idx[:, 1]
    assert np.all(np.diff(keys) > 0)          # sorted and distinct


def test_cache_manifest_detects_corruption(tmp_path, monkeypatch):
    """The on-disk workload cache carries a SHA-256 manifest: a corrupted
    cache file is detected and the workload regenerated."""
    import glob

    import numpy as np

    from synth import generate
    monkeypatch.setenv("SYSTEC_CACHE", str(tmp_path))
    w = generate("c1")
    assert generate("c1").meta.get("cached")
    f = glob.glob(str(tmp_path / "c1_*.npz"))[0]
    z = dict(np.load(f))
    z["vals"] = z["vals"] + 1
    np.savez(f, **z)
    w2 = generate("c1")
    assert not w2.meta.get("cached") and np.array_equal(w2.vals, w.vals)
    w3 = generate("c1", seed=9)
    assert w3.meta["seed"] == 9 and not np.array_equal(w3.idx, w.idx)
