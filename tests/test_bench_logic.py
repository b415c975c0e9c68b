"""bench.py's host logic on CPU: the roofline arithmetic (the bound of the
binding memory class, achieved / peak), the gather:reduction mix ratio, the
reduced-row count from plan statistics, and the clock sampler's report
without NVML samples."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class W:
    order, dim, R = 3, 100, 32


def test_mix_shapes():
    assert bench.mix_shapes(30, 20) == [(3, 2)]
    assert bench.mix_shapes(20.08, 20.09) == [(1, 1), (2, 2), (3, 3), (4, 4)]
    assert bench.mix_shapes(10, 0) == [(3, 0)] and bench.mix_shapes(0, 5) == [(0, 2)]
    g, r = bench.mix_shapes(78.5, 52.0)[0]
    assert abs(g / r - 78.5 / 52.0) < 0.05


def test_memory_terms_counts_reduced_rows():
    # 10 entries, all strict (code 0: c1 != c0), G = 30; 4 leading runs; 6 position-1 runs
    st = {"G": 30, "lead_runs": 4, "pos1_runs": 6, "pattern_hist": [10, 0, 0, 0] + [0] * 12}
    t = bench.memory_terms(W, st, 10, {"pos1": 0})
    assert t["red_rows"] == 4 + 20 and t["stream"] == 10 * 16 and t["gather_alg"] == 30 * 128
    # L2 gathers: G less the 6 repeated leading rows and the 4 repeated position-1 rows
    assert t["gather_rows"] == 30 - (10 - 4) - (10 - 6) and t["gather"] == t["gather_rows"] * 128
    t1 = bench.memory_terms(W, st, 10, {"pos1": 1})
    assert t1["red_rows"] == 4 + 20 - (10 - 6)


def test_roofline_picks_the_binding_class():
    terms = {"stream": 160e6, "gather": 3.84e9, "red": 2.56e9}
    bounds = {"hbm_read_gbs": 6700.0, "l2_gather_gbs": 15000.0, "l2_red_gbs": 6000.0, "l2_mix_gbs": 13000.0,
              "clocks": {}}
    r = bench.roofline(dict(terms), bounds, 0.48, 4.0e9, 6553.0, {"dram_bytes_per_launch": 192e6})
    times = {"stream": 160e6 / 6700e9, "gather": 3.84e9 / 15000e9, "red": 2.56e9 / 6000e9,
             "mix": 6.4e9 / 13000e9}
    bind = max(times, key=times.get)
    assert r["bound"] == "l2" and r["terms_ms"].keys() == times.keys()
    assert math.isclose(r["frac"], r["achieved"] / r["peak"]) and math.isclose(r["frac"], times[bind] / 0.48e-3)
    assert math.isclose(r["hbm"]["physical_gbs"], 192e6 / 0.48e-3 / 1e9)
    r2 = bench.roofline(dict(terms), {"unavailable": "x"}, 0.48, 4.0e9, 6553.0, None)
    assert r2["bound"] == "hbm" and math.isclose(r2["frac"], 4.0e9 / 0.48e-3 / 1e9 / 6553.0)


def test_clock_sampler_reports_without_samples():
    rep = bench.ClockSampler.__new__(bench.ClockSampler)
    rep.ok, rep.samples, rep.max_mhz, rep.reasons = False, [], None, 0
    assert rep.report()["samples"] == 0


def test_mix_pairs_match_the_bounds_library():
    """bench.MIX_PAIRS are exactly the instantiated pairs of tools/bounds.cu."""
    import ctypes

    import __graft_entry__
    lib = ctypes.CDLL(__graft_entry__.build_bounds())
    buf = (ctypes.c_int * 64)()
    n = lib.bounds_mix_pairs(buf, 32)
    pairs = [(buf[2 * k], buf[2 * k + 1]) for k in range(n)]
    assert set(bench.MIX_PAIRS) <= set(pairs)


def test_bench_functions_reference_defined_globals():
    """Every global name a bench.py function loads (LOAD_GLOBAL, nested code
    included) is defined in the module or a builtin — a NameError there would
    only show on the GPU box."""
    import builtins
    import dis
    import types

    def globals_of(code):
        for ins in dis.get_instructions(code):
            if ins.opname == "LOAD_GLOBAL":
                yield ins.argval
        for c in code.co_consts:
            if isinstance(c, types.CodeType):
                yield from globals_of(c)

    checked = 0
    for name, obj in list(vars(bench).items()):
        fns = [obj] if isinstance(obj, types.FunctionType) else \
            [f for f in vars(obj).values() if isinstance(f, types.FunctionType)] if isinstance(obj, type) else []
        for fn in fns:
            if fn.__module__ != "bench":
                continue
            for ref in globals_of(fn.__code__):
                assert ref in vars(bench) or hasattr(builtins, ref), f"{name} loads undefined global {ref}"
                checked += 1
    assert checked > 50
