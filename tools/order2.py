"""NEXT-3 measurements: order-2 symmetric kernels (SSYMV R=1, SSYMM R=32, and
one Bellman-Ford (min,+) relaxation) on a synthetic symmetric sparse matrix,
vs the naive kernel over both triangles (the paper's SSYMV comparison,
PAPER.md:797-807; Bellman-Ford PAPER.md:809-817).  The paper's matrices (Vuduc
suite, tab:matrixtable) are not in the container: a uniform random symmetric
matrix of the same order of size stands in.  One JSON line per measurement.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps, flush):
    import numpy as np
    import torch
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=1_000_000)
    ap.add_argument("--nnz", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--variants", default="", help="';'-separated option sets to also time for R=1")
    ap.add_argument("--mode", default="uniform", help="uniform | banded (FEM-like profile, --band)")
    ap.add_argument("--band", type=int, default=64)
    ap.add_argument("--ranks", default="1,32")
    ap.add_argument("--no-sssp", action="store_true")
    ap.add_argument("--band-shifts", default="", help="also time band-ordered plans (symmetric and naive) "
                                                      "with these band shifts (bands on the column index)")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2406_09266_b200 as systec
    from synth.workloads import make
    w = make("sym2", 2, a.dim, a.nnz, 1, seed=11, mode=a.mode, band=a.band)
    rng = np.random.default_rng(12)
    flush = torch.empty(64 << 20, device="cuda")
    di, dv = torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda()
    sym = systec.Plan(2, a.dim, di, dv, window=True)
    ei, ev = systec.expand_symmetric(2, a.dim, di, dv)
    gen = systec.plan_create_general(2, a.dim, ei, ev)
    m = int(ev.shape[0])
    for R in (int(r) for r in a.ranks.split(",")):
        B = torch.from_numpy(rng.uniform(-1, 1, (a.dim, R)).astype(np.float32)).cuda()
        C1 = torch.empty((a.dim, R), device="cuda")
        C2 = torch.empty((a.dim, R), device="cuda")
        t_win = timed(lambda: sym.execute(B, C1), a.reps, flush)                  # windowed when the plan has it
        launch = sym.last_launch()
        t_sym = timed(lambda: sym.execute(B, C1, window=-1), a.reps, flush)      # the symmetric kernel: one red per entry
        t_gen = timed(lambda: gen.execute(B, C2), a.reps, flush)
        rel = float(((C1 - C2).abs().max() / C1.abs().max()).item())
        st = sym.stats()
        eff = (a.nnz * 12 + st["G"] * R * 4 + a.dim * R * 4) / (t_sym * 1e-3) / 1e9
        print(json.dumps({"kernel": "SSYMV" if R == 1 else f"SSYMM R={R}", "matrix": a.mode,
                          "band": a.band if a.mode == "banded" else None, "dim": a.dim, "stored_nnz": a.nnz,
                          "bandwidth": st["bandwidth"], "window_blocks": st["window_blocks"],
                          "window_kernel_ran": launch["kernel_id"] >= 2_000_000_000, "t_window_ms": t_win,
                          "expanded_nnz": m, "t_sym_ms": t_sym, "t_naive_ms": t_gen, "speedup": t_gen / t_sym,
                          "gnnz_s": a.nnz / t_sym / 1e6, "eff_gbs": eff, "paper_ssymv_speedup_vs_naive_finch": 1.45,
                          "max_rel_diff": rel}), flush=True)
    for sh in (int(x) for x in filter(None, a.band_shifts.split(","))):
        symb = systec.Plan(2, a.dim, di, dv, band_shift=sh)
        genb = systec.Plan(2, a.dim, ei, ev, band_shift=sh, general=True)
        for R in (int(r) for r in a.ranks.split(",")):
            B = torch.from_numpy(rng.uniform(-1, 1, (a.dim, R)).astype(np.float32)).cuda()
            C1 = torch.empty((a.dim, R), device="cuda")
            C2 = torch.empty((a.dim, R), device="cuda")
            t_sym = timed(lambda: symb.execute(B, C1), a.reps, flush)
            t_gen = timed(lambda: genb.execute(B, C2), a.reps, flush)
            t_gen_lex = timed(lambda: gen.execute(B, C2), a.reps, flush)
            rel = float(((C1 - C2).abs().max() / C1.abs().max()).item())
            print(json.dumps({"kernel": "SSYMV" if R == 1 else f"SSYMM R={R}", "matrix": a.mode, "band_shift": sh,
                              "plan_band_shift": symb.stats()["band_shift"], "t_sym_banded_ms": t_sym,
                              "t_naive_banded_ms": t_gen, "t_naive_lex_ms": t_gen_lex,
                              "speedup_vs_best_naive": min(t_gen, t_gen_lex) / t_sym, "max_rel_diff": rel}),
                  flush=True)
        symb.destroy()
        genb.destroy()
    if a.variants:
        B = torch.from_numpy(rng.uniform(-1, 1, (a.dim, 1)).astype(np.float32)).cuda()
        C1 = torch.empty((a.dim, 1), device="cuda")
        for v in a.variants.split(";"):
            o = {k: int(x) for k, x in (kv.split("=") for kv in filter(None, v.split(",")))}
            t1 = timed(lambda: sym.execute(B, C1, **o), a.reps, flush)
            t2 = timed(lambda: gen.execute(B, C1, **o), a.reps, flush)
            print(json.dumps({"kernel": "SSYMV", "opts": o, "t_sym_ms": t1, "t_naive_ms": t2,
                              "launch": sym.last_launch()}), flush=True)
    if a.no_sssp:
        return
    # Bellman-Ford to convergence (device-graph loop vs host loop); positive
    # weights (the uniform(-1, 1) values above would hold negative cycles)
    sp = systec.Plan(2, a.dim, di, (dv.abs() + 0.1).contiguous())
    for loop in ("graph", "host"):
        os.environ["SYSTEC_SSSP_LOOP"] = loop
        sp.sssp(0)
        torch.cuda.synchronize()
        t0 = __import__("time").perf_counter()
        dist, iters = sp.sssp(0)
        torch.cuda.synchronize()
        dt = (__import__("time").perf_counter() - t0) * 1e3
        print(json.dumps({"kernel": "SSSP (Bellman-Ford to convergence)", "loop": loop, "dim": a.dim,
                          "stored_nnz": a.nnz, "relaxations": iters, "t_ms": dt, "ms_per_relaxation": dt / iters}),
              flush=True)
    os.environ.pop("SYSTEC_SSSP_LOOP", None)
    d = torch.from_numpy(rng.uniform(0, 100, a.dim).astype(np.float32)).cuda()
    y = torch.empty_like(d)
    t_mp = timed(lambda: sym.minplus(d, y), a.reps, flush)
    print(json.dumps({"kernel": "Bellman-Ford (min,+) relaxation", "dim": a.dim, "stored_nnz": a.nnz,
                      "t_ms": t_mp, "gnnz_s": a.nnz / t_mp / 1e6}), flush=True)


if __name__ == "__main__":
    main()
