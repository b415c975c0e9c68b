"""NEXT-4 timing: symmetric TTM (canonical half of the output, packed) vs the
naive TTM over the expanded tensor (full output) — the paper's TTM experiment
(2.09x over naive Finch at high density, low rank).
Replication of the output is excluded, as in the paper."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2406_09266_b200 as systec
    from synth.workloads import make
    flush = torch.empty(64 << 20, device="cuda")

    def timed(fn, reps=20):
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

    for dim, nnz, R in ((500, 5_000_000, 8), (500, 5_000_000, 32), (1000, 10_000_000, 16)):
        w = make(f"ttm{dim}", 3, dim, nnz, R, seed=dim, mode="uniform")
        di, dv, dB = (torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda(), torch.from_numpy(w.B).cuda())
        sym = systec.Plan(3, dim, di, dv)
        Cp = torch.empty((dim * (dim + 1) // 2, R), device="cuda")
        t_sym = timed(lambda: sym.ttm(dB, packed=Cp))
        ei, ev = systec.expand_symmetric(3, dim, di, dv)
        gen = systec.plan_create_general(3, dim, ei, ev)
        Cf = torch.empty((dim * dim, R), device="cuda")
        t_gen = timed(lambda: gen.ttm(dB, packed=Cf))
        full = sym.ttm(dB, full=True)
        gen.ttm(dB, packed=Cf)
        torch.cuda.synchronize()
        rel = float(((full.view(-1, R) - Cf).abs().max() / Cf.abs().max()).item())
        print(json.dumps({"dim": dim, "nnz": nnz, "density": nnz / (dim * (dim + 1) * (dim + 2) / 6), "R": R,
                          "expanded_nnz": int(ev.shape[0]), "t_sym_ms": t_sym, "t_naive_ms": t_gen,
                          "speedup": t_gen / t_sym, "paper_speedup_vs_naive_finch": 2.09, "max_rel_diff": rel}),
              flush=True)
        for x in (sym, gen):
            x.destroy()
        del ei, ev, Cp, Cf, full
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
