"""Ablation of the paper's diagonal splitting (Listing 7, PAPER.md:711-729;
transform PAPER.md:616-638): the canonical entries split into A_nondiag
(strict, c_0 < ... < c_{n-1}) and A_diag (some repeated index), each its own
plan, executed back to back into the same C (the second accumulates) — vs the
single pass over all entries that the coefficient table allows.  One JSON
line per config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
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

    for name in (sys.argv[1] if len(sys.argv) > 1 else "c1,c3,c4,c5").split(","):
        w = generate(name)
        diag = np.any(w.idx[:, 1:] == w.idx[:, :-1], axis=1)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        one = systec.Plan(w.order, w.dim, dev(w.idx), dev(w.vals))
        nd = systec.Plan(w.order, w.dim, dev(w.idx[~diag]), dev(w.vals[~diag]))
        dg = systec.Plan(w.order, w.dim, dev(w.idx[diag]), dev(w.vals[diag]))
        B = dev(w.B)
        C1 = torch.empty((w.dim, w.R), device="cuda")
        C2 = torch.empty((w.dim, w.R), device="cuda")
        t_one = timed(lambda: one.execute(B, C1))

        def split():
            nd.execute(B, C2)
            dg.execute(B, C2, no_zero=1)
        t_split = timed(split)
        torch.cuda.synchronize()
        rel = float(((C1 - C2).abs().max() / C1.abs().max()).item())
        print(json.dumps({"config": name, "diag_fraction": float(diag.mean()), "t_single_pass_ms": t_one,
                          "t_split_two_nests_ms": t_split, "split_over_single": t_split / t_one,
                          "max_rel_diff": rel}), flush=True)


if __name__ == "__main__":
    main()
