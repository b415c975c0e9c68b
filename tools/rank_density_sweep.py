"""The paper's MTTKRP experiment shape (fig:mttkrp_performance, PAPER.md:868-884:
"3-, 4-, and 5-dimensional MTTKRP performance over varying sparsity and
numerical rank") on the B200: symmetric kernel vs the naive kernel over the
expanded tensor, for ranks R and densities per order.  Uniform random
symmetric tensors (the paper's are Erdős–Rényi, sizes in the omitted figure).
One JSON line per point."""
import json
import math
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

    def timed(fn, reps=10):
        for _ in range(2):
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

    # (order, dim, stored nnz list) — densities spanning ~3 orders of magnitude
    grid = [(3, 2000, [200_000, 2_000_000, 20_000_000]),
            (4, 400, [200_000, 2_000_000, 20_000_000]),
            (5, 120, [200_000, 2_000_000, 10_000_000])]
    rng = np.random.default_rng(0)
    for n, dim, nnzs in grid:
        canon = math.comb(dim + n - 1, n)
        for nnz in nnzs:
            w = make(f"rd{n}", n, dim, nnz, 1, seed=nnz + n, mode="uniform")
            di, dv = torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda()
            sym = systec.Plan(n, dim, di, dv)
            ei, ev = systec.expand_symmetric(n, dim, di, dv)
            gen = systec.plan_create_general(n, dim, ei, ev)
            m = int(ev.shape[0])
            del ei, ev
            for R in (4, 16, 32, 64):
                B = torch.from_numpy(rng.uniform(-1, 1, (dim, R)).astype(np.float32)).cuda()
                C = torch.empty((dim, R), device="cuda")
                t_s = timed(lambda: sym.execute(B, C))
                t_n = timed(lambda: gen.execute(B, C))
                print(json.dumps({"order": n, "dim": dim, "nnz": nnz, "density": nnz / canon, "expanded": m, "R": R,
                                  "t_sym_ms": t_s, "t_naive_ms": t_n, "speedup": t_n / t_s,
                                  "sym_gnnz_s": nnz / t_s / 1e6}), flush=True)
            sym.destroy()
            gen.destroy()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
