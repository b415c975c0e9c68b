"""Small invocations of every kernel path, for compute-sanitizer runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate, scramble, small_random

    def dev(*a):
        return [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in a]

    w = generate("c1", cache=False)
    si, sv = scramble(w.idx, w.vals, seed=1)
    di, dv, dB = dev(si, sv, w.B)
    systec.mttkrp(3, w.dim, di, dv, dB)
    for n, dim, nnz, R in ((3, 300, 120000, 32), (4, 50, 100000, 16), (5, 30, 100000, 16), (2, 400, 5000, 5),
                           (3, 100, 3000, 129)):
        w = small_random(n, dim, nnz, R, seed=n, diag_frac=0.1)
        di, dv, dB = dev(w.idx, w.vals, w.B)
        plan = systec.Plan(n, dim, di, dv)
        for opts in ({}, {"prefetch": 1}, {"copies": 4}, {"vpl": 2}, {"force_scalar": 1}, {"pos1_accumulate": 1}):
            plan.execute(dB, **opts)
        if (n, R) in ((3, 32), (5, 16)):
            for abl in (1, 2, 3):
                plan.execute(dB, ablation=abl, copies=1, pos1_accumulate=1 if n == 5 else -1)
        plan.destroy()
        ei, ev = systec.expand_symmetric(n, dim, di, dv)
        gplan = systec.plan_create_general(n, dim, ei, ev)
        gplan.execute(dB)
        gplan.destroy()
    # band-major plans (explicit shift) and the fixed-rank builds with every variant they have
    for n, dim, nnz, R, shift in ((3, 3000, 150000, 32, 8), (3, 3000, 150000, 16, 9), (4, 200, 100000, 16, 5),
                                  (5, 60, 80000, 32, 3)):
        w = small_random(n, dim, nnz, R, seed=n + 10, diag_frac=0.1)
        di, dv, dB = dev(w.idx, w.vals, w.B)
        plan = systec.Plan(n, dim, di, dv, band_shift=shift)
        for opts in ({}, {"occupancy": 1}, {"occupancy": 1, "pos1_accumulate": 1}, {"static_ranges": 1},
                     {"fixed_rank": -1}, {"copies": 3}):
            plan.execute(dB, **opts)
        if n == 3:
            plan.ttm(dB)
        plan.destroy()
    systec.mttkrp_host(3, 64, *[a for a in (generate("c1", cache=False).idx, generate("c1", cache=False).vals,
                                             generate("c1", cache=False).B)])
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
