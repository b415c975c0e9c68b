"""NEXT-2 timing: symmetric CP-ALS iterations on the BASELINE configs (the
plan is built once and reused by every iteration — the prepare cost is
amortised).  Prints one JSON line per config."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
    for name in (sys.argv[1] if len(sys.argv) > 1 else "c2,c4,c5").split(","):
        w = generate(name)
        plan = systec.Plan(w.order, w.dim, torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda())
        B = torch.from_numpy(w.B).cuda()
        plan.cp_als(B.clone(), max_iters=2, tol=0.0)       # warm-up
        torch.cuda.synchronize()
        iters = int(os.environ.get("CPD_ITERS", "50"))
        t0 = time.perf_counter()
        _, lam, fits = plan.cp_als(B.clone(), max_iters=iters, tol=0.0)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / (iters + 1)      # iters updates + 1 fit-only pass (whole call, wall)
        C = torch.empty_like(B)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            plan.execute(B, C)
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"config": name, "R": w.R, "iters": iters,
                          "loop": os.environ.get("SYSTEC_CPALS_LOOP", "auto (graph when iters >= 16)"),
                          "ms_per_iteration": dt * 1e3,
                          "mttkrp_ms": a.elapsed_time(b) / 10, "fits": fits.tolist()[-3:]}), flush=True)
        plan.destroy()


if __name__ == "__main__":
    main()
