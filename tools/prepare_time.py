"""Plan creation ("rearrangement", excluded from the paper's timings,
PAPER.md:740) and the one-shot device call, timed per config (SURVEY.md §8(d):
prepare timed separately, min of 5; one-shot timed too).  Wall clock around
synchronised calls (plan creation synchronises the stream itself).

    python tools/prepare_time.py --configs c2,c3,c4,c5
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c4,c5")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate, scramble

    def tmin(fn):
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
            del out
        return min(ts)

    for name in a.configs.split(","):
        w = generate(name)
        di, dv = torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda()
        si, sv = scramble(w.idx, w.vals, seed=9)
        dsi, dsv = torch.from_numpy(si).cuda(), torch.from_numpy(sv).cuda()
        B = torch.from_numpy(w.B).cuda()
        C = torch.empty((w.dim, w.R), device="cuda")
        res = {"config": name, "nnz": w.nnz}
        for tag, (i, v) in (("sorted", (di, dv)), ("shuffled", (dsi, dsv))):
            for band in (0, -1):
                def mk(i=i, v=v, band=band):
                    p = systec.Plan(w.order, w.dim, i, v, band_shift=band)
                    p.destroy()
                res[f"prepare_{tag}_{'auto' if band == 0 else 'lex'}_ms"] = tmin(mk)
        plan = systec.Plan(w.order, w.dim, di, dv)
        res["plan_band_shift"] = plan.stats()["band_shift"]
        res["execute_ms"] = tmin(lambda: plan.execute(B, C))
        plan.destroy()
        res["one_shot_device_ms"] = tmin(lambda: systec.mttkrp(w.order, w.dim, di, dv, B, C))
        print(json.dumps(res), flush=True)
        del di, dv, dsi, dsv, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
