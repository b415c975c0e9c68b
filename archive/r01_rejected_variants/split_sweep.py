"""Single-pass vs split plans (systec_plan_create_ex SYSTEC_PLAN_SPLIT) on the
BASELINE configs: device time per execute (CUDA events, L2 flushed between
calls, median of --reps), and the prepare time of each plan.  One JSON line per
config.

    python tools/split_sweep.py --configs c2,c3,c4,c5
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
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--opts", default="{}", help="extra execute options (JSON)")
    a = ap.parse_args()
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
    extra = json.loads(a.opts)
    flush = torch.empty(64 << 20, device="cuda")
    for name in a.configs.split(","):
        w = generate(name)
        di, dv = torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda()
        B = torch.from_numpy(w.B).cuda()
        res = {"config": name}
        variants = [("single", False, {})] + [(f"split_w{k}", True, {"split_warps": k}) for k in (2, 3, 4)]
        variants += [("split_seq", True, {"split": 1})]
        plans = {}
        for label, split, vo in variants:
            if split not in plans:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                plans[split] = systec.Plan(w.order, w.dim, di, dv, split=split)
                res[f"{'split' if split else 'single'}_prepare_ms"] = round(1e3 * (time.perf_counter() - t0), 2)
            plan = plans[split]
            C = torch.empty_like(B)
            for _ in range(3):
                plan.execute(B, C, **extra, **vo)
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.execute(B, C, **extra, **vo)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            res[f"{label}_ms"] = round(ts[len(ts) // 2], 4)
            lz = plan.last_launch()
            res[f"{label}_launch"] = {k: lz[k] for k in ("grid_x", "block", "kernel_id")}
        for p in plans.values():
            p.destroy()
        best = min((v, k) for k, v in res.items() if k.startswith("split") and k.endswith("_ms") and "prepare" not in k)
        res["best_split"] = best[1]
        res["speedup"] = round(res["single_ms"] / best[0], 3)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
