"""Time kernel option variants on one or more configs (CUDA events, L2 flushed
between runs) and print one JSON object per variant.  Tuning aid only.

    python tools/sweep.py --configs c2,c5 --variants "vpl=1;vpl=2;vpl=4,K=5"
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_variant(s):
    return {k: int(v) for k, v in (kv.split("=") for kv in filter(None, s.split(",")))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2")
    ap.add_argument("--variants", default="")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--split", type=int, default=-1, help="plan creation (split-plan experiment builds): -1 default, 1 split, 0 no split")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
    flush = torch.empty(64 << 20, device="cuda")
    variants = [parse_variant(v) for v in a.variants.split(";")] if a.variants else [{}]
    for name in a.configs.split(","):
        w = generate(name)
        kw = {} if a.split < 0 else {"split": bool(a.split)}   # split: experiment builds only
        plan = systec.Plan(w.order, w.dim, torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda(), **kw)
        st = plan.stats()
        B = torch.from_numpy(w.B).cuda()
        C = torch.empty((w.dim, w.R), device="cuda")
        ref = None
        bytes_eff = w.nnz * (4 * w.order + 4) + st["G"] * w.R * 4 + w.dim * w.R * 4
        for opts in variants:
            try:
                for _ in range(3):
                    plan.execute(B, C, **opts)
                torch.cuda.synchronize()
            except Exception as ex:  # noqa: BLE001
                print(json.dumps({"config": name, "opts": opts, "error": str(ex)}), flush=True)
                continue
            out = C.clone()
            if ref is None:
                ref = out
            diff = float((out - ref).abs().max())
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.execute(B, C, **opts)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            warm = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.execute(B, C, **opts)
                e1.record()
                torch.cuda.synchronize()
                warm.append(e0.elapsed_time(e1))
            med = float(np.median(ts))
            print(json.dumps({"config": name, "opts": opts, "launch": plan.last_launch(),
                              "ms_med": med, "ms_min": float(np.min(ts)), "warm_ms_med": float(np.median(warm)),
                              "gnnz_s": w.nnz / med / 1e6, "eff_gbs": bytes_eff / med / 1e6,
                              "max_abs_diff_vs_first": diff}), flush=True)
        plan.destroy()


if __name__ == "__main__":
    main()
