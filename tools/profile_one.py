"""Run a few executes of one config for ncu (no timing printed as a result).

    python tools/profile_one.py --config c2 --iters 3 [--opts K=33,stages=2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--opts", default="")
    a = ap.parse_args()
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
    opts = {k: int(v) for k, v in (kv.split("=") for kv in filter(None, a.opts.split(",")))}
    w = generate(a.config)
    plan = systec.Plan(w.order, w.dim, torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda())
    B = torch.from_numpy(w.B).cuda()
    C = torch.empty((w.dim, w.R), device="cuda")
    for _ in range(a.iters):
        plan.execute(B, C, **opts)
    torch.cuda.synchronize()
    print("ok", a.config, plan.last_launch(), flush=True)


if __name__ == "__main__":
    main()
