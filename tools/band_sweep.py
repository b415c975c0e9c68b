"""Band study: plans whose stream is grouped by bands of the last (largest)
index, c_{n-1} >> shift, lexicographic within a band (chosen at plan creation:
systec_plan_opts.band_shift, -1 lexicographic, 0 auto).  Times execute (CUDA
events, L2 flushed between runs) per shift and compares each result with the
first shift's.  Tuning aid only.

    python tools/band_sweep.py --configs c3 --shifts=-1,0,18,17,16 [--R 8] [--opts occupancy=1]
    python tools/band_sweep.py --configs "" --make "3:1000000:20000000:32:uniform" --shifts=-1,0
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c3")
    ap.add_argument("--shifts", default="-1,19,18,17,16")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--opts", default="")
    ap.add_argument("--make", default="", help="extra shapes 'order:dim:nnz:R:mode[;...]' drawn by synth.make (seed 7)")
    ap.add_argument("--R", type=int, default=0, help="rank override (B drawn uniform(-1,1), seed 0)")
    a = ap.parse_args()
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
    from synth.workloads import make
    opts = {k: int(v) for k, v in (kv.split("=") for kv in filter(None, a.opts.split(",")))}
    flush = torch.empty(64 << 20, device="cuda")
    shapes = [("cfg", n) for n in filter(None, a.configs.split(","))]
    shapes += [("make", m) for m in filter(None, a.make.split(";"))]
    for kind, name in shapes:
        if kind == "cfg":
            w = generate(name)
        else:
            o, d, z, r, mode = name.split(":")
            w = make(name, int(o), int(d), int(z), int(r), 7, mode)
        idx = torch.from_numpy(w.idx).cuda()
        vals = torch.from_numpy(w.vals).cuda()
        R = a.R or w.R
        if a.R:
            g = torch.Generator().manual_seed(0)
            B = (torch.rand((w.dim, R), generator=g) * 2 - 1).cuda()
        else:
            B = torch.from_numpy(w.B).cuda()
        C = torch.empty((w.dim, R), device="cuda")
        ref = None
        for sh in (int(x) for x in a.shifts.split(",")):
            plan = systec.Plan(w.order, w.dim, idx, vals, band_shift=sh)
            st = plan.stats()
            for _ in range(3):
                plan.execute(B, C, **opts)
            torch.cuda.synchronize()
            out = C.clone()
            if ref is None:
                ref = out
            rel = float((out - ref).abs().max() / ref.abs().max())
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.execute(B, C, **opts)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            print(json.dumps({"config": name, "R": R, "band_shift": sh, "plan_band_shift": st["band_shift"], "ms_min": ts[0], "ms_median": ts[len(ts) // 2],
                              "lead_runs": st["lead_runs"], "pos1_runs": st["pos1_runs"],
                              "max_lead_run": st["max_lead_run"], "max_abs_diff_rel_vs_unbanded": rel,
                              "launch": plan.last_launch()}), flush=True)
            del plan
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
