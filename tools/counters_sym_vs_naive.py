"""Run one symmetric and one naive (expanded-tensor) execute of a config, for
ncu to count what the paper claims: reads of A (TMA bytes of
the stream) at 1/n!, and floating-point work at ~1/(n-1)!.

    ncu --metrics ... -k regex:mttkrp_sym python tools/counters_sym_vs_naive.py --config c2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--make", default="", help="order:dim:nnz:R — a strict (no repeated index) random tensor instead")
    a = ap.parse_args()
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate, small_random
    if a.make:
        n, dim, nnz, R = (int(x) for x in a.make.split(":"))
        w = small_random(n, dim, nnz, R, seed=nnz + n, diag_frac=0.0)
    else:
        w = generate(a.config)
    di, dv = torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda()
    B = torch.from_numpy(w.B).cuda()
    sym = systec.Plan(w.order, w.dim, di, dv)
    sym.execute(B, copies=1)
    ei, ev = systec.expand_symmetric(w.order, w.dim, di, dv)
    gen = systec.plan_create_general(w.order, w.dim, ei, ev)
    del ei, ev
    gen.execute(B, copies=1)
    torch.cuda.synchronize()
    import json
    st = sym.stats()
    print("STATS " + json.dumps({"nnz": w.nnz, "order": w.order, "R": w.R, "G": st["G"], "expanded": st["expanded"],
                                 "lead_runs": st["lead_runs"], "pos1_runs": st["pos1_runs"],
                                 "pattern_hist": st["pattern_hist"], "launch": sym.last_launch()}), flush=True)


if __name__ == "__main__":
    main()
