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
    a = ap.parse_args()
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
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
    print("ok", a.config, sym.stats()["expanded"])


if __name__ == "__main__":
    main()
