"""One short CP-ALS run on a BASELINE config for ncu captures of the CP-ALS
kernels (pass_tc32 / gram / apply / cp_small / reduce_partials / finish):
    ncu --set full -k regex:pass_tc32 -s 1 -c 1 python tools/profile_cpd.py c3"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    w = generate(name)
    plan = systec.Plan(w.order, w.dim, torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda())
    B = torch.from_numpy(w.B).cuda()
    plan.cp_als(B, max_iters=iters, tol=0.0)
    torch.cuda.synchronize()
    plan.destroy()


if __name__ == "__main__":
    main()
