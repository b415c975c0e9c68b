import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle, paper_2406_09266_b200 as systec
from synth import small_random
from gpu_util import parity
for (n, dim, nnz, R) in [(3, 300, 20000, 32), (3, 5000, 100000, 64)]:
    w = small_random(n, dim, nnz, R, seed=3, diag_frac=0.1)
    Cref, S = oracle.mttkrp(n, dim, w.idx, w.vals, w.B)
    plan = systec.Plan(n, dim, torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda())
    for d in (2, 4, 8):
        for pos1 in (-1, 1):
            C = plan.execute(torch.from_numpy(w.B).cuda(), tma_gather=d, pos1_accumulate=pos1)
            torch.cuda.synchronize()
            print(n, dim, R, d, pos1, plan.last_launch()['kernel_id'], parity(C.cpu().numpy(), Cref, S))
print("tma ok")
