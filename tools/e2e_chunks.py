"""Time the pipelined host-buffer call for several pipeline depths (env
SYSTEC_HOST_CHUNKS is read once per process, so one process per depth)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, time, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2406_09266_b200 as systec
from synth import generate
w = generate(%r)
pin = [torch.from_numpy(a).pin_memory() for a in (w.idx, w.vals, w.B)]
C = torch.empty((w.dim, w.R), dtype=torch.float32).pin_memory()
systec.mttkrp_host(w.order, w.dim, *pin, C=C)
ts = []
for _ in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    systec.mttkrp_host(w.order, w.dim, *pin, C=C)
    ts.append(time.perf_counter() - t0)
h2d = pin[0].numel() * 4 + pin[1].numel() * 4 + pin[2].numel() * 4
x = torch.empty(h2d // 4, dtype=torch.float32).pin_memory(); d = torch.empty_like(x, device="cuda")
d.copy_(x); torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): d.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t_h2d = (time.perf_counter() - t0) / 5
print(json.dumps({"config": %r, "chunks": %s, "e2e_ms": 1e3 * float(np.median(ts)), "h2d_only_ms": 1e3 * t_h2d,
                  "h2d_gbs": h2d / t_h2d / 1e9}))
'''

for cfg in (sys.argv[1] if len(sys.argv) > 1 else "c2").split(","):
    for ch in (1, 4, 8, 16, 32, 64):
        env = dict(os.environ, SYSTEC_HOST_CHUNKS=str(ch))
        out = subprocess.run([sys.executable, "-c", CODE % (ROOT, cfg, cfg, ch)], env=env, capture_output=True,
                             text=True, timeout=600)
        print(out.stdout.strip() or out.stderr[-500:], flush=True)
