"""End-to-end host-call timing variants (dev aid): chunks x early-copy, one
process each (both knobs are read once per process).  JSON lines."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2406_09266_b200 as systec
from synth import generate
w = generate("c2")
pin = [torch.from_numpy(a).pin_memory() for a in (w.idx, w.vals, w.B)]
C = torch.empty((w.dim, w.R), dtype=torch.float32).pin_memory()
for _ in range(3):
    systec.mttkrp_host(w.order, w.dim, *pin, C=C)
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    systec.mttkrp_host(w.order, w.dim, *pin, C=C)
    b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print(json.dumps({"chunks": %s, "early": %s, "ms_min": min(ts), "ms_med": float(np.median(ts))}))
'''
for ch in (4, 8, 16):
    for early in (1, 0):
        for vc in (0, 1):
            env = dict(os.environ, SYSTEC_HOST_CHUNKS=str(ch), SYSTEC_HOST_EARLY=str(early),
                       SYSTEC_HOST_VALS_CHUNKED=str(vc))
            out = subprocess.run([sys.executable, "-c", CODE % (ROOT, ch, early)], env=env, capture_output=True,
                                 text=True, timeout=600)
            print((out.stdout.strip()[:-1] + f', "vals_chunked": {vc}}}') if out.stdout.strip() else out.stderr[-400:],
                  flush=True)
