"""The one-shot device call systec_mttkrp on a config (for ncu launch lists and
event timings of prepare + execute).

    python tools/profile_oneshot.py c2 [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate

    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    w = generate(name)
    di, dv = torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda()
    B = torch.from_numpy(w.B).cuda()
    C = torch.empty((w.dim, w.R), device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps + 2):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        systec.mttkrp(w.order, w.dim, di, dv, B, C)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"config": name, "one_shot_ms_min": min(ts[2:]), "one_shot_ms_med": sorted(ts[2:])[len(ts[2:]) // 2]}))


if __name__ == "__main__":
    main()
