"""Host->device copy throughput of this box (dev aid for the host-buffer
call): one pinned buffer of c2's input size copied in 1..64 chunks on 1, 2
or 4 streams.  Prints JSON lines."""
import json

import torch


def main():
    nbytes = 172_800_000
    src = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    dst = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    for chunks in (1, 4, 16, 64):
        for ns in (1, 2, 4):
            streams = [torch.cuda.Stream() for _ in range(ns)]
            per = (src.numel() + chunks - 1) // chunks
            best = 1e9
            for rep in range(6):
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                for s in streams:
                    s.wait_event(a)
                for k in range(chunks):
                    lo, hi = k * per, min(src.numel(), (k + 1) * per)
                    with torch.cuda.stream(streams[k % ns]):
                        dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
                for s in streams:
                    torch.cuda.current_stream().wait_stream(s)
                b.record()
                torch.cuda.synchronize()
                if rep:
                    best = min(best, a.elapsed_time(b))
            print(json.dumps({"chunks": chunks, "streams": ns, "ms": best, "gbs": nbytes / best / 1e6}), flush=True)


if __name__ == "__main__":
    main()
