"""Time the CPU oracle (and the symmetric fp64 CPU reference) on the host:
T = all cores and T = 1, on a bounded sample of each config.  Context for
BASELINE.md (the oracle is a reported baseline, never tuned)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    from oracle import symmetric_ref
    from synth import generate
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]
    T = oracle.default_threads()
    for name in cfgs:
        w = generate(name)
        out = {"config": name, "nnz": w.nnz, "threads": T}
        for threads, budget in ((T, 6.0), (1, 6.0)):
            m = min(w.nnz, 2000)
            while True:
                t0 = time.perf_counter()
                oracle.mttkrp(w.order, w.dim, w.idx[:m], w.vals[:m], w.B, threads=threads)
                dt = time.perf_counter() - t0
                if dt > budget / 4 or m >= w.nnz:
                    break
                m = min(w.nnz, m * 4)
            out[f"oracle_T{threads}_nnz_per_s"] = m / dt
            out[f"oracle_T{threads}_sample"] = m
            out[f"oracle_T{threads}_full_s_est"] = w.nnz / (m / dt)
        m = min(w.nnz, 200_000)
        t0 = time.perf_counter()
        symmetric_ref.mttkrp(w.order, w.dim, w.idx[:m], w.vals[:m], w.B)
        dt = time.perf_counter() - t0
        out["symmetric_numpy_nnz_per_s"] = m / dt
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
