#!/usr/bin/env python
"""Benchmark of the B200 symmetric sparse MTTKRP (SySTeC hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl systec|reference]

A step = one execute of the whole hot path on one batch: zero C + the MTTKRP
kernel over every stored non-zero of the config (inputs resident in HBM, the
plan — canonicalised sorted stream — built once before timing, as the paper
excludes rearrangement).  With N > 1 (torchrun) the sorted
stream is split into N contiguous nnz-balanced slices, each rank computes a
partial C, and C is summed with one NCCL all-reduce per step:
strong scaling of one problem.

Prints ONE JSON line on rank 0.  See DESIGN.md §Measurement for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stored nonzeros/sec and achieved HBM GB/s (fraction of roofline) for symmetric MTTKRP"
UNIT = "nnz/s"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="systec", choices=["systec", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline-only", action="store_true",
                    help="print only the cpu_baseline leg (the oracle on the host), e.g. with --oracle-threads 1")
    ap.add_argument("--oracle-threads", type=int, default=0, help="threads for the cpu_baseline leg (0 = all)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--opts", default="", help="kernel options, e.g. K=33,stages=2,pos1_accumulate=1")
    ap.add_argument("--dist-backend", default="nccl", help="collective backend for N>1 (gloo: code-path tests)")
    ap.add_argument("--same-device", action="store_true",
                    help="test mode: every rank on cuda:0 (with --dist-backend gloo; no kernel waits on another)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(config):
    """DRAM bytes per launch of the kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(config, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.02):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.period, self.index = period, index
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def report(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def bytes_eff(order, nnz, G, R, dim):
    """SURVEY.md §8(d) / DESIGN.md: indices + values + one B row per distinct
    index of each stored entry + one write of C."""
    return nnz * (4 * order + 4) + G * R * 4 + dim * R * 4


def l2_model(w, st, nnz_local, kern_ms, launch):
    """Lower bound from the measured L2 rates (profiles/r01_microbench.json):
    t >= max(stream / HBM read, gathers / L2 gather rate, reds / L2 red rate),
    with the rates of the row size (64-B rows for R = 16, 128-B rows
    otherwise) and of the measured table size nearest the footprint (B for
    the gathers; C and its replicas for the reductions)."""
    import math
    try:
        with open(os.path.join(ROOT, "profiles", "r01_microbench.json")) as f:
            mb = json.load(f)
    except Exception:
        return None
    n, R = w.order, w.R
    row = R * 4
    kind = "64B" if row == 64 and "gather_64B_rows_gbs" in mb else "128B"

    def nearest(table, mbytes):
        key = min(table, key=lambda k: abs(math.log(float(k[:-2])) - math.log(max(mbytes, 1e-3))))
        return table[key] * 1e9, key

    hbm = mb["hbm_read_gbs"] * 1e9
    gat, gkey = nearest(mb[f"gather_{kind}_rows_gbs"], w.dim * row / 1e6)
    red, rkey = nearest(mb[f"red_v4_{kind}_rows_gbs"], max(1, launch.get("copies", 1)) * w.dim * row / 1e6)
    stream = nnz_local * (4 * n + 4)
    gathers = st["G"] * row
    n1 = sum(h for code, h in enumerate(st["pattern_hist"]) if not code & 1)   # entries with c1 != c0
    pos1 = launch.get("pos1", 0) == 1
    red_rows = st["lead_runs"] + (st["G"] - nnz_local) - ((n1 - min(n1, st["pos1_runs"])) if pos1 else 0)
    reds = red_rows * row
    t = max(stream / hbm, gathers / gat, reds / red)
    return {"stream_bytes": stream, "gather_bytes": gathers, "red_payload_bytes": reds,
            "hbm_read_gbs": hbm / 1e9, "l2_gather_gbs": gat / 1e9, "l2_red_gbs": red / 1e9,
            "t_lower_ms": t * 1e3, "frac_of_l2_bound": t * 1e3 / kern_ms,
            "source": f"profiles/r01_microbench.json (tools/microbench.cu): {kind} rows, gathers from a "
                      f"{gkey} table, red.v4 into a {rkey} table"}


def cpu_baseline(w, target_wall=4.0, max_entries=None, threads=0):
    """The oracle as it stands on the host cores, on a bounded sample (the
    first m stored entries), scaled up until one run takes ~target_wall s."""
    import oracle
    T = threads if threads > 0 else oracle.default_threads()
    m = min(w.nnz, 50_000)
    while True:
        t0 = time.perf_counter()
        oracle.mttkrp(w.order, w.dim, w.idx[:m], w.vals[:m], w.B, threads=T)
        dt = time.perf_counter() - t0
        if dt >= target_wall or m >= w.nnz or (max_entries and m >= max_entries):
            break
        m = min(w.nnz, int(m * max(2.0, min(8.0, target_wall / max(dt, 1e-3)))))
    out = {"value": m / dt, "unit": UNIT, "cores": T, "kind": "oracle",
           "sample": f"first {m} of {w.nnz} stored entries of {w.name} (sorted order), "
                     f"full expansion + fp64 accumulation into [dim][R], {dt:.2f} s wall on {T} threads"}
    out["one_core_context"] = one_core_context(w)
    return out


def one_core_context(w, target_wall=1.0):
    """The paper's own experiment is symmetric vs naive on ONE core
    (PAPER.md:740, 886): the expansion oracle and the symmetric method, both
    plain C in fp64 on one thread, on the same bounded sample.  Context only."""
    import oracle
    m = min(w.nnz, 20_000)
    while True:
        t0 = time.perf_counter()
        oracle.mttkrp(w.order, w.dim, w.idx[:m], w.vals[:m], w.B, threads=1)
        t_exp = time.perf_counter() - t0
        if t_exp >= target_wall or m >= w.nnz:
            break
        m = min(w.nnz, int(m * max(2.0, min(8.0, target_wall / max(t_exp, 1e-3)))))
    t0 = time.perf_counter()
    oracle.mttkrp_symmetric(w.order, w.dim, w.idx[:m], w.vals[:m], w.B)
    t_sym = time.perf_counter() - t0
    return {"sample_entries": m, "expansion_nnz_s": m / t_exp, "symmetric_nnz_s": m / t_sym,
            "speedup": t_exp / t_sym, "paper_one_core_speedup_max": {"3": 3.38, "4": 7.35, "5": 29.8}[str(w.order)]
            if w.order in (3, 4, 5) else None}


def run_reference(args, w):
    """--impl reference: the oracle, as it stands, on the host cores."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    T = oracle.default_threads()
    budget = 150.0 / max(1, args.steps + args.warmup)           # seconds per step
    m = min(w.nnz, 20_000)
    while True:                                                   # calibrate the sample
        t0 = time.perf_counter()
        oracle.mttkrp(w.order, w.dim, w.idx[:m], w.vals[:m], w.B, threads=T)
        dt = time.perf_counter() - t0
        if dt >= 0.5 * budget or m >= w.nnz:
            break
        m = min(w.nnz, int(m * max(2.0, min(8.0, 0.6 * budget / max(dt, 1e-3)))))
    for _ in range(args.warmup):
        oracle.mttkrp(w.order, w.dim, w.idx[:m], w.vals[:m], w.B, threads=T)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.mttkrp(w.order, w.dim, w.idx[:m], w.vals[:m], w.B, threads=T)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = m * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(w, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "oracle",
                             "sample": f"first {m} of {w.nnz} stored entries per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(w, args):
    from synth import CONFIGS
    return {"workload": f"{w.name}: {CONFIGS[w.name].describe}" if w.name in CONFIGS else w.name,
            "order": w.order, "dim": w.dim, "nnz": w.nnz, "R": w.R,
            "l2": "flushed between timed steps (256 MiB write outside the events)",
            "parallelism": f"nnz-slices x{args.gpus} + all-reduce(C)" if args.gpus > 1 else "1 GPU"}


def parse_opts(s):
    out = {}
    for kv in filter(None, s.split(",")):
        k, v = kv.split("=")
        out[k.strip()] = int(v)
    return out


def main():
    args = parse()
    from synth import generate
    w = generate(args.config)
    if args.impl == "reference":
        run_reference(args, w)
        return
    if args.cpu_baseline_only:
        print(json.dumps({"config": config_dict(w, args),
                          "cpu_baseline": cpu_baseline(w, threads=args.oracle_threads)}), flush=True)
        return

    import torch
    import paper_2406_09266_b200 as systec
    from paper_2406_09266_b200.shard import reduce_partials, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    # this rank's slice of the sorted stream (whole stream at N = 1)
    lo, hi = shard_range(w.nnz, rank, world)
    idx_d = torch.from_numpy(w.idx[lo:hi]).to(dev)
    vals_d = torch.from_numpy(w.vals[lo:hi]).to(dev)
    B_d = torch.from_numpy(w.B).to(dev)
    C_d = torch.empty((w.dim, w.R), dtype=torch.float32, device=dev)
    plan = systec.Plan(w.order, w.dim, idx_d, vals_d)
    del idx_d, vals_d
    st = plan.stats()
    opts = parse_opts(args.opts)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step(ev=None):
        # one pass of the hot path: zero C (+ replicas) + MTTKRP kernel (+ replica sum)
        if ev:
            ev[0].record(stream)
        plan.execute(B_d, C_d, **opts)
        if ev:
            ev[1].record(stream)
        if dist is not None:
            reduce_partials(C_d)
        if ev:
            ev[2].record(stream)

    for _ in range(max(3, args.warmup)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))              # L2 flush between timed steps, outside the events
            step(ev[k])
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [e[0].elapsed_time(e[2]) for e in ev]
    kern_ms = [e[0].elapsed_time(e[1]) for e in ev]
    tot_ms = float(np.sum(step_ms))
    if dist is not None:
        t = torch.tensor([tot_ms, float(np.sum(kern_ms))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, kern_tot = t.tolist()
    else:
        kern_tot = float(np.sum(kern_ms))
    ms_per_step = tot_ms / args.steps
    kern_avg_ms = kern_tot / args.steps

    # warm back-to-back (B L2-resident from the previous call): context number
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        plan.execute(B_d, C_d, **opts)
    e1.record(stream)
    torch.cuda.synchronize()
    warm_ms = e0.elapsed_time(e1) / 20

    value = w.nnz / (ms_per_step * 1e-3)          # all ranks together process the whole tensor
    # roofline of the dominant kernel (mttkrp_sym_kernel) on this rank's slice
    G_all = st["G"]
    if dist is not None:
        t = torch.tensor([G_all], device=dev, dtype=torch.float64)
        dist.all_reduce(t)
        G_all = int(t.item())
    local_bytes = bytes_eff(w.order, hi - lo, st["G"], w.R, w.dim)
    achieved = local_bytes / (kern_avg_ms * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    traffic = load_traffic(w.name) if world == 1 else None

    line = None
    if rank == 0:
        launch = plan.last_launch()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(w, args),
            "eff_gbs": bytes_eff(w.order, w.nnz, G_all, w.R, w.dim) / (ms_per_step * 1e-3) / 1e9,
            "bytes_eff_per_step": bytes_eff(w.order, w.nnz, G_all, w.R, w.dim),
            "frac_of_8tbs": bytes_eff(w.order, w.nnz, G_all, w.R, w.dim) / (ms_per_step * 1e-3) / 8e12,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "mttkrp_sym_kernel", "kernel_ms": kern_avg_ms,
                         "kernel_ms_includes": "C zeroing (memset) + kernel (+ replica sum when C < 4 MB)",
                         "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                         "algorithmic_bytes_per_launch": local_bytes,
                         "note": "B gathers and C reductions are served by L2 (B, C L2-resident): "
                                 "bytes_eff/t can exceed the HBM copy peak; l2_model gives the "
                                 "binding L2 bound"},
            "l2_model": l2_model(w, st, hi - lo, kern_avg_ms, launch),
            "warm_ms_per_step": warm_ms,
            "step_ms_min": float(np.min(step_ms)), "step_ms_median": float(np.median(step_ms)),
            # our kernels per execute: the MTTKRP kernel, + the replica sum (copies > 1; the
            # replicas are zeroed by cudaMemsetAsync), + zero_output_kernel when a single C
            # is zeroed together with the dynamic-distribution counter
            "gpu_launches": args.steps * (1 + (launch.get("copies", 1) > 1)
                                          + (launch.get("copies", 1) == 1 and launch.get("dynamic", 0) == 1)),
            "launch": launch,
            "plan_stats": {k: st[k] for k in ("G", "expanded", "lead_runs", "max_lead_run", "pos1_runs")},
        }
        line["clocks"] = clk.report()

    # end to end through the public host-buffer call: H2D idx/vals/B from pinned
    # memory, prepare, execute, D2H C — every step
    if rank == 0 and world == 1 and not args.no_e2e:
        pin_idx = torch.from_numpy(w.idx).pin_memory()
        pin_vals = torch.from_numpy(w.vals).pin_memory()
        pin_B = torch.from_numpy(w.B).pin_memory()
        pin_C = torch.empty((w.dim, w.R), dtype=torch.float32).pin_memory()
        systec.mttkrp_host(w.order, w.dim, pin_idx, pin_vals, pin_B, C=pin_C)   # warm-up
        ts = []
        for _ in range(args.e2e_steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            systec.mttkrp_host(w.order, w.dim, pin_idx, pin_vals, pin_B, C=pin_C)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        e2e_ms = float(np.mean(ts))
        line["e2e"] = {"value": w.nnz / (e2e_ms * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": w.idx.nbytes + w.vals.nbytes + w.B.nbytes,
                       "d2h_bytes_per_step": pin_C.numel() * 4, "ms_per_step": e2e_ms,
                       "includes": "H2D + validate/canonicalise/sort-check/gather/stats + execute + D2H"}
    # N > 1: every rank, every step: H2D of its slice + B from pinned memory,
    # plan creation (validate/canonicalise/sort-check/gather/stats), execute,
    # one all-reduce of C, D2H of C; time = max over ranks
    if world > 1 and not args.no_e2e:
        pin_idx = torch.from_numpy(np.ascontiguousarray(w.idx[lo:hi])).pin_memory()
        pin_vals = torch.from_numpy(np.ascontiguousarray(w.vals[lo:hi])).pin_memory()
        pin_B = torch.from_numpy(w.B).pin_memory()
        pin_C = torch.empty((w.dim, w.R), dtype=torch.float32).pin_memory()

        def e2e_step():
            di = pin_idx.to(dev, non_blocking=True)
            dv = pin_vals.to(dev, non_blocking=True)
            dB = pin_B.to(dev, non_blocking=True)
            pl = systec.Plan(w.order, w.dim, di, dv)
            Cd = pl.execute(dB)
            reduce_partials(Cd)
            pin_C.copy_(Cd, non_blocking=True)
            torch.cuda.synchronize()
            pl.destroy()

        e2e_step()
        ts = []
        for _ in range(args.e2e_steps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t0)
        t = torch.tensor([float(np.mean(ts))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            e2e_ms = t.item() * 1e3
            line["e2e"] = {"value": w.nnz / (e2e_ms * 1e-3), "unit": UNIT,
                           "h2d_bytes_per_step": (w.idx.nbytes + w.vals.nbytes) + world * w.B.nbytes,
                           "d2h_bytes_per_step": world * pin_C.numel() * 4, "ms_per_step": e2e_ms,
                           "includes": "per rank: H2D slice + plan creation + execute + all-reduce(C) + D2H; "
                                       "max over ranks (host clock around synchronised steps)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, threads=args.oracle_threads)
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.destroy()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
