#!/usr/bin/env python
"""Benchmark of the B200 symmetric sparse MTTKRP (SySTeC hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl systec|reference]

A step = one execute of the whole hot path on one batch: zero C + the MTTKRP
kernel over every stored non-zero of the config (inputs resident in HBM, the
plan — canonicalised sorted stream — built once before timing, as the paper
excludes rearrangement).  With N > 1 (torchrun) the sorted
stream is split into N contiguous nnz-balanced slices, each rank computes a
partial C, and C is summed with one NCCL all-reduce per step — or, with
``--collective reduce_scatter``, reduce-scattered into row blocks
(SURVEY.md §8(e)): strong scaling of one problem.

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
    ap.add_argument("--collective", default="all_reduce", choices=["all_reduce", "reduce_scatter"],
                    help="N>1 exchange: whole C on every rank, or a row block of C per rank")
    ap.add_argument("--no-bounds", action="store_true", help="skip the in-run L2/HBM bound measurement")
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-run ncu DRAM-traffic capture")
    ap.add_argument("--paper-rule-s", "--budget-s", type=float, default=3.0,
                    help="the paper's timing rule (min over up to 10,000 runs or this many seconds, PAPER.md:740)")
    ap.add_argument("--seed", type=int, default=None, help="another draw of the config's shape (default: its seed)")
    ap.add_argument("--warm", action="store_true",
                    help="no L2 flush between timed steps (B warm in L2); default: flushed (cold)")
    ap.add_argument("--dump-c", default="",
                    help="test mode: after timing, write the final C (rank 0; row blocks gathered) to this .npy")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(config, opts_str, timeout=240):
    """DRAM traffic of one launch of the MTTKRP kernel, measured by ncu in a
    child process of THIS bench run (same box, same build, same plan): the
    physical HBM bytes behind the roofline.  Returns a dict, or the reason it
    is unavailable."""
    import shutil
    import subprocess
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"unavailable": "ncu not found"}
    metrics = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
               "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
               "lts__t_requests_srcunit_tex_op_red.sum", "lts__t_sector_hit_rate.pct"]
    cmd = [ncu, "--metrics", ",".join(metrics), "--clock-control", "none", "--print-units", "base", "--csv",
           "-k", "regex:mttkrp_sym", "-s", "2", "-c", "1",
           sys.executable, os.path.join(ROOT, "tools", "profile_one.py"), "--config", config, "--iters", "3"]
    if opts_str:
        cmd += ["--opts", opts_str]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"ncu failed: {e!r}"[:200]}
    import csv
    import io
    vals = {}
    for row in csv.reader(io.StringIO("\n".join(l for l in out.stdout.splitlines() if l.startswith('"')))):
        if len(row) > 3 and row[-3] in metrics:
            try:
                vals[row[-3]] = float(row[-1].replace(",", ""))
            except ValueError:
                pass
    if "dram__bytes_read.sum" not in vals:
        return {"unavailable": f"ncu rc={out.returncode}: " + (out.stderr or out.stdout)[-200:]}
    return {"dram_bytes_per_launch": vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0.0),
            "dram_read_bytes": vals["dram__bytes_read.sum"], "dram_write_bytes": vals.get("dram__bytes_write.sum"),
            "ncu_kernel_ms": vals.get("gpu__time_duration.sum", 0.0) / 1e6,
            "sm_l2_port_pct": vals.get("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "l2_red_requests": vals.get("lts__t_requests_srcunit_tex_op_red.sum"),
            "l2_hit_rate_pct": vals.get("lts__t_sector_hit_rate.pct"),
            "how": "ncu --metrics dram__bytes_{read,write}.sum --clock-control none -k regex:mttkrp_sym -s 2 -c 1 "
                   "python tools/profile_one.py (cold L2: ncu flushes caches per replay), in this bench run"}


MIX_PAIRS = [(1, 1), (2, 2), (3, 3), (4, 4), (2, 1), (3, 1), (3, 2), (4, 3), (5, 2), (5, 3), (5, 4), (7, 3), (7, 4),
             (7, 5), (8, 3)]


def mix_shapes(gathers, reds):
    """The instantiated (ng, nr) pairs of tools/bounds.cu (bounds_mix_pairs)
    within 5 % of the ratio gathers / reds (at least the closest one): the
    mix is measured with each and its fastest rate is the bound — the rate
    the memory system reaches for this mix given enough operations in
    flight per unit."""
    if reds <= 0:
        return [(3, 0)]
    if gathers <= 0:
        return [(0, 2)]
    target = gathers / reds
    err = {p: abs(p[0] / p[1] - target) / target for p in MIX_PAIRS}
    best = min(err.values())
    return sorted((p for p in MIX_PAIRS if err[p] <= max(0.05, best + 1e-12)), key=lambda p: (err[p], p))


L2_TABLE_CAP = 48 << 20     # the L2 roofline: tables of at most 48 MB stay L2-resident (L2 126 MB)


def in_run_bounds(w, launch, st, nnz_local, dev_index=0):
    """The memory-system rates of this workload, measured on this GPU right
    now (tools/bounds.cu), for the L2 roofline: HBM stream read; random
    whole-row gathers from a table of B's footprint; red.global.add.v4.f32 of
    rows into a table of C's footprint (x the replicas the launch used); and
    the kernel's MIX of the two (its ratio of L2 gathers to reduced rows,
    reduced values depending on gathered ones).  Rows of R*4 bytes; tables
    capped at L2_TABLE_CAP (L2-resident) — where a footprint exceeds L2
    (c3), DRAM misses are the kernel's distance to this bound and the
    physical DRAM traffic is reported beside it."""
    import ctypes
    import __graft_entry__
    lib = ctypes.CDLL(__graft_entry__.build_bounds())
    for f in (lib.bounds_gather, lib.bounds_red):
        f.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.bounds_hbm_read.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.bounds_mix.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_double)]
    row = w.R * 4
    rb = min(512, 1 << max(4, (row - 1).bit_length()))   # the kernel's float4 row tile
    hbm, gat, red, mix = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    copies = max(1, launch.get("copies", 1))
    terms = memory_terms(w, st, nnz_local, launch)
    shapes = mix_shapes(terms["gather_rows"], terms["red_rows"])
    tb = min(w.dim * rb, L2_TABLE_CAP)
    tc = min(copies * w.dim * rb, L2_TABLE_CAP)
    mix_gbs = {}
    with ClockSampler(dev_index, period=0.01) as clk:
        rc = [lib.bounds_hbm_read(2 << 30, 5, ctypes.byref(hbm)),
              lib.bounds_gather(rb, tb, 5, ctypes.byref(gat)),
              lib.bounds_red(rb, tc, 5, ctypes.byref(red))]
        for ng, nr in shapes:
            rc.append(lib.bounds_mix(rb, tb, tc, ng, nr, 5, ctypes.byref(mix)))
            mix_gbs[f"{ng}g{nr}r"] = mix.value * (ng + nr) * rb / 1e9
    if any(rc):
        return {"unavailable": f"bounds library returned {rc}"}
    best = max(mix_gbs, key=mix_gbs.get)
    return {"hbm_read_gbs": hbm.value, "l2_gather_gbs": gat.value, "l2_red_gbs": red.value,
            "l2_mix_gbs": mix_gbs[best], "mix_shape": best, "mix_shapes_gbs": mix_gbs, "row_bytes": rb,
            "gather_table_bytes": tb, "red_table_bytes": tc,
            "clocks": clk.report(),
            "how": "tools/bounds.cu in this run: best of 5 launches each (148x8 blocks of 256 threads, >= 0.6 ms per launch), "
                   "2 GiB stream read; random whole-row float4 gathers / red.global.add.v4.f32 over tables of "
                   "the footprints (capped at 48 MB: L2-resident); the mix = ng gathers + nr reductions per "
                   "unit in the plan's ratio, reduced values from the gathered rows, fastest unit shape"}


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


def memory_terms(w, st, nnz_local, launch):
    """Bytes of each memory operation class of one launch, from the plan
    statistics (SURVEY.md §8(d) per-entry figures x the entries of the
    launch):
      stream   indices + value of every stored entry, read once;
      gather   the B rows the kernel must fetch past L1: one per distinct
               index of each entry (G), less the leading-index rows equal to
               the previous entry's (a leading run gathers its row once) and
               the position-1 rows equal to the previous entry's (c_1 runs);
               `gather_alg` is the north_star's algorithmic G rows;
      red      the C rows reduced: one per run-first position >= 1 of each
               entry (G - nnz), less the position-1 runs accumulated in
               registers when the launch did that, plus one row per
               leading-run fragment."""
    n, R = w.order, w.R
    row = R * 4
    n1 = sum(h for code, h in enumerate(st["pattern_hist"]) if not code & 1)   # entries with c1 != c0
    pos1 = launch.get("pos1", 0) == 1
    rep1 = n1 - min(n1, st["pos1_runs"])                                        # c1 equal to the previous entry's
    red_rows = st["lead_runs"] + (st["G"] - nnz_local) - (rep1 if pos1 else 0)
    gather_rows = st["G"] - (nnz_local - st["lead_runs"]) - rep1
    return {"stream": nnz_local * (4 * n + 4), "gather": gather_rows * row, "red": red_rows * row,
            "gather_alg": st["G"] * row, "gather_rows": gather_rows, "red_rows": red_rows}


def roofline(terms, bounds, kern_ms, local_bytes_eff, peak_hbm, traffic):
    """The kernel against the bound of the unit that binds it.  Each memory
    class at its measured rate gives a time — the stream alone, the gathers
    alone, the reductions alone, and the gathers and reductions together in
    the kernel's mix (they share the SM->L2 port and the L2); the largest is
    the bound.  achieved = that class's algorithmic bytes / kernel time,
    peak = its measured rate, frac = achieved / peak (= t_bound / t_kernel)."""
    t = kern_ms * 1e-3
    eff = {"effective_gbs": local_bytes_eff / t / 1e9, "frac_of_measured_copy_peak": local_bytes_eff / t / 1e9 / peak_hbm,
           "frac_of_8tbs": local_bytes_eff / t / 8e12, "algorithmic_bytes_per_launch": local_bytes_eff}
    phys = None
    if traffic and "dram_bytes_per_launch" in traffic:
        phys = traffic["dram_bytes_per_launch"] / t / 1e9
    if not bounds or "unavailable" in bounds:
        return {"bound": "hbm", "achieved": eff["effective_gbs"], "peak": peak_hbm, "unit": "GB/s",
                "frac": eff["effective_gbs"] / peak_hbm, "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "note": "in-run bounds unavailable: effective bytes against the HBM copy peak", "hbm": eff}
    rates = {"stream": bounds["hbm_read_gbs"], "gather": bounds["l2_gather_gbs"], "red": bounds["l2_red_gbs"],
             "mix": bounds["l2_mix_gbs"]}
    terms = dict(terms, mix=terms["gather"] + terms["red"])
    extra = {k: terms[k] for k in ("gather_alg", "gather_rows", "red_rows") if k in terms}
    times = {k: terms[k] / (rates[k] * 1e9) for k in rates}
    bind = max(times, key=times.get)
    achieved = terms[bind] / t / 1e9
    out = {"bound": "hbm" if bind == "stream" else "l2",
           "binding_op": {"stream": "index/value stream read (HBM)",
                          "gather": "random B-row gathers (L2)",
                          "red": "red.global.add.v4.f32 of C rows (SM->L2 request/write port, L2 atomic units)",
                          "mix": "the kernel's mix of random B-row gathers and red.v4 C-row reductions (SM->L2 "
                                 "request port / L2)"}[bind],
           "achieved": achieved, "peak": rates[bind], "unit": "GB/s", "frac": achieved / rates[bind],
           "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
           "algorithmic_bytes_per_launch": terms[bind], "kernel_ms": kern_ms, "t_bound_ms": times[bind] * 1e3,
           "terms_ms": {k: v * 1e3 for k, v in times.items()}, "terms_bytes": {k: terms[k] for k in rates},
           "counts": extra,
           "rates_gbs": rates, "peak_kind": "measured in this run on this GPU (tools/bounds.cu), clocks in bounds",
           "bounds": bounds,
           "hbm": dict(eff, physical_gbs=phys, physical_frac_of_copy_peak=(phys / peak_hbm) if phys else None)}
    return out


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
            "l2": ("not flushed (--warm)" if args.warm else
                   "flushed between timed steps (256 MiB write outside the events)"),
            "seed": w.meta.get("seed"),
            "parallelism": f"nnz-slices x{args.gpus} + {args.collective}(C)" if args.gpus > 1 else "1 GPU"}


def parse_opts(s):
    out = {}
    for kv in filter(None, s.split(",")):
        k, v = kv.split("=")
        out[k.strip()] = int(v)
    return out


def main():
    args = parse()
    from synth import generate
    w = generate(args.config, seed=args.seed)
    if args.impl == "reference":
        run_reference(args, w)
        return
    if args.cpu_baseline_only:
        print(json.dumps({"config": config_dict(w, args),
                          "cpu_baseline": cpu_baseline(w, threads=args.oracle_threads)}), flush=True)
        return

    import torch
    import paper_2406_09266_b200 as systec
    from paper_2406_09266_b200.shard import ShardedMTTKRP, shard_range

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
    sh = ShardedMTTKRP(w.order, w.dim, idx_d, vals_d, w.R, collective=args.collective)
    plan = sh.plan
    del idx_d, vals_d
    st = plan.stats()
    opts = parse_opts(args.opts)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step(ev=None):
        # one pass of the hot path: zero C (+ replicas) + MTTKRP kernel (+ replica sum),
        # then (N > 1) the exchange of the partial C's
        if ev:
            ev[0].record(stream)
        sh.compute(B_d, **opts)
        if ev:
            ev[1].record(stream)
        if dist is not None:
            sh.exchange()
        if ev:
            ev[2].record(stream)

    for _ in range(max(3, args.warmup)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    launch = plan.last_launch()
    # the memory-system bounds of this workload, measured on this GPU before the timed region
    bounds = None if args.no_bounds else in_run_bounds(w, launch, st, hi - lo, local)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            if not args.warm:
                flush.fill_(float(k))          # L2 flush between timed steps, outside the events
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
        sh.compute(B_d, **opts)
    e1.record(stream)
    torch.cuda.synchronize()
    warm_ms = e0.elapsed_time(e1) / 20

    # the paper's timing rule: minimum over up to 10,000 runs or
    # a time budget, each run L2-flushed and timed alone (kernel only, rank 0)
    paper_rule = None
    if rank == 0 and args.paper_rule_s > 0:
        runs, best, t_start = 0, float("inf"), time.perf_counter()
        while runs < 10_000 and time.perf_counter() - t_start < args.paper_rule_s:
            batch = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
            for a_, b_ in batch:
                flush.fill_(0.5)
                a_.record(stream)
                sh.compute(B_d, **opts)
                b_.record(stream)
            torch.cuda.synchronize()
            best = min(best, min(a_.elapsed_time(b_) for a_, b_ in batch))
            runs += len(batch)
        paper_rule = {"ms_min": best, "runs": runs, "rule": "min over up to 10,000 runs or the time budget "
                      f"({args.paper_rule_s} s), L2 flushed before each run (PAPER.md:740)",
                      "value_at_min": (hi - lo) / (best * 1e-3)}

    # the final C of the step (test mode): rank 0 writes it to disk
    if args.dump_c:
        out = sh.execute(B_d, **opts)
        if sh.collective == "reduce_scatter" and dist is not None:
            per = sh.C_rows.shape[0]
            full = torch.empty((per * world, w.R), dtype=torch.float32, device=dev)
            if args.dist_backend == "gloo":
                f_cpu = full.cpu()
                dist.all_gather_into_tensor(f_cpu, sh.C_rows.cpu())
                full.copy_(f_cpu)
            else:
                dist.all_gather_into_tensor(full, sh.C_rows)
            out = full[: w.dim]
        torch.cuda.synchronize()
        if rank == 0:
            np.save(args.dump_c, out.cpu().numpy())

    value = w.nnz / (ms_per_step * 1e-3)          # all ranks together process the whole tensor
    G_all = st["G"]
    if dist is not None:
        t = torch.tensor([G_all], device=dev, dtype=torch.float64)
        dist.all_reduce(t)
        G_all = int(t.item())
    # roofline of the dominant kernel (mttkrp_sym_kernel) on this rank's slice
    local_bytes = bytes_eff(w.order, hi - lo, st["G"], w.R, w.dim)
    peak, peak_kind = load_peaks()
    traffic = ncu_traffic(w.name, args.opts) if (rank == 0 and world == 1 and not args.no_ncu) else None

    line = None
    if rank == 0:
        terms = memory_terms(w, st, hi - lo, launch)
        rl = roofline(terms, bounds, kern_avg_ms, local_bytes, peak, traffic)
        rl.update(kernel="mttkrp_sym_kernel", kernel_ms=kern_avg_ms,
                  kernel_ms_includes="C zeroing + kernel (+ replica sum when C < 4 MB), CUDA events on the launch stream",
                  hbm_peak_kind=f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs = {peak})")
        if traffic is not None:
            rl["ncu"] = traffic
        be = bytes_eff(w.order, w.nnz, G_all, w.R, w.dim)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(w, args),
            "eff_gbs": be / (ms_per_step * 1e-3) / 1e9, "bytes_eff_per_step": be,
            "frac_of_8tbs": be / (ms_per_step * 1e-3) / 8e12,
            "roofline": rl,
            "timing": {"value": "whole-job nnz / mean step time over the K timed steps (driver contract)",
                       "step_ms_min": float(np.min(step_ms)), "step_ms_median": float(np.median(step_ms)),
                       "paper_rule": paper_rule},
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
        rows = sh.C_rows.shape[0] if sh.collective == "reduce_scatter" else w.dim
        pin_C = torch.empty((rows, w.R), dtype=torch.float32).pin_memory()

        def e2e_step():
            di = pin_idx.to(dev, non_blocking=True)
            dv = pin_vals.to(dev, non_blocking=True)
            dB = pin_B.to(dev, non_blocking=True)
            s2 = ShardedMTTKRP(w.order, w.dim, di, dv, w.R, collective=args.collective)
            out = s2.execute(dB)
            pin_C[: out.shape[0]].copy_(out, non_blocking=True)
            torch.cuda.synchronize()
            s2.destroy()

        e2e_step()
        ts = []
        for _ in range(args.e2e_steps):
            dist.barrier()
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            e2e_step()
            b_.record(stream)
            b_.synchronize()
            ts.append(a_.elapsed_time(b_))
        t = torch.tensor([float(np.mean(ts))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            e2e_ms = t.item()
            line["e2e"] = {"value": w.nnz / (e2e_ms * 1e-3), "unit": UNIT,
                           "h2d_bytes_per_step": (w.idx.nbytes + w.vals.nbytes) + world * w.B.nbytes,
                           "d2h_bytes_per_step": world * pin_C.numel() * 4, "ms_per_step": e2e_ms,
                           "includes": f"per rank: H2D slice + B, plan creation + execute + {args.collective}(C) "
                                       "+ D2H of the rank's result; CUDA events, max over ranks"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, threads=args.oracle_threads)
    if rank == 0:
        print(json.dumps(line), flush=True)
    sh.destroy()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
