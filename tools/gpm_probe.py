"""Probe: can NVML GPM (GPU performance monitoring) give the physical DRAM
bandwidth of a kernel loop inside a normal (non-profiled) run?

Calibrates DRAM_BW_UTIL with a torch copy of known bytes, then reads it over
back-to-back executes of a config.  Prints JSON lines.

    python tools/gpm_probe.py --config c2
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gpm_window(nv, h, fn, min_s=0.5):
    s1, s2 = nv.nvmlGpmSampleAlloc(), nv.nvmlGpmSampleAlloc()
    import torch
    torch.cuda.synchronize()
    nv.nvmlGpmSampleGet(h, s1)
    t0 = time.perf_counter()
    n = 0
    while True:
        fn()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
            if time.perf_counter() - t0 >= min_s:
                break
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    nv.nvmlGpmSampleGet(h, s2)
    mg = nv.c_nvmlGpmMetricsGet_t()
    mg.version = nv.NVML_GPM_METRICS_GET_VERSION
    ids = [nv.NVML_GPM_METRIC_DRAM_BW_UTIL, nv.NVML_GPM_METRIC_SM_UTIL, nv.NVML_GPM_METRIC_SM_OCCUPANCY]
    mg.numMetrics = len(ids)
    mg.sample1, mg.sample2 = s1, s2
    for i, m in enumerate(ids):
        mg.metrics[i].metricId = m
    nv.nvmlGpmMetricsGet(mg)
    vals = [mg.metrics[i].value for i in range(len(ids))]
    nv.nvmlGpmSampleFree(s1)
    nv.nvmlGpmSampleFree(s2)
    return {"dram_bw_util_pct": vals[0], "sm_util_pct": vals[1], "sm_occ_pct": vals[2], "calls": n, "wall_s": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2")
    a = ap.parse_args()
    import pynvml as nv
    import torch

    import paper_2406_09266_b200 as systec
    from synth import generate
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    sup = nv.c_nvmlGpmSupport_t()
    sup.version = 1
    try:
        nv.nvmlGpmQueryDeviceSupport(h, sup)
        print(json.dumps({"gpm_supported": int(sup.isSupportedDevice)}), flush=True)
    except Exception as e:
        print(json.dumps({"gpm_supported": 0, "err": repr(e)}), flush=True)
    src = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    dst = torch.empty_like(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        dst.copy_(src)
    e0.record()
    for _ in range(20):
        dst.copy_(src)
    e1.record()
    torch.cuda.synchronize()
    copy_gbs = 20 * 2 * src.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    r = gpm_window(nv, h, lambda: dst.copy_(src))
    r.update(what="copy 1 GiB", copy_gbs_events=copy_gbs)
    print(json.dumps(r), flush=True)
    idle = gpm_window(nv, h, lambda: time.sleep(0.01))
    idle["what"] = "idle"
    print(json.dumps(idle), flush=True)
    for cfg in a.configs.split(","):
        w = generate(cfg)
        plan = systec.Plan(w.order, w.dim, torch.from_numpy(w.idx).cuda(), torch.from_numpy(w.vals).cuda())
        B = torch.from_numpy(w.B).cuda()
        C = torch.empty((w.dim, w.R), device="cuda")
        for _ in range(5):
            plan.execute(B, C)
        e0.record()
        for _ in range(100):
            plan.execute(B, C)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 100
        g = gpm_window(nv, h, lambda: plan.execute(B, C), min_s=1.0)
        util = g["dram_bw_util_pct"] / r["dram_bw_util_pct"]
        g.update(what=f"{cfg} execute back-to-back", exec_ms=ms,
                 dram_gbs_est=util * copy_gbs,
                 dram_bytes_per_launch_est=util * copy_gbs * 1e9 * ms * 1e-3)
        print(json.dumps(g), flush=True)
        plan.destroy()


if __name__ == "__main__":
    main()
