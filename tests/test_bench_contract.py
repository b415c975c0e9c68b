"""bench.py keeps the driver contract: one JSON line with the required keys.
The reference arm runs on CPU; the GPU arm (1 and 2 ranks) needs a B200.
The 2-rank runs also dump the final C of the step and compare every element
with the oracle (the N > 1 CUDA path: slicing, per-rank plans, collective)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "e2e"]


def run(args, env=None, timeout=900):
    out = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                         env=dict(os.environ, **(env or {})))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run(["bench.py", "--impl", "reference", "--config", "c1", "--steps", "3", "--warmup", "1"])
    for k in REQUIRED + ["impl", "cpu_baseline"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_gpu_arm_line_one_rank():
    d = run(["bench.py", "--config", "c1", "--steps", "5", "--warmup", "3", "--e2e-steps", "2",
             "--paper-rule-s", "0.5"])
    for k in REQUIRED + ["roofline", "cpu_baseline", "clocks", "gpu_launches", "timing"]:
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] in ("hbm", "l2") and r["achieved"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert "unavailable" not in r["bounds"] and r["bounds"]["clocks"]["samples"] >= 0
    assert r["hbm"]["effective_gbs"] > 0
    assert d["gpu_launches"] >= d["steps"] and d["n_gpus"] == 1
    assert d["timing"]["paper_rule"]["runs"] >= 100


@pytest.mark.gpu
@pytest.mark.parametrize("config,collective,port", [("c1", "all_reduce", 29541), ("c1", "reduce_scatter", 29542),
                                                    ("c2", "all_reduce", 29543), ("c2", "reduce_scatter", 29544)])
def test_gpu_arm_two_ranks_gloo_same_device(tmp_path, config, collective, port):
    """bench.py's N = 2 path on one GPU (gloo, every rank on cuda:0; no kernel
    waits on another): the final C of a step equals the oracle everywhere."""
    import oracle
    from synth import generate

    from gpu_util import parity
    dump = str(tmp_path / "C.npy")
    d = run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
             "--master-port", str(port), "bench.py", "--gpus", "2", "--config", config, "--steps", "3",
             "--warmup", "3", "--dist-backend", "gloo", "--same-device", "--e2e-steps", "1",
             "--collective", collective, "--dump-c", dump, "--no-bounds"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "e2e" in d and collective in d["config"]["parallelism"]
    w = generate(config)
    Cref, S = oracle.mttkrp(w.order, w.dim, w.idx, w.vals, w.B)
    err = parity(np.load(dump), Cref, S)
    print(f"{config} 2 ranks {collective}: all {Cref.size} elements max_rel_err={err:.3e}")
