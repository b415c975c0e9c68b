"""World-size-2 gloo test of the multi-GPU path's host logic on CPU: each rank
takes its slice of the sorted stream, computes a partial C (the oracle stands
in for the per-rank device call), and one all-reduce gives the full result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_09266_b200.shard import reduce_partials, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from synth import small_random
    w = small_random(4, 20, 3001, 6, seed=7, diag_frac=0.3)
    lo, hi = shard_range(w.nnz, rank, world)
    C, S = oracle.mttkrp(4, 20, w.idx[lo:hi], w.vals[lo:hi], w.B, threads=1)
    Ct = torch.from_numpy(C)
    St = torch.from_numpy(S)
    reduce_partials(Ct)
    reduce_partials(St)
    if rank == 0:
        Cf, Sf = oracle.mttkrp(4, 20, w.idx, w.vals, w.B, threads=1)
        err = float(np.max(np.abs(Ct.numpy() - Cf) / np.where(Sf > 0, Sf, 1)))
        out.put((err, float(np.max(np.abs(St.numpy() - Sf)))))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_exactly():
    for nnz in (0, 1, 7, 1000, 10_000_001):
        for world in (1, 2, 3, 8):
            parts = [shard_range(nnz, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == nnz
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gloo_partials_sum_to_full():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, serr = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-13 and serr < 1e-9
