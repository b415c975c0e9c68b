"""World-size-2 tests of the multi-GPU path (SURVEY.md §8(e),
paper_2406_09266_b200/shard.py).

CPU (gloo): the host logic — slices of the sorted stream, the row blocks of
a reduce-scatter, and both collectives — with the oracle computing each
rank's partial (the compute on a GPU box is the per-rank CUDA plan).

GPU (gloo, both ranks on cuda:0 — no kernel waits on another): the real N>1
CUDA path, ShardedMTTKRP on each rank's slice with the CUDA plan, both
collectives, every element of the result against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_09266_b200.shard import (reduce_partials, reduce_scatter_partials, row_range, rows_per_rank,
                                         shard_range)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _cpu_worker(rank, world, port, out, dim):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from synth import small_random
    w = small_random(4, dim, 3001, 6, seed=7, diag_frac=0.3)
    lo, hi = shard_range(w.nnz, rank, world)
    C, S = oracle.mttkrp(4, dim, w.idx[lo:hi], w.vals[lo:hi], w.B, threads=1)
    # all-reduce: every rank holds the whole C
    Ct, St = reduce_partials(torch.from_numpy(C.copy())), reduce_partials(torch.from_numpy(S.copy()))
    # reduce-scatter: rank holds rows row_range(rank) of C
    per = rows_per_rank(dim, world)
    Cpad = torch.zeros((per * world, 6), dtype=torch.float64)
    Cpad[:dim] = torch.from_numpy(C)
    block = reduce_scatter_partials(Cpad, torch.empty((per, 6), dtype=torch.float64))
    r0, r1 = row_range(dim, rank, world)
    blocks = [torch.empty((per, 6), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(blocks, block)
    if rank == 0:
        Cf, Sf = oracle.mttkrp(4, dim, w.idx, w.vals, w.B, threads=1)
        den = np.where(Sf > 0, Sf, 1)
        err_ar = float(np.max(np.abs(Ct.numpy() - Cf) / den))
        full = torch.cat(blocks)[:dim].numpy()
        err_rs = float(np.max(np.abs(full - Cf) / den))
        out.put((err_ar, float(np.max(np.abs(St.numpy() - Sf))), err_rs, (r0, r1)))
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


def test_row_range_covers_exactly():
    for dim in (1, 5, 64, 100_000, 1_000_001):
        for world in (1, 2, 3, 8):
            parts = [row_range(dim, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == dim
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert all(h - l <= rows_per_rank(dim, world) for l, h in parts)


@pytest.mark.parametrize("dim", [20, 21])     # 21: world does not divide dim (padded last block)
def test_two_rank_gloo_partials_sum_to_full(dim):
    err_ar, serr, err_rs, rr = _spawn(_cpu_worker, 2, dim)
    assert err_ar < 1e-13 and serr < 1e-9 and err_rs < 1e-13
    assert rr == (0, (dim + 1) // 2)


def _gpu_worker(rank, world, port, out, config, collective):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2406_09266_b200.shard import ShardedMTTKRP
    from synth import generate, small_random
    w = generate(config) if config.startswith("c") else small_random(5, 40, 200_003, 16, seed=11, diag_frac=0.1)
    lo, hi = shard_range(w.nnz, rank, world)
    sh = ShardedMTTKRP(w.order, w.dim, torch.from_numpy(w.idx[lo:hi]).cuda(),
                       torch.from_numpy(w.vals[lo:hi]).cuda(), w.R, collective=collective)
    B = torch.from_numpy(w.B).cuda()
    res = sh.execute(B)
    for _ in range(2):        # repeated executes: C is re-zeroed inside, the padding stays zero
        res = sh.execute(B)
    torch.cuda.synchronize()
    blocks = [torch.empty_like(res.cpu()) for _ in range(world)] if collective == "all_reduce" else \
        [torch.empty((sh.C_rows.shape[0], w.R)) for _ in range(world)]
    mine = res.cpu() if collective == "all_reduce" else sh.C_rows.cpu()
    dist.all_gather(blocks, mine)
    if rank == 0:
        out.put((blocks[0].numpy() if collective == "all_reduce" else torch.cat(blocks)[: w.dim].numpy(),
                 [b.numpy() for b in blocks] if collective == "all_reduce" else None))
    dist.barrier()
    sh.destroy()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c1", "small5"])
@pytest.mark.parametrize("collective", ["all_reduce", "reduce_scatter"])
def test_two_rank_cuda_path_matches_oracle(config, collective):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import oracle
    from synth import generate, small_random

    from gpu_util import parity
    C, all_blocks = _spawn(_gpu_worker, 2, config, collective)
    w = generate(config) if config.startswith("c") else small_random(5, 40, 200_003, 16, seed=11, diag_frac=0.1)
    Cref, S = oracle.mttkrp(w.order, w.dim, w.idx, w.vals, w.B)
    err = parity(C, Cref, S)
    if all_blocks is not None:     # every rank holds the same whole C after the all-reduce
        assert all(np.array_equal(b, all_blocks[0]) for b in all_blocks)
    print(f"{config} 2 ranks {collective}: max_rel_err={err:.3e}")
