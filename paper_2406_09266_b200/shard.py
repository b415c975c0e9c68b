"""Multi-GPU sharding of the symmetric MTTKRP: stored entries
are independent, so the sorted stream splits into contiguous nnz-balanced
slices, one per rank; each rank's partial C is summed with one all-reduce.
Host logic only (the compute is the C ABI call on each rank's slice)."""
from __future__ import annotations


def shard_range(nnz: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the sorted stream owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or nnz < 0:
        raise ValueError("bad shard request")
    return nnz * rank // world, nnz * (rank + 1) // world


def reduce_partials(C, group=None):
    """Sum the per-rank partial outputs in place (one all-reduce of dim x R)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(C, op=dist.ReduceOp.SUM, group=group)
    return C
