"""Multi-GPU symmetric MTTKRP: one process per GPU.

Stored entries are independent units, so the sorted canonical stream splits
into contiguous nnz-balanced slices, one per rank (a leading run cut by a
slice boundary becomes two run fragments, which the kernel handles like any
unit boundary).  Each rank builds a plan over its slice and computes a full
partial ``C_g`` [dim][R] with the CUDA kernel; the exchange step is one
collective over the ``dim x R`` partials:

* ``"all_reduce"`` — every rank ends with the whole C (the a7 hand-off of the
  single-GPU path: C [dim][R] on every rank);
* ``"reduce_scatter"`` — rank g ends with rows ``row_range(dim, g, world)`` of
  C only, half the traffic of the all-reduce; the form a row-sharded consumer
  such as a distributed CP-ALS row update wants.

The paper names "a distributed decomposition" with atomics as its future
parallelisation.  Pushing per-entry updates to the owner of a
C row over NVLink would move the ~2.5 GB of reduction payload of c2 instead of
one 12.8 MB C, so the collective stays one NCCL call after the kernel
(DESIGN.md §11).  Everything here is host-side plumbing: the compute is the C
ABI plan on each rank's slice, the collective is torch.distributed (NCCL on
GPUs; gloo only for code-path tests).
"""
from __future__ import annotations

COLLECTIVES = ("all_reduce", "reduce_scatter")


def shard_range(nnz: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the sorted stream owned by ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or nnz < 0:
        raise ValueError("bad shard request")
    return nnz * rank // world, nnz * (rank + 1) // world


def rows_per_rank(dim: int, world: int) -> int:
    """Rows of C each rank holds after a reduce-scatter (C is padded to
    ``world * rows_per_rank`` rows so every rank's block has the same size,
    as the collective requires)."""
    if world < 1 or dim < 0:
        raise ValueError("bad shard request")
    return -(-dim // world)


def row_range(dim: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the C rows rank ``rank`` owns after a reduce-scatter
    (the last ranks may own fewer rows, or none, when world does not divide dim)."""
    if not 0 <= rank < world:
        raise ValueError("bad shard request")
    per = rows_per_rank(dim, world)
    return min(dim, rank * per), min(dim, (rank + 1) * per)


def _world(group=None) -> int:
    import torch.distributed as dist
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def _rank(group=None) -> int:
    import torch.distributed as dist
    return dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0


def reduce_partials(C, group=None):
    """Sum the per-rank partial outputs in place (one all-reduce of dim x R)."""
    import torch.distributed as dist
    if _world(group) > 1:
        dist.all_reduce(C, op=dist.ReduceOp.SUM, group=group)
    return C


def reduce_scatter_partials(C_padded, out, group=None):
    """out[rows_per][R] = rows ``row_range(rank)`` of the sum over ranks of
    ``C_padded`` [world * rows_per][R].  With the gloo backend (code-path
    tests only) CUDA tensors are staged through host memory."""
    import torch.distributed as dist
    if _world(group) == 1:
        out.copy_(C_padded[: out.shape[0]])
        return out
    if C_padded.is_cuda and dist.get_backend(group) == "gloo":
        o = out.cpu()
        dist.reduce_scatter_tensor(o, C_padded.cpu(), op=dist.ReduceOp.SUM, group=group)
        out.copy_(o)
        return out
    dist.reduce_scatter_tensor(out, C_padded, op=dist.ReduceOp.SUM, group=group)
    return out


class ShardedMTTKRP:
    """This rank's part of a multi-GPU symmetric MTTKRP.

    ``idx``/``vals`` are this rank's slice of the stored entries (CUDA tensors,
    e.g. ``shard_range`` of the sorted stream; any slicing is correct, the
    contiguous one keeps runs whole).  ``execute(B)`` runs the kernel on the
    slice (zeroing C inside, as the single-GPU execute) and the collective,
    and returns the whole C (``all_reduce``) or this rank's row block
    (``reduce_scatter``; rows ``self.rows``)."""

    def __init__(self, order: int, dim: int, idx, vals, R: int, collective: str = "all_reduce", group=None,
                 **plan_opts):
        import torch

        from .systec import Plan
        if collective not in COLLECTIVES:
            raise ValueError(f"collective must be one of {COLLECTIVES}")
        self.order, self.dim, self.R = order, dim, R
        self.collective, self.group = collective, group
        self.world, self.rank = _world(group), _rank(group)
        self.plan = Plan(order, dim, idx, vals, **plan_opts)
        dev = idx.device
        per = rows_per_rank(dim, self.world)
        # padded partial: rows [dim, world*per) stay zero (the kernel writes rows < dim)
        self._C_pad = torch.zeros((per * self.world if collective == "reduce_scatter" else dim, R),
                                  dtype=torch.float32, device=dev)
        self.C = self._C_pad[:dim]
        self.rows = row_range(dim, self.rank, self.world)
        self.C_rows = torch.empty((per, R), dtype=torch.float32, device=dev) if collective == "reduce_scatter" \
            else None

    def compute(self, B, **exec_opts):
        """The kernel only: this rank's partial C (no exchange)."""
        self.plan.execute(B, self.C, **exec_opts)
        return self.C

    def exchange(self):
        """The collective: returns the whole C or this rank's row block."""
        if self.collective == "all_reduce":
            return reduce_partials(self.C, self.group)
        reduce_scatter_partials(self._C_pad, self.C_rows, self.group)
        return self.C_rows[: self.rows[1] - self.rows[0]]

    def execute(self, B, **exec_opts):
        self.compute(B, **exec_opts)
        return self.exchange()

    def stats(self):
        return self.plan.stats()

    def last_launch(self):
        return self.plan.last_launch()

    def destroy(self):
        self.plan.destroy()
