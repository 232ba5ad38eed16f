"""Sharded fit across GPUs: one process per GPU, one exchange step.

The reference's only parallelism is contiguous chunks with an ascending
element-wise combine (proj/src/power_sums.cpp:61-87). Across GPUs the same
contract becomes:

1. rank g owns points ``[n*g//G, n*(g+1)//G)`` (the chunk formula of
   power_sums.cpp:69-70);
2. the fused kernel reduces its shard to 3m+1 double-double partials
   (an ``lsqfit_result`` record, written on the GPU);
3. ONE collective: an all-gather of the G records (1016 B each) over NCCL /
   NVLink — the records, not a reduction, so every rank then combines them
   in the same ascending rank order and all ranks hold bit-identical sums
   regardless of NCCL's algorithm choice;
4. ``combine_device`` folds them (double-double), checks finiteness and runs
   the one-warp solve redundantly on every rank.

The host logic here is backend-agnostic (``partial_fn`` / ``combine_fn``), so
the CPU tests drive it with ``gloo`` and the oracle standing in for the
device kernels; the product wiring (``gpu_fit_sharded``) uses the CUDA path.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from . import _capi


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard of rank ``rank``: [n*g/G, n*(g+1)/G) (power_sums.cpp:69-70)."""
    return n * rank // world, n * (rank + 1) // world


def all_gather_records(record: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather one uint8 record per rank into a [world * bytes] tensor (rank order)."""
    world = dist.get_world_size(group)
    if record.is_cuda and dist.get_backend(group) != "nccl":
        # gloo (tests, shared-GPU emulation): stage the 1 KB records through the host
        return all_gather_records(record.cpu(), group).to(record.device)
    out = torch.empty(world * record.numel(), dtype=record.dtype, device=record.device)
    dist.all_gather_into_tensor(out, record, group=group)
    return out


def fit_sharded(partial_fn: Callable[[int, int], torch.Tensor],
                combine_fn: Callable[[torch.Tensor, int], torch.Tensor],
                n: int, group=None) -> torch.Tensor:
    """Generic sharded fit: partial over this rank's shard, gather, combine."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_bounds(n, rank, world)
    rec = partial_fn(lo, hi)
    gathered = all_gather_records(rec, group)
    return combine_fn(gathered, world)


def gpu_fit_sharded(xy_shard: torch.Tensor, degree: int, flags: int = _capi.SOLVE, group=None,
                    part: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Product path: ``xy_shard`` is this rank's resident shard (CUDA float64 (k, 2)).

    Kernel launches and the NCCL all-gather are all enqueued on the current
    stream; nothing synchronises with the host.
    """
    from . import device as D
    part = D.fit(xy_shard, degree, flags=_capi.SUMS, out=part)
    gathered = all_gather_records(part, group)
    return D.combine(gathered, dist.get_world_size(group), degree, flags=flags, out=out)
