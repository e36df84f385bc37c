"""Photon-split multi-GPU plumbing (one process per GPU, torch.distributed).

MC shards naturally by photon: rank r simulates the contiguous global range
the reference's run_multi_device would give device r (scheduler.cpp:405-413,
partition by S1/S2/S3), all ranks share the quantum of the global count, and
the only exchange step is the sum of the int64 fluence maps and disposition
quanta onto rank 0 (the merge at scheduler.cpp:444) — an NCCL reduce over
NVLink on B200s (gloo in the CPU tests). Integer sums make the merged map
bit-identical for any GPU count.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

from .runtime import DeviceProfile, Strategy, make_partition


def rank_ranges(total: int, world: int, strategy: Strategy = Strategy.S1,
                profiles: Optional[Sequence[DeviceProfile]] = None) -> List[Tuple[int, int]]:
    """[(first, count)] per rank, contiguous in rank order."""
    devs = list(profiles) if profiles else [DeviceProfile(name=f"gpu{i}", cores=1, a=1.0, gpu=i)
                                            for i in range(world)]
    if len(devs) != world:
        raise ValueError("one profile per rank")
    counts = make_partition(total, devs, strategy).counts
    out, first = [], 0
    for c in counts:
        out.append((first, c))
        first += c
    return out


def reduce_to_root(cells, totals, dst: int = 0) -> None:
    """Sum int64 maps and disposition quanta onto `dst` (in place). NCCL: one
    reduce each (NVLink); gloo with CUDA tensors (plumbing tests, ranks sharing
    a GPU) has no device reduce, so it all-reduces instead."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend() == "gloo" and cells.is_cuda:
            dist.all_reduce(cells, op=dist.ReduceOp.SUM)
            dist.all_reduce(totals, op=dist.ReduceOp.SUM)
        else:
            dist.reduce(cells, dst=dst, op=dist.ReduceOp.SUM)
            dist.reduce(totals, dst=dst, op=dist.ReduceOp.SUM)


def run_sharded(total: int, compute: Callable[[int, int], tuple], rank: int, world: int,
                strategy: Strategy = Strategy.S1, profiles=None):
    """compute(first, count) -> (cells int64 tensor, totals int64[4] tensor) on
    this rank's device; returns the reduced pair (valid on rank 0)."""
    first, count = rank_ranges(total, world, strategy, profiles)[rank]
    cells, totals = compute(first, count)
    reduce_to_root(cells, totals)
    return cells, totals
