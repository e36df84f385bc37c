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


def run_group_distributed(scene, config, total: Optional[int] = None, strategy: Strategy = Strategy.S1,
                          profiles=None, device: Optional[int] = None, cells_out=None):
    """One process per GPU: this rank's contiguous share of photons [0, total)
    (default config.photon_count) through the C-ABI plan (scene upload,
    transport into device buffers), the NCCL reduce of the int64 map and
    disposition quanta onto rank 0, and on rank 0 the download of the merged
    map into `cells_out` (e.g. a pinned host array of shape
    (ngates, nz, ny, nx)). The multi-process form of run_multi_device
    (scheduler.cpp:395-451). Returns (cells_host or None, totals_q list or
    None) on rank 0 and (None, None) elsewhere."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from .runtime import Plan

    rank = dist.get_rank() if dist.is_initialized() else 0
    world = dist.get_world_size() if dist.is_initialized() else 1
    total = config.photon_count if total is None else total
    dev = torch.cuda.current_device() if device is None else device
    first, count = rank_ranges(total, world, strategy, profiles)[rank]
    plan = Plan(scene, config, dev)
    try:
        cells = torch.empty(plan.ncells, dtype=torch.int64, device=f"cuda:{dev}")
        totals = torch.empty(4, dtype=torch.int64, device=f"cuda:{dev}")
        det = det_n = None
        if config.detectors:
            det = torch.empty(max(1, config.det_capacity) * plan.rec_bytes, dtype=torch.uint8, device=f"cuda:{dev}")
            det_n = torch.empty(1, dtype=torch.int64, device=f"cuda:{dev}")
        plan.run_torch(first, count, cells, totals, det, det_n, zero=True)
        reduce_to_root(cells, totals)
        if rank != 0:
            torch.cuda.synchronize(dev)
            return None, None
        if cells_out is None:
            cells_out = np.empty(plan.ncells, np.int64)
        torch.from_numpy(cells_out.reshape(-1)).copy_(cells)
        return cells_out, totals.cpu().tolist()
    finally:
        plan.close()


def run_sharded(total: int, compute: Callable[[int, int], tuple], rank: int, world: int,
                strategy: Strategy = Strategy.S1, profiles=None):
    """compute(first, count) -> (cells int64 tensor, totals int64[4] tensor) on
    this rank's device; returns the reduced pair (valid on rank 0)."""
    first, count = rank_ranges(total, world, strategy, profiles)[rank]
    cells, totals = compute(first, count)
    reduce_to_root(cells, totals)
    return cells, totals
