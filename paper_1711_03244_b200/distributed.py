"""Photon-split multi-GPU plumbing (one process per GPU, torch.distributed).

MC shards naturally by photon: rank r simulates the contiguous global range
the reference's run_multi_device would give device r (scheduler.cpp:405-413,
partition by S1/S2/S3), all ranks share the quantum of the global count
(run_config.photon_count = total, scheduler.cpp:412-413), and the exchange
steps are
  * the sum of the int64 fluence maps and disposition quanta onto rank 0 (the
    merge at scheduler.cpp:444) — an NCCL reduce over NVLink on B200s (gloo in
    the CPU tests);
  * the detector records: each rank sorts its own records by photon index on
    the device, the per-rank counts are all-gathered, and the records are sent
    to rank 0 and concatenated in rank order. Ranges ascend with the rank, so
    the result is globally sorted.
Integer sums and the sorted gather make the merged map and the record list
bit-identical for any GPU count.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass
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


def _world():
    import torch.distributed as dist
    if dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


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


def gather_records(recs, n: int, rec_bytes: int, out=None, dst: int = 0):
    """Concatenate every rank's first n sorted records (uint8 tensor, n *
    rec_bytes bytes) on rank `dst` in rank order. Returns (records tensor on
    dst or None elsewhere, per-rank counts). NCCL moves device buffers
    point to point; gloo stages through host memory."""
    import torch
    import torch.distributed as dist
    rank, world = _world()
    dev = recs.device
    if world == 1:
        return (recs[: n * rec_bytes] if out is None else out[: n * rec_bytes].copy_(recs[: n * rec_bytes])), [n]
    gloo = dist.get_backend() == "gloo"
    cnt = torch.tensor([n], dtype=torch.int64, device="cpu" if gloo else dev)
    allc = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(allc, cnt)
    counts = [int(c.item()) for c in allc]
    total = sum(counts)
    if rank == dst:
        buf = out if out is not None else torch.empty(max(1, total * rec_bytes), dtype=torch.uint8, device=dev)
        off = 0
        ops = []
        staged = []
        for r, c in enumerate(counts):
            nb = c * rec_bytes
            if r == dst:
                buf[off:off + nb].copy_(recs[:nb])
            elif nb:
                if gloo:
                    t = torch.empty(nb, dtype=torch.uint8)
                    staged.append((t, off, nb))
                    ops.append(dist.P2POp(dist.irecv, t, r))
                else:
                    ops.append(dist.P2POp(dist.irecv, buf[off:off + nb], r))
            off += nb
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for t, o, nb in staged:
            buf[o:o + nb].copy_(t.to(dev))
        return buf[: total * rec_bytes], counts
    nb = n * rec_bytes
    if nb:
        src = recs[:nb].cpu() if gloo else recs[:nb]
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, src, dst)]):
            w.wait()
    return None, counts


@dataclass
class DistributedResult:
    """Rank 0: merged map (host int64, [ngates*V]), disposition quanta, detector
    records (numpy structured array, sorted by photon index) and the total
    record count. Other ranks: all None."""
    cells: Optional[object] = None
    totals_q: Optional[List[int]] = None
    detections: Optional[object] = None
    det_count: Optional[int] = None


def run_group_distributed(scene, config, total: Optional[int] = None, strategy: Strategy = Strategy.S1,
                          profiles=None, device: Optional[int] = None, cells_out=None,
                          det_out=None) -> DistributedResult:
    """One process per GPU: this rank's contiguous share of photons [0, total)
    (default config.photon_count) through the C-ABI plan (scene upload,
    transport into device buffers, on-device record sort), the NCCL reduce of
    the int64 map and disposition quanta onto rank 0, the detector-record
    gather, and on rank 0 the download of the merged map into `cells_out`
    (e.g. a pinned host array) and of the records into `det_out`. The
    multi-process form of run_multi_device (scheduler.cpp:395-451); every rank
    uses the quantum of `total` (scheduler.cpp:412-413)."""
    import numpy as np
    import torch

    from . import _abi
    from .runtime import Plan

    rank, world = _world()
    total = config.photon_count if total is None else total
    cfg = copy.copy(config)
    cfg.photon_count = total  # shared quantum of the global count
    dev = torch.cuda.current_device() if device is None else device
    first, count = rank_ranges(total, world, strategy, profiles)[rank]
    plan = Plan(scene, cfg, dev)
    try:
        cells = torch.empty(plan.ncells, dtype=torch.int64, device=f"cuda:{dev}")
        totals = torch.empty(4, dtype=torch.int64, device=f"cuda:{dev}")
        det = det_n = None
        if cfg.detectors:
            det = torch.empty(max(1, cfg.det_capacity) * plan.rec_bytes, dtype=torch.uint8, device=f"cuda:{dev}")
            det_n = torch.empty(1, dtype=torch.int64, device=f"cuda:{dev}")
        plan.run_torch(first, count, cells, totals, det, det_n, zero=True)
        reduce_to_root(cells, totals)
        recs = None
        n_all = 0
        if det is not None:
            n_found = int(det_n.item())
            n = min(n_found, cfg.det_capacity)
            srt = torch.empty_like(det)
            plan.sort_records_torch(det, n, first, count, srt)
            recs, counts = gather_records(srt, n, plan.rec_bytes)
            allf = [n_found]
            import torch.distributed as dist
            if world > 1:
                gloo = dist.get_backend() == "gloo"
                t = torch.tensor([n_found], dtype=torch.int64, device="cpu" if gloo else f"cuda:{dev}")
                lst = [torch.zeros_like(t) for _ in range(world)]
                dist.all_gather(lst, t)
                allf = [int(x.item()) for x in lst]
            n_all = sum(allf)
        if rank != 0:
            torch.cuda.synchronize(dev)
            return DistributedResult()
        if cells_out is None:
            cells_out = np.empty(plan.ncells, np.int64)
        torch.from_numpy(cells_out.reshape(-1)).copy_(cells)
        dets = None
        if recs is not None:
            dt = _abi.det_record_dtype(plan.nmedia)
            nrec = recs.numel() // plan.rec_bytes if n_all else 0
            if det_out is None:
                det_out = np.empty(max(1, nrec), dt)
            keep = min(nrec, len(det_out))
            if keep:
                torch.from_numpy(det_out.view(np.uint8).reshape(-1)[: keep * plan.rec_bytes]).copy_(
                    recs[: keep * plan.rec_bytes])
            dets = det_out[:keep]
        return DistributedResult(cells_out, totals.cpu().tolist(), dets, n_all if cfg.detectors else None)
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
