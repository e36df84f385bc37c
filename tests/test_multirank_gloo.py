"""The N>1 path on CPU: world_size-2 gloo run of the sharding + reduce plumbing
(paper_1711_03244_b200/distributed.py, also used by bench.py). The per-rank
compute here is the oracle (test stand-in for the GPU kernel); the test checks
that contiguous per-rank ranges + the int64 reduce reproduce the single-process
map bit for bit (reference contract test_scheduler.cpp:246-264)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 6_000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, strategy, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_1711_03244_b200 as v
    from paper_1711_03244_b200.distributed import run_sharded
    st = v.baseline_setup("b1", photons=N, seed=11)
    C = oracle.corc()

    def compute(first, count):
        out = C.walk(st.scene, st.config, first, count, threads=2)
        q = v.quantum_for(N)
        tq = [int(round(x / q)) for x in out["disp"]]
        return torch.from_numpy(out["cells"].copy()), torch.tensor(tq, dtype=torch.int64)

    profiles = [v.DeviceProfile(cores=1 + r, a=1e-3 * (1 + r), t0=r) for r in range(world)]
    cells, totals = run_sharded(N, compute, rank, world, v.Strategy(strategy), profiles)
    if rank == 0:
        np.save(out_path, cells.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("strategy", [1, 3])
def test_two_rank_shard_and_reduce(tmp_path, strategy):
    import oracle
    import paper_1711_03244_b200 as v
    out = str(tmp_path / "cells.npy")
    mp.spawn(_worker, args=(2, _free_port(), strategy, out), nprocs=2, join=True)
    got = np.load(out)
    st = v.baseline_setup("b1", photons=N, seed=11)
    whole = oracle.corc().walk(st.scene, st.config, 0, N, threads=4)["cells"]
    assert np.array_equal(got, whole)


def test_rank_ranges_contiguous():
    import paper_1711_03244_b200 as v
    from paper_1711_03244_b200.distributed import rank_ranges
    for world in (1, 2, 3, 8):
        r = rank_ranges(10**9 + 7, world)
        assert r[0][0] == 0
        assert sum(c for _, c in r) == 10**9 + 7
        for (f0, c0), (f1, _) in zip(r, r[1:]):
            assert f0 + c0 == f1
        assert max(c for _, c in r) - min(c for _, c in r) <= 1
    prof = [v.DeviceProfile(cores=1, a=1e-6, t0=0.1), v.DeviceProfile(cores=1, a=2e-6, t0=0.0)]
    r = rank_ranges(1_000_000, 2, v.Strategy.S3, prof)
    assert r[0][1] > r[1][1]


def _gather_worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_03244_b200.distributed import gather_records
    rec_bytes = 16
    # rank r holds r + 2 sorted records of its own contiguous range (rank 1: none)
    n = 0 if rank == 1 else rank + 2
    recs = torch.zeros(8 * rec_bytes, dtype=torch.uint8)
    view = recs.view(torch.int64).view(-1, 2)
    for i in range(n):
        view[i, 0] = 1000 * rank + i  # photon index
        view[i, 1] = rank             # payload
    got, counts = gather_records(recs, n, rec_bytes)
    if rank == 0:
        np.save(out_path, got.numpy())
        assert counts == [0 + 2, 0, 2 + 2][:world]
    dist.barrier()
    dist.destroy_process_group()


def test_detector_record_gather_in_rank_order(tmp_path):
    """distributed.gather_records: per-rank sorted records (ragged counts, one
    rank empty) concatenated on rank 0 in rank order, byte for byte."""
    out = str(tmp_path / "recs.npy")
    mp.spawn(_gather_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    got = np.load(out).view(np.int64).reshape(-1, 2)
    assert got[:, 0].tolist() == [0, 1, 2000, 2001, 2002, 2003]
    assert got[:, 1].tolist() == [0, 0, 2, 2, 2, 2]
