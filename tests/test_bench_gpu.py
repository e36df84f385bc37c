"""bench.py contract on the GPU: one JSON line with the required keys; the
N>1 torchrun path (2 ranks) run end to end with the gloo backend on one GPU
(NCCL refuses two ranks on one device), which exercises the rank ranges, the
reduce of the int64 maps and the rank-0 energy audit."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
            "gpu_launches"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_bench_single_gpu_line(gpu):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--photons", "2000000",
                        "--cpu-seconds", "1", "--e2e-steps", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in REQUIRED:
        assert k in line, k
    assert line["value"] > 0 and line["n_gpus"] == 1
    # per step: transport + replica fold + the record sort's key/gather kernels
    assert line["gpu_launches"] >= 3 * 2
    assert line["roofline"]["bound"] == "fp32" and 0 < line["roofline"]["frac"] < 1
    assert line["roofline"]["kernel"] == "k_flight<float,0,1,0,0,0>"  # the B3 production variant
    assert line["scaling"] == "strong" and "configs[4]" in line["config"]["workload"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] > 0
    assert line["cpu_baseline"]["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["config"]["detections_per_step"] > 0


def _dump(path):
    import numpy as np
    d = np.load(path)
    return d["cells"], d["totals"], d["recs"], int(d["det_count"][0])


@pytest.mark.gpu
def test_bench_two_ranks_gloo_equals_one_rank(gpu, tmp_path):
    """The multi-GPU entry point end to end with 2 ranks (gloo: NCCL refuses
    two ranks on one device): contiguous S1 ranges, the int64 map reduce and
    the sorted detector-record gather give rank 0 the 1-rank result bit for
    bit (the multi-device contract, test_scheduler.cpp:246-264)."""
    import numpy as np
    one, two = str(tmp_path / "one.npz"), str(tmp_path / "two.npz")
    base = ["bench.py", "--workload", "scale", "--photons", "1000000", "--steps", "2", "--warmup", "3",
            "--e2e-steps", "1", "--no-cpu-baseline"]
    r1 = subprocess.run([sys.executable] + base + ["--dump", one], cwd=ROOT, capture_output=True, text=True,
                        timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + base + [
               "--gpus", "2", "--backend", "gloo", "--dump", two]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["photons_total"] == 1_000_000
    c1, t1, rec1, n1 = _dump(one)
    c2, t2, rec2, n2 = _dump(two)
    assert n1 == n2 > 100
    assert np.array_equal(c1, c2) and np.array_equal(t1, t2)
    assert np.array_equal(rec1, rec2)
    import paper_1711_03244_b200 as v
    recs = rec1.view(v.runtime._abi.det_record_dtype(3))
    assert len(recs) == n1 and np.all(np.diff(recs["photon_index"].astype(np.int64)) > 0)


@pytest.mark.gpu
def test_bench_more_gpus_than_present_fails_loudly(gpu):
    n = gpu.device_count() + 1
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "1", "--warmup", "3"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert f"--gpus {n}" in r.stderr


def test_bench_reference_arm():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
