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
    assert line["gpu_launches"] >= 3 and line["gpu_launches"] % 3 == 0  # transport (+ replica fold) per step
    assert line["roofline"]["bound"] == "fp32" and 0 < line["roofline"]["frac"] < 1
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_two_ranks_gloo(gpu):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--backend", "gloo", "--steps", "2", "--warmup", "3", "--photons", "500000", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["photons_total"] == 1_000_000


def test_bench_reference_arm():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
