"""Small-N tail probe: how long do the longest photons of a run take on their
own? Traces N photons of a workload, picks the three with the most scatters,
times a one-photon run of each (the latency floor of the run's tail), then the
full N-photon run.
usage: python tools/tail_probe.py b1 1e6
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_03244_b200 as v  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "b1"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1000000
st = v.baseline_setup(name, photons=n)
plan = v.Plan(st.scene, st.config, 0)
tr = plan.trace(0, n)
sc = tr["scatters"].astype(np.int64)
order = np.argsort(-sc)
print(f"{name} N={n}: scatters mean {sc.mean():.1f} p99 {np.percentile(sc, 99):.0f} p99.9 "
      f"{np.percentile(sc, 99.9):.0f} max {sc.max()} (photon {order[0]})", flush=True)
cells = torch.empty(plan.ncells, dtype=torch.int64, device="cuda")
tot = torch.empty(4, dtype=torch.int64, device="cuda")
det = det_n = None
if st.config.detectors:
    det = torch.empty(max(1, st.config.det_capacity) * plan.rec_bytes, dtype=torch.uint8, device="cuda")
    det_n = torch.empty(1, dtype=torch.int64, device="cuda")


def dev_ms(first, count, reps=3):
    best = 1e30
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        plan.run_torch(first, count, cells, tot, det, det_n)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


dev_ms(0, 1000)
for k in range(3):
    i = int(order[k])
    ms = dev_ms(i, 1)
    print(f"photon {i}: {sc[i]} scatters alone: {ms:.3f} ms = {1e3 * ms / max(1, sc[i]):.2f} us/scatter", flush=True)
ms = dev_ms(0, n)
print(f"full run N={n}: {ms:.3f} ms -> {n / ms:.0f} photons/ms", flush=True)
plan.close()
