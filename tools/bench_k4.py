"""K4 (vmc_plan_normalize) bandwidth on the head 256^3 x 10-gate map.

The normalize/export pass is the one HBM-bound kernel of the path: it streams
the int64 map (1.34 GB) and writes float32 fluence (0.67 GB). Prints one JSON
line with achieved GB/s against MEASURED_PEAKS.json hbm_gbs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_03244_b200 as v  # noqa: E402


def main():
    st = v.baseline_setup("head", photons=100_000_000)
    plan = v.Plan(st.scene, st.config)
    n = plan.ncells
    cells = torch.randint(0, 1 << 40, (n,), dtype=torch.int64, device="cuda")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        plan.normalize_torch(cells, out, st.config.photon_count, sum_gates=False)
    ms = []
    for i in range(10):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.normalize_torch(cells, out, st.config.photon_count, sum_gates=False)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = sorted(ms)[len(ms) // 2]
    nbytes = n * 8 + n * 4 + st.grid.voxel_count  # map in, fluence out, labels once
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json"))) if os.path.exists("MEASURED_PEAKS.json") else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    gbs = nbytes / (t * 1e-3) / 1e9
    print(json.dumps({"kernel": "k_normalize (K4)", "cells": n, "ms_median": t, "algorithmic_bytes": nbytes,
                      "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak}))


if __name__ == "__main__":
    main()
