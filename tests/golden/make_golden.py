"""Generates tests/golden/golden.json from the COMPILED REFERENCE (oracle/_ref,
built by oracle/Makefile from /root/reference/proj/core/src). Run in the
build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

The fixture pins (a) the reference's own recorded whole-run checksum
(proj/test_output.txt:25: B1, 1e5 photons, seed 1 -> 428b1d605a48eb37), (b) the
RNG known-answer vectors and per-photon values of SURVEY.md Appendix A, (c)
run-level numbers for every BASELINE workload at small N, used by the GPU parity
tests on the box where /root/reference is absent.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1711_03244_b200 import scene as S  # noqa: E402


def main():
    R = oracle.ref()
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj (voxmc)"}
    out["mix64_0"] = f"{R.lib.ref_mix64(0):016x}"
    kats = []
    for seed, sid in [(0, 0), (1, 0), (1, 1), (42, 1), (20260826, 123456789), (2**64 - 1, 7)]:
        o, st, u = R.rng_kat(seed, sid, 16)
        kats.append({"seed": seed, "id": sid, "state": [f"{x:016x}" for x in st],
                     "u64": [f"{x:016x}" for x in o], "first_unit": u})
    out["rng"] = kats

    photons = []
    for name, bench in [("B1", S.Benchmark.B1), ("B2", S.Benchmark.B2)]:
        st = S.benchmark_preset(bench)
        st.config.master_seed = 1
        for idx in [0, 1, 2, 3, 12345, 99999]:
            deps, disp = R.trace(st.scene, st.config, idx)
            photons.append({"bench": name, "index": idx, "ndeps": len(deps),
                            "first_cell": deps[0][0] if deps else -1,
                            "first_dw": deps[0][1] if deps else 0.0, "disp": disp})
    out["photons"] = photons

    runs = []
    for name, bench in [("B1", S.Benchmark.B1), ("B2", S.Benchmark.B2)]:
        st = S.benchmark_preset(bench)
        st.config.master_seed = 1
        st.config.photon_count = 100_000
        cells, disp, _ = R.run_group(st.scene, st.config, 0, 100_000, 8)
        q = R.quantum_for(100_000)
        runs.append({"bench": name, "photons": 100_000, "seed": 1,
                     "checksum": oracle.volume_checksum(cells, q), "raw_sum": int(cells.sum()),
                     "disp": disp, "quantum": q})
    out["runs"] = runs

    # BASELINE workloads at N = 2e5 (seed 1): run-level numbers + the map
    # summary used by the GPU gates (absorbed fraction, voxels with >= 100 deposits)
    # plus the head at its production size (256^3, 10 gates; 5e4 photons) and
    # B1 at BASELINE's own photon count (1e6)
    work = {}
    for name, n in [("b1", 200_000), ("b2", 200_000), ("b3", 200_000), ("head64", 200_000),
                    ("head256", 50_000), ("b1_1e6", 1_000_000)]:
        if name == "head64":
            st = S.baseline_setup("head", photons=n, head_n=64)
        elif name == "head256":
            st = S.baseline_setup("head", photons=n, head_n=256)
        else:
            st = S.baseline_setup(name.split("_")[0], photons=n)
        w = R.walk(st.scene, st.config, 0, n, threads=os.cpu_count() or 8, cells=True,
                   counts=True, traces=False, detectors=bool(st.config.detectors))
        rec = {"photons": n, "disp": w["disp"], "raw_sum": int(w["cells"].sum()),
               "gate_sums": [int(x) for x in w["cells"].reshape(st.config.ngates, -1).sum(axis=1)],
               "voxels_ge100": int((w["counts"] >= 100).sum())}
        if "det_count" in w:
            rec["det_count"] = int(w["det_count"])
            rec["det_per_detector"] = [int((w["det"]["det_id"] == k).sum())
                                       for k in range(len(st.config.detectors))]
            rec["det_w_sum"] = float(w["det"]["w_exit"].astype(np.float64).sum())
        work[name] = rec
    out["workloads"] = work

    parts = []
    rng = np.random.default_rng(7)
    for _ in range(40):
        k = int(rng.integers(1, 6))
        prof = [(int(rng.integers(1, 17)), float(rng.uniform(1e-4, 5e-3)), float(rng.uniform(0, 50)))
                for _ in range(k)]
        total = int(rng.integers(0, 100_000))
        rec = {"total": total, "profiles": prof}
        for s in (1, 2, 3):
            rec[f"s{s}"] = R.partition(s, total, prof)[0]
        parts.append(rec)
    out["partitions"] = parts

    with open(os.path.join(os.path.dirname(__file__), "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote golden.json")


if __name__ == "__main__":
    main()
