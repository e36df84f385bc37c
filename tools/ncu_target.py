"""Minimal launcher for ncu captures: one warm-up + one measured transport run.
usage: python tools/ncu_target.py <workload> <photons> [precision]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1711_03244_b200 as v  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "b2"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10_000_000
st = v.baseline_setup(wl, photons=n)
if len(sys.argv) > 3 and sys.argv[3] == "fp64":
    st.config.precision = v.Precision.FP64
plan = v.Plan(st.scene, st.config, 0)
cells = torch.zeros(plan.ncells, dtype=torch.int64, device="cuda")
tot = torch.zeros(4, dtype=torch.int64, device="cuda")
det = torch.zeros(max(1, st.config.det_capacity) * plan.rec_bytes, dtype=torch.uint8, device="cuda")
dn = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(2):
    plan.run_torch(0, n, cells, tot, det, dn)
torch.cuda.synchronize()
print("ok", tot.tolist())
