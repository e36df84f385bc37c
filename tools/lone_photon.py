"""One photon alone on the GPU (the small-N tail's latency floor), for an ncu
capture of where a lone warp's time goes: python tools/lone_photon.py b1 587956"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1711_03244_b200 as v  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "b1"
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 587956
st = v.baseline_setup(name, photons=1_000_000)
plan = v.Plan(st.scene, st.config, 0)
cells = torch.empty(plan.ncells, dtype=torch.int64, device="cuda")
tot = torch.empty(4, dtype=torch.int64, device="cuda")
for _ in range(2):
    plan.run_torch(idx, 1, cells, tot)
torch.cuda.synchronize()
plan.close()
