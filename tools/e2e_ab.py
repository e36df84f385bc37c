"""A/B the two launch paths of the same kernel in one process: Plan.run_torch
(device buffers owned by torch) vs run_group_dynamic (vmc_run_range, cached
library buffers). usage: python tools/e2e_ab.py [workload] [photons]"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1711_03244_b200 as v
wl = sys.argv[1] if len(sys.argv) > 1 else "b1"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000_000
st = v.baseline_setup(wl, photons=n)
plan = v.Plan(st.scene, st.config, 0)
cells = torch.zeros(plan.ncells, dtype=torch.int64, device="cuda")
tot = torch.zeros(4, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
def plan_ms():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); plan.run_torch(0, n, cells, tot, None, None, stream=s, zero=True); e1.record(s)
    torch.cuda.synchronize(); return e0.elapsed_time(e1)
for rnd in range(2):
    print("plan.run_torch ms:", " ".join(f"{plan_ms():.1f}" for _ in range(3)), flush=True)
    print("run_group_dynamic ms:", " ".join(f"{v.run_group_dynamic(0, n, 1, st.scene, st.config).wall_ms:.1f}" for _ in range(3)), flush=True)
