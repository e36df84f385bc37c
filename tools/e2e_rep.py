import sys, time
sys.path.insert(0, ".")
import torch
import paper_1711_03244_b200 as v
n = 100_000_000
st = v.baseline_setup("b1", photons=n)
def rgd(tag):
    print(tag, " ".join(f"{v.run_group_dynamic(0, n, 1, st.scene, st.config).wall_ms:.1f}" for _ in range(2)), flush=True)
rgd("fresh")
plan = v.Plan(st.scene, st.config, 0)
cells = torch.zeros(plan.ncells, dtype=torch.int64, device="cuda")
tot = torch.zeros(4, dtype=torch.int64, device="cuda")
rgd("after plan")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
rgd("after flush alloc")
s = torch.cuda.current_stream()
for i in range(3):
    plan.run_torch(0, n, cells, tot, None, None, stream=s, zero=True)
torch.cuda.synchronize()
rgd("after plan runs")
for i in range(5):
    flush.fill_(i & 0xFF)
    plan.run_torch(0, n, cells, tot, None, None, stream=s, zero=True)
torch.cuda.synchronize()
rgd("after flush loop")
x = tot.cpu()
rgd("after tot.cpu")
