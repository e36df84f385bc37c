"""Kernel time vs the device address of the fluence map (B200 = two dies, each
with its own L2 half): the same launch with the int64 map placed at different
offsets of one large allocation. usage: python tools/map_placement.py [workload] [photons]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1711_03244_b200 as v
wl = sys.argv[1] if len(sys.argv) > 1 else "b1"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 20_000_000
st = v.baseline_setup(wl, photons=n)
plan = v.Plan(st.scene, st.config, 0)
big = torch.zeros(64 * 1024 * 1024 // 8 * 8, dtype=torch.int64, device="cuda")  # 512 MB
tot = torch.zeros(4, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
print("base address", hex(big.data_ptr()))
for off_mb in [0, 0.5, 1, 2, 3, 4, 6, 8, 16, 32, 64, 128, 256]:
    off = int(off_mb * 1024 * 1024) // 8
    cells = big[off:off + plan.ncells]
    ts = []
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); plan.run_torch(0, n, cells, tot, None, None, stream=s, zero=True); e1.record(s)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"offset {off_mb:6.1f} MB  addr {hex(cells.data_ptr())}: " + " ".join(f"{t:.2f}" for t in ts) + " ms", flush=True)
