"""Break down the e2e (host-buffer) path: wall vs device time per call."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1711_03244_b200 as v
st = v.baseline_setup("b2", photons=100_000_000)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
pinned = torch.empty(60 ** 3, dtype=torch.int64, pin_memory=True).numpy()
for mode in ["pageable", "pinned"] * 2:
    rows = []
    for i in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = v.run_group_dynamic(0, n, 1, st.scene, st.config, cells_out=pinned if mode == "pinned" else None)
        t1 = time.perf_counter()
        rows.append(f"{(t1 - t0) * 1e3:.1f}/{r.wall_ms:.1f}")
    print(mode, "wall/kernel ms:", " ".join(rows), flush=True)
