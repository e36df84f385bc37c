"""Throughput sweep used during kernel tuning (device time, 1 GPU)."""
import sys
sys.path.insert(0, ".")
import paper_1711_03244_b200 as v  # noqa: E402
for name, n in [("b1", 10_000_000), ("b2", 10_000_000), ("b3", 10_000_000), ("head", 2_000_000)]:
    st = v.baseline_setup(name, photons=n)
    best = 1e30
    for _ in range(3):
        best = min(best, v.run_group_dynamic(0, n, 1, st.scene, st.config).wall_ms)
    print(f"tp {name} N={n}: {best:.2f} ms -> {n / best:.0f} photons/ms", flush=True)
