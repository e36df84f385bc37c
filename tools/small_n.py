"""Throughput vs photon count (drain tail + fixed costs): device time of one
run_group_dynamic call and its wall time (host buffers), best of 3."""
import sys, time
sys.path.insert(0, ".")
import paper_1711_03244_b200 as v
SIZES = {"b1": (100_000, 1_000_000, 10_000_000, 100_000_000), "b2": (100_000, 1_000_000, 10_000_000, 100_000_000),
         "b3": (100_000, 1_000_000, 10_000_000, 100_000_000), "head": (100_000, 1_000_000, 10_000_000)}
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("b1", "b2")):
    for n in SIZES[name]:
        st = v.baseline_setup(name, photons=n)
        best_dev, best_wall = 1e30, 1e30
        for _ in range(3):
            t0 = time.perf_counter()
            r = v.run_group_dynamic(0, n, 1, st.scene, st.config)
            best_wall = min(best_wall, (time.perf_counter() - t0) * 1e3)
            best_dev = min(best_dev, r.wall_ms)
        print(f"{name} N={n:>10d}: device {best_dev:9.3f} ms -> {n / best_dev:9.0f} photons/ms; "
              f"wall {best_wall:9.3f} ms -> {n / best_wall:9.0f} photons/ms", flush=True)
