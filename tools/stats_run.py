"""One run per workload with the -DVMC_STATS debug build (prints warp-scheduling counters)."""
import sys
sys.path.insert(0, ".")
import paper_1711_03244_b200 as v  # noqa: E402
for name in (sys.argv[1:] or ["b1", "b2", "b3", "head"]):
    n = 10_000_000 if name != "head" else 2_000_000
    st = v.baseline_setup(name, photons=n)
    r = v.run_group_dynamic(0, n, 1, st.scene, st.config)
    print(f"{name}: {n / r.wall_ms:.0f} photons/ms", flush=True)
