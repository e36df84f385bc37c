"""B3 with and without its 4 detectors (same scene, same photons): the cost of
the detector machinery (per-label path lengths, exit hit test, record append)."""
import sys
sys.path.insert(0, ".")
import paper_1711_03244_b200 as v  # noqa: E402
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
for det in (True, False):
    st = v.baseline_setup("b3", photons=n)
    if not det:
        st.config.detectors = []
        st.config.det_capacity = 0
    else:
        st.config.det_capacity = int(n * 1e-2)
    p = v.Plan(st.scene, st.config); k = p.kernel; p.close()
    best = min(v.run_group_dynamic(0, n, 1, st.scene, st.config).wall_ms for _ in range(3))
    print(f"detectors={det}: {k} {n / best:.0f} photons/ms", flush=True)
