"""Quick GPU probe: RNG KAT, per-photon FP64/FP32 parity vs the reference, run-level
parity and throughput. Developer tool (imports the oracle as the checker)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1711_03244_b200 as v  # noqa: E402

R = oracle.ref()
print("devices", v.device_count(), flush=True)
kat = v.rng_kat(20260826, 123456789, 4)
print("kat", [hex(x) for x in kat], kat == R.rng_kat(20260826, 123456789, 4)[0], flush=True)


def parity(name, n_trace=20000, n_run=200000):
    st = v.baseline_setup(name, photons=n_run, head_n=64)
    st.config.master_seed = 1
    for prec in (v.Precision.FP64, v.Precision.FP32):
        st.config.precision = prec
        t0 = time.time()
        tr = v.trace_photons(st.scene, st.config, 0, n_trace)
        t1 = time.time()
        ref = R.walk(st.scene, st.config, 0, n_trace, threads=8, cells=False, traces=True)["traces"]
        same = (tr["draws"] == ref["draws"]).mean()
        dd = np.abs(tr["deposited"] - ref["deposited"])
        ok = tr["draws"] == ref["draws"]
        print(f"{name} {prec.name}: draws identical {same:.5f}; |ddep| max(same-draw) "
              f"{dd[ok].max():.3e} mean {dd.mean():.3e}; gpu {t1-t0:.2f}s", flush=True)
    st.config.precision = v.Precision.FP32
    t0 = time.time()
    g = v.run_group_dynamic(0, n_run, 1, st.scene, st.config)
    t1 = time.time()
    rc, rd, rw = R.run_group(st.scene, st.config, 0, n_run, 8)
    gc = g.map.cw_cells()
    print(f"{name} run {n_run}: gpu wall {g.wall_ms:.2f} ms (host {1e3*(t1-t0):.1f} ms); ref {rw:.0f} ms", flush=True)
    print("   totals gpu", g.totals, " books", g.totals.books() / n_run, flush=True)
    print("   totals ref", rd, sum(rd) / n_run, flush=True)
    absr = g.totals.deposited / rd[0] - 1
    m = rc > 0
    l2 = np.sqrt(((gc[m] - rc[m]).astype(np.float64) ** 2).sum() / (rc[m].astype(np.float64) ** 2).sum())
    print(f"   absorbed rel diff {absr:.3e}; map L2 rel {l2:.3e}", flush=True)


for name in ["b1", "b2", "b3"]:
    parity(name)

# throughput
for name, n in [("b1", 1_000_000), ("b1", 10_000_000), ("b2", 10_000_000), ("b3", 10_000_000)]:
    st = v.baseline_setup(name, photons=n)
    st.config.detectors = []
    g = v.run_group_dynamic(0, n, 1, st.scene, st.config)
    g = v.run_group_dynamic(0, n, 1, st.scene, st.config)
    print(f"throughput {name} N={n}: {g.wall_ms:.2f} ms -> {n / g.wall_ms:.0f} photons/ms", flush=True)
