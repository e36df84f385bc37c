"""Per-photon RNG draw-count agreement of the FP32 kernels with the compiled
reference (FP64, same seed and photon indices): K1f (default) and K1
(VMC_KERNEL=step). usage: python tools/draw_parity.py [n]"""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_1711_03244_b200 as v
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20000
ref = oracle.ref()
for name in ("b1", "b2", "b3", "head"):
    st = v.baseline_setup(name, photons=200_000, head_n=64) if name == "head" else v.baseline_setup(name, photons=200_000)
    rt = ref.walk(st.scene, st.config, 0, n, threads=os.cpu_count() or 8, cells=False, traces=True)["traces"]
    out = []
    for k in ("flight", "step"):
        if k == "step":
            os.environ["VMC_KERNEL"] = "step"
        else:
            os.environ.pop("VMC_KERNEL", None)
        tr = v.trace_photons(st.scene, st.config, 0, n)
        same = tr["draws"] == rt["draws"]
        out.append(f"{k}: draws identical {same.mean():.5f}, |absorbed - ref| mean {np.abs(tr['deposited'] - rt['deposited']).mean():.2e}")
    print(f"{name} ({n} photons): " + "; ".join(out), flush=True)
