"""Per-photon RNG draw identity on the 'mosaic' corner scene: FP32 flight kernel,
FP32 per-step kernel (VMC_KERNEL=step), FP64 flight kernel, against the compiled
reference; plus where the FP32 divergences sit (roulette / horizon / exits)."""
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1711_03244_b200 as v  # noqa: E402
from scenes import corner_scene  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "mosaic"
scene, cfg = corner_scene(kind)
n = 5000
rt = oracle.ref().walk(scene, cfg, 0, n, threads=8, cells=False, traces=True)["traces"]
for label, env, prec in (("flight fp32", None, v.Precision.FP32), ("step fp32", "step", v.Precision.FP32),
                         ("flight fp64", None, v.Precision.FP64)):
    if env:
        os.environ["VMC_KERNEL"] = env
    else:
        os.environ.pop("VMC_KERNEL", None)
    cfg.precision = prec
    tr = v.trace_photons(scene, cfg, 0, n)
    same = tr["draws"] == rt["draws"]
    diff = ~same
    fl = rt["flags"]
    print(f"{label:12s} identical {same.mean():.4f}; diverged: ref killed {np.mean(fl[diff] & 2 > 0):.2f} "
          f"truncated {np.mean(fl[diff] & 4 > 0):.2f} escaped {np.mean(fl[diff] & 1 > 0):.2f}; "
          f"all photons: killed {np.mean(fl & 2 > 0):.2f} truncated {np.mean(fl & 4 > 0):.2f}", flush=True)
