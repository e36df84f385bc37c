"""Generic A/B over environment knobs of the library: device photons/ms of one
run_group_dynamic call (best of 3) per workload and photon count, one process
per setting. usage:
  python tools/env_ab.py b1,b2 1e6,1e7,1e8 "VMC_SPILL_PHASES=0 VMC_SPILL_KEEP=16" "VMC_SPILL_PHASES=6" ...
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json
sys.path.insert(0, %r)
import paper_1711_03244_b200 as v
out = {}
for name in %r:
    for n in %r:
        st = v.baseline_setup(name, photons=n)
        best = min(v.run_group_dynamic(0, n, 1, st.scene, st.config).wall_ms for _ in range(3))
        out[f"{name}@{n:.0e}"] = n / best
print(json.dumps(out))
"""

if __name__ == "__main__":
    work = sys.argv[1].split(",")
    ns = [int(float(x)) for x in sys.argv[2].split(",")]
    for setting in sys.argv[3:]:
        env = dict(os.environ)
        for kv in setting.split():
            k, val = kv.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, work, ns)], env=env, capture_output=True, text=True)
        if r.returncode:
            print(setting, "FAILED", r.stderr[-1500:], flush=True)
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"{setting:40s}", {k: round(x) for k, x in d.items()}, flush=True)
