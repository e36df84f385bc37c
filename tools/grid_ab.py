"""A/B of the persistent grid size (VMC_CTAS_PER_SM) vs photon count: device
photons/ms, best of 3. usage: python tools/grid_ab.py [workloads] [ctas]"""
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
    for n in (100_000, 300_000, 1_000_000, 3_000_000, 10_000_000):
        st = v.baseline_setup(name, photons=n)
        best = min(v.run_group_dynamic(0, n, 1, st.scene, st.config).wall_ms for _ in range(3))
        out[f"{name}@{n:.0e}"] = n / best
print(json.dumps(out))
"""

if __name__ == "__main__":
    work = sys.argv[1].split(",") if len(sys.argv) > 1 else ["b1", "b2"]
    ctas = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 3, 4]
    for c in ctas:
        env = dict(os.environ, VMC_CTAS_PER_SM=str(c))
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, work)], env=env, capture_output=True, text=True)
        if r.returncode:
            print(r.stderr[-2000:], file=sys.stderr)
            continue
        print(c, {k: round(x) for k, x in json.loads(r.stdout.strip().splitlines()[-1]).items()}, flush=True)
