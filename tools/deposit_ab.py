"""A/B of K1f's deposit paths (VMC_DEPOSIT=direct|warp|hotbox): device
photons/ms per BASELINE workload, best of 3 launches, one process per mode so
each plan selects its kernel at creation. Usage: python tools/deposit_ab.py [N]"""
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
for name, n in %s:
    st = v.baseline_setup(name, photons=n)
    p = v.Plan(st.scene, st.config); k = p.kernel; p.close()
    best = min(v.run_group_dynamic(0, n, 1, st.scene, st.config).wall_ms for _ in range(3))
    out[name] = {"kernel": k, "ms": best, "photons_per_ms": n / best}
print(json.dumps(out))
"""

if __name__ == "__main__":
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
    work = [("b1", n), ("b2", n), ("b3", n), ("head", max(1, n // 5))]
    res = {}
    for mode in ("direct", "warp", "hotbox", "direct"):
        env = dict(os.environ, VMC_DEPOSIT=mode)
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, work)], env=env, capture_output=True, text=True)
        if r.returncode:
            print(r.stderr[-2000:], file=sys.stderr)
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        res.setdefault(mode, []).append(d)
        print(mode, {k: (x["kernel"], round(x["photons_per_ms"])) for k, x in d.items()}, flush=True)
    print(json.dumps(res))
