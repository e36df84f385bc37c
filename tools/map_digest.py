"""Digest of integer fluence maps + disposition quanta for fixed runs (A/B
bit-identity checks between kernel builds). usage: map_digest.py [libpath]"""
import hashlib
import sys
sys.path.insert(0, ".")
import paper_1711_03244_b200 as v  # noqa: E402
from paper_1711_03244_b200 import runtime  # noqa: E402

if len(sys.argv) > 1:
    runtime.LIB_PATH = sys.argv[1]
for name, n in [("b1", 1_000_000), ("b2", 1_000_000), ("b3", 1_000_000), ("head", 100_000)]:
    st = v.baseline_setup(name, photons=n)
    r = v.run_group_dynamic(0, n, 1, st.scene, st.config)
    h = hashlib.sha1(r.map.cells.tobytes()).hexdigest()[:16]
    print(f"digest {name} {h} {tuple(r.totals_q)}", flush=True)
