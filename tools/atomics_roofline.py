"""Secondary roofline of the transport kernel: L2 red.add.u64 throughput.
Samples a 2^22-long cell-index stream from the per-voxel deposit COUNTS of the
compiled reference on B1 (oracle, 2e5 photons: the address distribution the
kernel's deposits follow), runs lib/atomics_bench on it (plus uniform / hot-spot
/ single-address streams), and prints one JSON line.
usage: python tools/atomics_roofline.py [out.json]"""
import json, os, subprocess, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_1711_03244_b200 as v
st = v.baseline_setup("b1", photons=200_000)
w = oracle.ref().walk(st.scene, st.config, 0, 200_000, threads=os.cpu_count() or 8, cells=False, counts=True)
counts = w["counts"].astype(np.float64)
p = counts / counts.sum()
rng = np.random.default_rng(1)
stream = rng.choice(len(p), size=1 << 22, p=p).astype(np.int32)
path = "/tmp/vmc_b1_deposit_stream.i32"
stream.tofile(path)
exe = os.path.join("paper_1711_03244_b200", "lib", "atomics_bench")
out = json.loads(subprocess.run([exe, "256", path], capture_output=True, text=True, check=True).stdout)
top = np.sort(p)[::-1]
out["replay_source"] = ("B1 per-voxel deposit counts of the compiled reference (2e5 photons): top-256 voxels "
                        f"{top[:256].sum():.3f}, top-4096 {top[:4096].sum():.3f} of all deposits")
line = json.dumps(out)
print(line)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(line + "\n")
