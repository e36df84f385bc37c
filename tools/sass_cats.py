"""Per-region breakdown (warp-inst, thread-inst, simt) of the transport kernel
from an ncu report. usage: sass_cats.py rep obj kernel N_photons  'name:lo-hi,...' """
import collections, csv, io, os, subprocess, sys
sys.path.insert(0, "tools")
import sass_lines as S
rep, obj, kern, n = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
cats = [(c.split(":")[0], *map(int, c.split(":")[1].split("-"))) for c in sys.argv[5].split(",")]
lm = S.line_map(obj, kern)
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt))); hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
base = int(rows[2][0], 16)
agg = collections.defaultdict(lambda: [0, 0, 0])
for r in rows[2:]:
    if len(r) < len(hdr): continue
    (f, ln), _ = lm.get(int(r[0], 16) - base, ((None, 0), ""))
    name = "other"
    if f == "rng.cuh": name = "rng"
    elif f == os.environ.get("CATFILE", "transport.cuh"):
        for c, lo, hi in cats:
            if lo <= ln <= hi: name = c; break
    elif f and "atomic" in f: name = "atomics"
    elif f and "intrinsics" in f: name = "warp-intrinsics"
    a = agg[name]; a[0] += int(r[ix["Instructions Executed"]] or 0); a[1] += int(r[ix["Thread Instructions Executed"]] or 0)
    a[2] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tw = sum(a[0] for a in agg.values()); ts = sum(a[2] for a in agg.values())
print(f"{'region':16s} {'warp/ph':>9s} {'thr/ph':>9s} {'simt':>6s} {'%inst':>6s} {'%samp':>6s}")
for k, (w, t, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:16s} {w/n:9.1f} {t/n:9.1f} {t/max(1,32*w):6.2f} {100*w/tw:6.1f} {100*s/ts:6.1f}")
