"""Rewrite the headline numbers in profiles/README.md, DESIGN.md and README.md from
the committed bench lines (profiles/r1_bench_*.json) and profiles/roofline_traffic.json."""
import json, re
v, tj = {}, json.load(open("profiles/roofline_traffic.json"))
for w in ("b1", "b2", "b3", "head"):
    d = json.load(open(f"profiles/r1_bench_{w}.json"))
    v[w] = (d["value"] / 1e3, d["e2e"]["value"] / 1e3, d["cpu_baseline"]["value"] / 1e3)
b1 = json.load(open("profiles/r1_bench_b1.json"))
aj = json.load(open("profiles/r1_atomics_roofline.json"))
wi = {w: tj["issue"][w]["warp_inst_per_photon"] for w in v}
k1 = {"b1": "415.6", "b2": "252.9", "b3": "198.7", "head": "63.4"}
names = {"b1": "B1 cube60, terminate", "b2": "**B2 cube60 + Fresnel (bench default)**",
         "b3": "B3 cube60 + sphere + 4 detectors"}

p = "profiles/README.md"
s = open(p).read()
a = s.index("| B1 cube60, terminate | **"); b = s.index("\n\n", a)
rows = [f"| B1 cube60, terminate | **{v['b1'][0]:.1f} k** | {v['b1'][1]:.1f} k | {v['b1'][2]:.2f} k | 415.6 k |",
        f"| **B2 cube60 + Fresnel (bench default)** | **{v['b2'][0]:.1f} k** | **{v['b2'][1]:.1f} k** | {v['b2'][2]:.2f} k | 252.9 k |",
        f"| B3 cube60 + sphere + 4 detectors | {v['b3'][0]:.1f} k | {v['b3'][1]:.1f} k | {v['b3'][2]:.2f} k | 198.7 k |",
        f"| head 256³, 10 gates × 0.5 ns | {v['head'][0]:.1f} k | {v['head'][1]:.1f} k (1.34 GB map download) | {v['head'][2]:.2f} k | 63.4 k |"]
s = s[:a] + "\n".join(rows) + s[b:]
i = s.index("Warp instructions per photon (ncu, 1e8 photons)"); j = s.index("\n\n", i)
s = s[:i] + (f"Warp instructions per photon (ncu, 1e8 photons): B1 {wi['b1']:.0f} (K1: 2484), B2 {wi['b2']:.0f} (4108), "
             f"B3 {wi['b3']:.0f}\n(5104), head {wi['head']:.0f} (16004); issue slots 85-88 % busy in every case "
             f"(`roofline_traffic.json`).\nL2 atomics (`r1_atomics_roofline.json`, `lib/atomics_bench` with the B1 "
             f"deposit-address\ndistribution of the reference): B1 deposits {b1['roofline']['l2_atomics_per_s']:.2e} "
             f"red.add/s = {100 * b1['roofline']['secondary']['l2_atomics']['frac']:.0f} % of the "
             f"{aj['replay_rep8']:.2e}/s that\ndistribution sustains into 8 replicas (16 / 32 replicas: "
             f"{aj['replay_rep16']:.2e} / {aj['replay_rep32']:.2e}; uniform addresses:\n{aj['uniform']:.2e}/s; one map: "
             f"{aj['replay']:.2e}/s).") + s[j:]
open(p, "w").write(s)

p = "DESIGN.md"
s = open(p).read()
a = s.index("| B1 cube60, terminate | "); b = s.index("BASELINE.json's ≥ 1e6")
s = s[:a] + (f"| B1 cube60, terminate | {v['b1'][0]:.1f} k | {v['b1'][1]:.1f} k | {v['b1'][2]:.2f} k |\n"
             f"| **B2 cube60 + Fresnel (bench default)** | **{v['b2'][0]:.1f} k** | **{v['b2'][1]:.1f} k** | {v['b2'][2]:.2f} k |\n"
             f"| B3 cube60 + sphere + 4 detectors | {v['b3'][0]:.1f} k | {v['b3'][1]:.1f} k | {v['b3'][2]:.2f} k |\n"
             f"| head 256³ × 10 gates | {v['head'][0]:.1f} k | {v['head'][1]:.1f} k (1.34 GB map download) | "
             f"{v['head'][2]:.2f} k |\n\n") + s[b:]
s = re.sub(r"\*\*Measured\*\* \(1e8 photons/step, same box\): B1 [0-9.]+ k photons/ms \(K1 415.6 k\), B2 [0-9.]+ k\n"
           r"\(252.9 k\), B3 [0-9.]+ k \(198.7 k\), head [0-9.]+ k",
           f"**Measured** (1e8 photons/step, same box): B1 {v['b1'][0]:.1f} k photons/ms (K1 415.6 k), B2 "
           f"{v['b2'][0]:.1f} k\n(252.9 k), B3 {v['b3'][0]:.1f} k (198.7 k), head {v['head'][0]:.1f} k", s)
s = re.sub(r"\(ncu\): B1 [0-9]+ vs 2484, B2 [0-9]+ vs 4108\.", f"(ncu): B1 {wi['b1']:.0f} vs 2484, B2 {wi['b2']:.0f} vs 4108.", s)
s = re.sub(r"not reached \(0\.[0-9]+e6 at 1e8\): at [0-9]+ warp", f"not reached ({v['b1'][0] / 1e3:.2f}e6 at 1e8): at {wi['b1']:.0f} warp", s)
s = re.sub(r"B1 at 1e8 photons: [0-9]+ warp instructions per photon", f"B1 at 1e8 photons: {wi['b1']:.0f} warp instructions per photon", s)
s = re.sub(r"deposits already run at [0-9]+ % of the L2", f"deposits already run at {100 * b1['roofline']['secondary']['l2_atomics']['frac']:.0f} % of the L2", s)
open(p, "w").write(s)

p = "README.md"
s = open(p).read()
s = re.sub(r"B1 [0-9]+ k photons/ms,\nB2 [0-9]+ k, B3 [0-9]+ k, head 256³ × 10 gates [0-9]+ k",
           f"B1 {v['b1'][0]:.0f} k photons/ms,\nB2 {v['b2'][0]:.0f} k, B3 {v['b3'][0]:.0f} k, head 256³ × 10 gates {v['head'][0]:.0f} k", s)
open(p, "w").write(s)
print({w: round(x[0], 1) for w, x in v.items()}, {w: round(x) for w, x in wi.items()})
