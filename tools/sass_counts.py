"""Per-instruction execution counts from an ncu report, in address order.
usage: python tools/sass_counts.py <ncu-rep> <photons> [lo_hex hi_hex]"""
import csv, io, subprocess, sys
rep, n = sys.argv[1], float(sys.argv[2])
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
base = int(rows[2][0], 16)
for r in rows[2:]:
    if len(r) < len(hdr): continue
    off = int(r[0], 16) - base
    if not (lo <= off < hi): continue
    w = int(r[ix["Instructions Executed"]] or 0); t = int(r[ix["Thread Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{off:05x} {w/n:8.2f} {t/max(1,32*w):5.2f} {s:6d}  {r[ix['Source']]}")
