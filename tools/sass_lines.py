"""Join an ncu SASS source page (CSV) with nvdisasm line info -> per-source-line
instruction counts and stall samples (header-inlined code is invisible to
ncu's CUDA source view).

usage: python tools/sass_lines.py <ncu-rep> <object.o> <mangled kernel name> [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_map(obj, kernel):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   stdout=subprocess.DEVNULL)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    out, cur, inside = {}, None, False
    for ln in txt.split("\n"):
        if ln.startswith(".text." + kernel + ":"):
            inside = True
            continue
        if inside and ln.startswith(".text.") and kernel not in ln:
            break
        if not inside:
            continue
        m = re.match(r"\s*//## File \"(.*)\", line (\d+)", ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m:
            out[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return out


def main():
    rep, obj, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(obj, kernel)
    csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                            capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csvtxt)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    base = int(rows[2][0], 16)
    agg = collections.defaultdict(lambda: [0, 0, 0])
    tot = [0, 0, 0]
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        off = int(r[0], 16) - base
        key = lm.get(off, (None, ""))[0] or ("?", 0)
        inst = int(r[ix["Instructions Executed"]] or 0)
        thr = int(r[ix["Thread Instructions Executed"]] or 0)
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        a = agg[key]
        a[0] += inst
        a[1] += thr
        a[2] += smp
        tot[0] += inst
        tot[1] += thr
        tot[2] += smp
    print(f"total warp-inst {tot[0]:.3e} thread-inst {tot[1]:.3e} samples {tot[2]} "
          f"simt {tot[1] / max(1, 32 * tot[0]):.3f}")
    print(f"{'file:line':40s} {'warp-inst%':>10s} {'samples%':>9s} {'simt':>6s}")
    for key, (i, t, s) in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
        print(f"{key[0] + ':' + str(key[1]):40s} {100 * i / tot[0]:10.2f} {100 * s / max(1, tot[2]):9.2f} "
              f"{t / max(1, 32 * i):6.2f}")


if __name__ == "__main__":
    main()
