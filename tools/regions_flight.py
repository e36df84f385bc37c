"""Print the sass_cats.py region spec for csrc/flight.cuh from its lambda definitions."""
import re
src = open("paper_1711_03244_b200/csrc/flight.cuh").read().split("\n")
names = {"quant", "absorb", "decode", "deposit_run", "scat_len", "finish", "setup", "end_flight", "walk", "scatter",
         "face", "launch"}
marks = []
for i, l in enumerate(src, 1):
    m = re.match(r"\s*auto (\w+) = \[&\]", l)
    if m:
        marks.append((i, m.group(1)))
    if "// ================= event phase" in l:
        marks.append((i - 1, "evsched"))
    if "// ================= walk phase" in l:
        marks.append((i, "walksched"))
    if "// ---- epilogue" in l:
        marks.append((i, "epi"))
marks.sort()
out = []
for k, (i, n) in enumerate(marks):
    j = marks[k + 1][0] - 1 if k + 1 < len(marks) else i + 100
    if n in names or n in ("evsched", "walksched", "epi"):
        out.append(f"{n}:{i}-{j}")
print(",".join(out))
