"""ptxas register / spill summary of the FP32 transport kernels (compiled here, no GPU).
usage: python tools/regs.py [extra nvcc flags...]"""
import re, subprocess, sys
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
       "-I", "include", "-I", "paper_1711_03244_b200/csrc", "-DVMC_REAL=float", "-DVMC_REAL_IS_FLOAT=1", "-Xptxas", "-v",
       "-c", "paper_1711_03244_b200/csrc/transport_kernels.cu", "-o", "/tmp/regs_tk.o"] + sys.argv[1:]
err = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for ln in err.split("\n"):
    m = re.search(r"Compiling entry function '_ZN3vmc(\d+)(k_\w+?)I(\w+?)EEvNS_10KernelArgsE'", ln)
    if m:
        args = m.group(3)
        real = "float" if args.startswith("f") else ("double" if args.startswith("d") else "")
        parts = [("1" if b == "1" else "0") for b in re.findall(r"Lb(\d)", args)] + re.findall(r"Li(\d+)E", args)
        cur = m.group(2) + "<" + ",".join(([real] if real else []) + parts) + ">"
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur: spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur:
        print(f"{cur:28s} regs {m.group(1):>3s}  spill st/ld {spill[0]}/{spill[1]}")
        cur = None
