"""Summarise an ncu --set full report of the transport kernel into a text file
for profiles/ (the report itself stays in gpurun_out/).

usage: python tools/make_profile_summary.py <rep> <obj> <kernel-mangled> <photons> <out.txt> [title]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp", "Executed Instructions",
        "Registers Per Thread", "Block Size", "Grid Size", "Theoretical Occupancy", "Achieved Occupancy",
        "Branch Efficiency", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_requests_op_red.sum",
       "lts__t_requests_op_atom.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
       "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed.avg.per_cycle_active",
       "gpu__time_duration.sum"]
STALLS = ["not_selected", "wait", "math_pipe_throttle", "selected", "long_scoreboard", "short_scoreboard",
          "branch_resolving", "no_instructions", "dispatch_stall", "mio_throttle", "lg_throttle", "barrier"]


def ncu(rep, page, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                          text=True).stdout


def main():
    rep, obj, kern, n, out = sys.argv[1:6]
    title = sys.argv[6] if len(sys.argv) > 6 else rep
    lines = [f"# {title}", f"report: {rep}", f"photons in the profiled launch: {float(n):.0f}", ""]
    rows = list(csv.reader(io.StringIO(ncu(rep, "details"))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    lines.append("## ncu details (subset)")
    for r in rows[1:]:
        if r[ix["Metric Name"]] in KEYS:
            lines.append(f"{r[ix['Metric Name']]:45s} {r[ix['Metric Value']]:>20s} {r[ix['Metric Unit']]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "raw"))))
    h, u, v = raw[0], raw[1], raw[2]
    lines += ["", "## raw metrics"]
    for i, name in enumerate(h):
        if name in RAW:
            lines.append(f"{name:60s} {v[i]:>20s} {u[i]}")
    lines += ["", "## warp stall samples (pc sampling, all samples)"]
    tot = 0
    st = {}
    for i, name in enumerate(h):
        for s in STALLS:
            if name == f"smsp__pcsamp_warps_issue_stalled_{s}":
                st[s] = float(v[i].replace(",", "") or 0)
                tot += st[s]
    for s, c in sorted(st.items(), key=lambda kv: -kv[1]):
        lines.append(f"{s:25s} {100 * c / max(tot, 1):6.1f} %")
    lines += ["", "## per-region breakdown (SASS joined with -lineinfo)"]
    reg = subprocess.run([sys.executable, "tools/sass_cats.py", rep, obj, kern, n, sys.argv[7] if len(sys.argv) > 7
                          else "all:1-100000"], capture_output=True, text=True).stdout
    lines += reg.rstrip().split("\n")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
