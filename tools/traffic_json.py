"""Build profiles/roofline_traffic.json from the per-launch ncu metrics of the
transport kernel at the bench size (tools/gpu_prof_r2.sh -> gpurun_out/r2/traffic_<w>_<tag>.csv).
usage: python tools/traffic_json.py <tag> [out.json]"""
import csv
import io
import json
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r2a"
PHOTONS = 1e8
out = {"note": ("per transport-kernel launch at the bench size (1e8 photons), ncu --metrics ... "
                "--clock-control none (tools/gpu_prof_r2.sh); traffic = dram__bytes_read.sum + "
                "dram__bytes_write.sum. red traffic: l1tex red sectors = lanes that issued a red "
                "(profiles/README.md: the L2 request counter reads 1.5x that on B200)"),
       "issue": {}, "source": {}}
for w in ("b1", "b2", "b3", "head"):
    path = f"gpurun_out/r2/traffic_{w}_{TAG}.csv"
    rows = [r for r in csv.reader(io.StringIO(open(path).read())) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    m = {r[ix["Metric Name"]]: float(r[ix["Metric Value"]].replace(",", "")) for r in rows[1:]}
    kern = rows[1][ix["Kernel Name"]]
    out[w] = int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    ipc = m["sm__inst_executed.avg.per_cycle_active"]
    out["issue"][w] = {"kernel": kern, "ipc_active": ipc, "peak_ipc": 4.0, "frac": ipc / 4.0,
                       "simt": m["smsp__thread_inst_executed_per_inst_executed.ratio"] / 32,
                       "thread_inst_per_inst": m["smsp__thread_inst_executed_per_inst_executed.ratio"],
                       "warp_inst_per_photon": m["smsp__inst_executed.sum"] / PHOTONS,
                       "red_lanes_per_photon": m["l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum"] / PHOTONS,
                       "red_instructions_per_photon": m["smsp__sass_inst_executed_op_global_red.sum"] / PHOTONS,
                       "l2_red_requests_per_photon": m["lts__t_requests_op_red.sum"] / PHOTONS,
                       "kernel_ms_under_ncu": m["gpu__time_duration.sum"] / 1e6}
    out["source"][w] = f"profiles/r2_ncu_traffic_{w}.csv"
json.dump(out, open(sys.argv[2] if len(sys.argv) > 2 else "profiles/roofline_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
