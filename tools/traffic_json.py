"""Build profiles/roofline_traffic.json from gpurun_out/traffic_<w>.csv (tools/gpu_traffic.sh).
usage: python tools/traffic_json.py [out.json]"""
import csv, io, json, sys
PHOTONS = 1e8
out = {"note": "per transport-kernel launch at the bench size (1e8 photons), ncu --metrics ... --clock-control none "
               "(tools/gpu_traffic.sh); traffic = dram__bytes_read.sum + dram__bytes_write.sum", "issue": {}}
for w in ("b1", "b2", "b3", "head"):
    rows = [r for r in csv.reader(io.StringIO(open(f"gpurun_out/traffic_{w}.csv").read())) if len(r) > 10]
    hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
    m = {r[ix["Metric Name"]]: float(r[ix["Metric Value"]].replace(",", "")) for r in rows[1:]}
    kern = rows[1][ix["Kernel Name"]]
    out[w] = int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    ipc = m["sm__inst_executed.avg.per_cycle_active"]
    out["issue"][w] = {"kernel": kern, "ipc_active": ipc, "peak_ipc": 4.0, "frac": ipc / 4.0,
                       "simt": m["smsp__thread_inst_executed_per_inst_executed.ratio"] / 32,
                       "warp_inst_per_photon": m["smsp__inst_executed.sum"] / PHOTONS,
                       "l2_red_requests_per_photon": m["lts__t_requests_op_red.sum"] / PHOTONS,
                       "kernel_ms_under_ncu": m["gpu__time_duration.sum"] / 1e6}
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "profiles/roofline_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
