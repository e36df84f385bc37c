#!/usr/bin/env python
"""bench.py — photons/ms of the B200 voxel Monte Carlo hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload b2] [--photons P]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference        # the reference's own CPU path (oracle/_ref)

A step = one pass of the hot path over one batch: P photons per GPU through
the persistent transport kernel into the int64 fluence map (zeroed in the
step), plus, for N > 1, the NCCL reduce of the maps and dispositions onto rank
0 (the reference's run_multi_device merge, scheduler.cpp:444). Weak scaling:
each rank simulates its own contiguous photon range of the global index space
[0, N*P) (quantum of the global count). Default workload: BASELINE.json
configs[1] ("B2": cube60, Fresnel reflection at the mismatched boundary,
1e8 photons, 1 gate).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic work per photon (counted from the reference
# source: add/sub/mul/div/min = 1 FLOP, FMA-able pair = 2; transcendentals extra).
FLOP_PER_PHOTON = {"b1": 12.7e3, "b2": 20.0e3, "b3": 22.9e3, "head": 99.0e3}
ATOMICS_PER_PHOTON = {"b1": 120.7, "b2": 189.0, "b3": 187.8, "head": 169.3}
DEFAULT_PHOTONS = {"b1": 100_000_000, "b2": 100_000_000, "b3": 100_000_000, "head": 100_000_000}
WORKLOAD_DESC = {
    "b1": "B1 cube60 homogeneous, pencil, terminate at boundary",
    "b2": "B2 cube60 with refractive-index mismatch (Fresnel reflection on), 1 time gate",
    "b3": "B3 cube60 + 15 mm sphere inclusion, reflect, 4 disk detectors",
    "head": "head-like 256^3 5-label volume, reflect, 10 time gates x 0.5 ns",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="b2", choices=sorted(FLOP_PER_PHOTON))
    ap.add_argument("--photons", type=int, default=0, help="photons per GPU per step")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo only for plumbing tests)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
def cpu_reference_rate(workload: str, seconds: float, seed: int, threads: int):
    """The compiled reference (oracle/_ref: run_group_dynamic, all host threads)
    on a bounded sample of the same workload. Returns (photons/ms, sample desc)."""
    import oracle
    import paper_1711_03244_b200 as v
    R = oracle.ref()
    head_n = 256
    st = v.baseline_setup(workload, photons=DEFAULT_PHOTONS[workload], seed=seed, head_n=head_n)
    # run_group_dynamic has no gates/detectors; the CW walk is the same work
    st.config.detectors = []
    st.config.ngates = 1
    n = 2_000 if workload == "head" else 20_000
    t0 = time.perf_counter()
    R.run_group(st.scene, st.config, 0, n, threads, want_cells=False)
    dt = time.perf_counter() - t0
    n2 = max(n, int(n * seconds / max(dt, 1e-3)))
    _, _, wall_ms = R.run_group(st.scene, st.config, 0, n2, threads, want_cells=False)
    return n2 / wall_ms, f"{n2} photons of {workload} [0,{n2}) seed {seed}, run_group_dynamic, {threads} threads"


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        rate, sample = cpu_reference_rate(args.workload, max(2.0, args.cpu_seconds / 3), args.seed, threads)
        if i >= args.warmup:
            vals.append(rate)
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": "photons/ms", "value": v, "unit": "photons/ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.workload], "photons_per_step": "bounded CPU sample"},
        "cpu_baseline": {"value": v, "unit": "photons/ms", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "photons/ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_b200(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_1711_03244_b200 as v
    from paper_1711_03244_b200.distributed import rank_ranges, reduce_to_root, run_group_distributed

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    per_gpu = args.photons or DEFAULT_PHOTONS[args.workload]
    total = per_gpu * world
    st = v.baseline_setup(args.workload, photons=total, seed=args.seed)
    cfg = st.config
    # contiguous range of this rank (partition_s1 over identical GPUs)
    first, mine = rank_ranges(total, world)[rank]

    plan = v.Plan(st.scene, cfg, local_rank)
    cells = torch.zeros(plan.ncells, dtype=torch.int64, device=dev)
    totals = torch.zeros(4, dtype=torch.int64, device=dev)
    det = det_n = None
    if cfg.detectors:
        det = torch.zeros(max(1, cfg.det_capacity) * plan.rec_bytes, dtype=torch.uint8, device=dev)
        det_n = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step(k_ev=None):
        if k_ev is not None:
            k_ev[0].record(stream)
        plan.run_torch(first, mine, cells, totals, det, det_n, stream=stream, zero=True)
        if k_ev is not None:
            k_ev[1].record(stream)
        if world > 1:  # the one exchange step: int64 map + dispositions onto rank 0
            reduce_to_root(cells, totals)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # correctness guard on the warm-up result: energy audit (config.cpp:316-319)
    tq = totals.cpu().tolist()
    if rank == 0:
        q = v.quantum_for(total)
        resid = (sum(tq) * q - (total if world > 1 else mine)) / (total if world > 1 else mine)
        if abs(resid) > 1e-6:
            raise RuntimeError(f"energy audit failed: residual {resid}")

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush between timed steps (outside the step events)
            evs[i][0].record(stream)
            step(kevs[i])
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    kern_ms = [a.elapsed_time(b) for a, b in kevs]
    t_local = sum(step_ms)
    t = torch.tensor([t_local, sum(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms, kern_total = float(t[0]), float(t[1])
    ms_per_step = t_ms / args.steps
    value = total / ms_per_step  # whole-job photons per ms

    # ---- end to end through the reference-facing C-ABI call (host buffers) ----
    e2e = None
    if args.e2e_steps > 0:
        ecfg = v.baseline_setup(args.workload, photons=total, seed=args.seed).config
        # pinned host outputs, allocated once (the step's D2H reads land here)
        pinned_cells = torch.empty(plan.ncells, dtype=torch.int64, pin_memory=True).numpy()
        pinned_det = None
        if ecfg.detectors:
            raw = torch.empty(max(1, ecfg.det_capacity) * plan.rec_bytes, dtype=torch.uint8, pin_memory=True)
            pinned_det = raw.numpy().view(v.runtime._abi.det_record_dtype(plan.nmedia))
        times = []
        eclocks = ClockSampler(local_rank)
        eclocks.__enter__()
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if world == 1:  # the reference-facing C-ABI call (vmc_run_range), host buffers
                res = v.run_group_dynamic(first, mine, 1, st.scene, ecfg, device=local_rank,
                                          cells_out=pinned_cells, det_out=pinned_det)
            else:  # per rank: scene upload + transport, NCCL reduce, merged map to rank-0 host
                run_group_distributed(st.scene, ecfg, total, device=local_rank, cells_out=pinned_cells)
            t1 = time.perf_counter()
            if i > 0:
                times.append(t1 - t0)
            if os.environ.get("BENCH_DEBUG"):
                print(f"[bench] e2e call {i}: {(t1 - t0) * 1e3:.2f} ms", file=sys.stderr, flush=True)
        eclocks.__exit__()
        tt = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nm = len(st.grid.media)
        h2d = (st.grid.voxel_count + nm * 4 * 8 + len(ecfg.detectors) * 32) * world  # scene, every rank
        if world == 1:
            d2h = plan.ncells * 8 + 4 * 8 + (min(res.det_count, ecfg.det_capacity) * plan.rec_bytes
                                             if ecfg.detectors else 0)
        else:
            d2h = plan.ncells * 8 + 4 * 8  # merged map + dispositions on rank 0
        e2e = {"value": total / (float(tt[0]) * 1e3), "unit": "photons/ms", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "clocks": eclocks.summary(),
               "path": ("run_group_dynamic -> vmc_run_range (scene upload, kernel, map + records download into pinned "
                        "host buffers), wall clock" if world == 1 else
                        "distributed.run_group_distributed per rank (scene upload, kernel, NCCL reduce, merged map "
                        "download to rank-0 pinned host buffer), wall clock, max over ranks")}

    if rank != 0:
        return
    peaks = measured_peaks()
    csum = clocks.summary()
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    max_mhz = csum.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    fp32_peak = sms * 128 * 2 * max_mhz * 1e6 / 1e12  # TFLOP/s (no FP32 peak in MEASURED_PEAKS.json)
    kern_ms_per = kern_total / args.steps
    achieved = FLOP_PER_PHOTON[args.workload] * mine / (kern_ms_per * 1e-3) / 1e12
    roof = {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": achieved / fp32_peak, "traffic": None,
            "kernel": ("k_transport<float>" if os.environ.get("VMC_KERNEL") == "step" else "k_flight<float>"), "kernel_ms": kern_ms_per,
            "flop_per_photon": FLOP_PER_PHOTON[args.workload],
            "peak_basis": f"{sms} SMs x 128 FP32 lanes x 2 x {max_mhz:.0f} MHz (SIMT FP32; neither HBM nor tensor bound)",
            "l2_atomics_per_s": ATOMICS_PER_PHOTON[args.workload] * mine / (kern_ms_per * 1e-3)}
    # secondary: the HBM roofline the contract names, to show it does not bound
    # this kernel (algorithmic bytes = labels + media + fluence map, read once)
    alg_bytes = st.grid.voxel_count + len(st.grid.media) * 64 + plan.ncells * 8
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof["secondary"] = {"hbm": {"achieved": alg_bytes / (kern_ms_per * 1e-3) / 1e9, "peak": hbm_peak,
                                 "unit": "GB/s", "frac": alg_bytes / (kern_ms_per * 1e-3) / 1e9 / hbm_peak,
                                 "algorithmic_bytes": alg_bytes,
                                 "peak_basis": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}}
    # secondary: L2 atomics. Deposits per second (SURVEY §8(d) runs/photon) against the
    # measured red.global.add.u64 rate of the B1 deposit-address distribution into 8
    # replicas (tools/atomics_roofline.py; uniform addresses for the head map)
    aprof = os.path.join(ROOT, "profiles", "r1_atomics_roofline.json")
    if os.path.exists(aprof):
        try:
            with open(aprof) as f:
                aj = json.load(f)
            key = "uniform" if args.workload == "head" else "replay_rep8"
            rate = roof["l2_atomics_per_s"]
            roof["secondary"]["l2_atomics"] = {
                "achieved": rate, "peak": aj[key], "unit": "red.add.u64/s", "frac": rate / aj[key],
                "peak_basis": f"profiles/r1_atomics_roofline.json[{key}] (lib/atomics_bench, same B200 model)"}
        except Exception:
            pass
    prof = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            roof["traffic"] = pj.get(args.workload)
            # issue-slot roofline of the same kernel (what actually bounds it):
            # ncu IPC vs the 4 warp-instructions/cycle/SM issue peak, plus SIMT lanes
            if args.workload in pj.get("issue", {}):
                roof["secondary"]["issue"] = dict(pj["issue"][args.workload],
                                                  source="profiles/r1_ncu_traffic_%s.csv" % args.workload)
        except Exception:
            pass
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, sample = cpu_reference_rate(args.workload, args.cpu_seconds, args.seed, threads)
        cpu = {"value": rate, "unit": "photons/ms", "cores": threads, "kind": "reference", "sample": sample}
    line = {
        "metric": "photons/ms", "value": value, "unit": "photons/ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.workload], "photons_per_gpu": per_gpu,
                   "photons_total": total, "seed": args.seed, "parallelism": f"photon-split x{world}",
                   "l2": "flushed between timed steps (256 MiB write); fluence map stays L2-resident within a step",
                   "accumulator": "int64 fixed point, quantum of the global photon count"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": csum,
        "gpu_launches": args.steps * plan.launches_per_run(),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.backend == "gloo":
        # plumbing test mode: ranks may share a GPU
        import torch
        local_rank %= max(1, torch.cuda.device_count())
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
