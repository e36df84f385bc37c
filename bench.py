#!/usr/bin/env python
"""bench.py — photons/ms of the B200 voxel Monte Carlo hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload scale|b1|b2|b3|head]
                    [--photons P] [--precision fp32|fp64]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference        # the reference's own CPU path (oracle/_ref)

`--gpus N` with N > 1 outside a launcher re-executes itself under
torch.distributed.run (one rank per GPU, NCCL); it fails loudly when the box
has fewer than N GPUs.

Default workload: BASELINE.json configs[4], the one configuration its metric
("photons/ms ... at 1/2/4/8 B200") is defined on at every GPU count: BASELINE-B3
(cube60 + 15 mm sphere, Fresnel/TIR at mismatched faces, 4 disk detectors
recording partial pathlengths), 1e9 photons per step IN TOTAL, strong scaling,
S1 (equal contiguous) photon split. The N = 1 point is the same command.
`--workload b1|b2|b3|head` times the per-GPU BASELINE configs[0-3] at 1e8
photons per GPU (weak scaling).

A step = one pass of the hot path over one batch of photons: on every rank
the persistent transport kernel over its contiguous range of the global
photon index space into the int64 fluence map (zeroed in the step; quantum of
the global count), the on-device sort of its detector records by photon
index, and for N > 1 the exchange the reference's run_multi_device merge
(scheduler.cpp:395-451) does: NCCL reduce of the maps and disposition quanta
onto rank 0 and the gather of the sorted detector records to rank 0 in rank
order.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic work per photon (counted from the reference
# source: add/sub/mul/div/min = 1 FLOP, FMA-able pair = 2; transcendentals extra).
FLOP_PER_PHOTON = {"b1": 12.7e3, "b2": 20.0e3, "b3": 22.9e3, "head": 99.0e3, "scale": 22.9e3}
# distinct-voxel deposit runs per photon: the algorithmic atomics
RUNS_PER_PHOTON = {"b1": 120.7, "b2": 189.0, "b3": 187.8, "head": 169.3, "scale": 187.8}
DEFAULT_PHOTONS = {"b1": 100_000_000, "b2": 100_000_000, "b3": 100_000_000, "head": 100_000_000,
                   "scale": 1_000_000_000}
SCENE = {"b1": "b1", "b2": "b2", "b3": "b3", "head": "head", "scale": "b3"}
STRONG = {"scale"}  # total photons fixed as N grows
WORKLOAD_DESC = {
    "b1": "configs[0] B1 cube60 homogeneous, pencil, terminate at boundary (1e8 photons per GPU)",
    "b2": "configs[1] B2 cube60 with refractive-index mismatch (Fresnel reflection on), 1 time gate",
    "b3": "configs[2] B3 cube60 + 15 mm sphere inclusion, reflect, 4 disk detectors",
    "head": "configs[3] head-like 256^3 5-label volume, reflect, 10 time gates x 0.5 ns",
    "scale": ("configs[4] 1e9-photon B3 scaling sweep (cube60 + 15 mm sphere, reflect, 4 disk detectors "
              "with partial pathlengths), S1 photon split, NCCL map reduce + detector-record gather"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="scale", choices=sorted(FLOP_PER_PHOTON))
    ap.add_argument("--photons", type=int, default=0,
                    help="photons per step: in total for 'scale' (strong), per GPU otherwise (weak)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--dump", default="", help="rank 0 writes the last step's merged map, totals and "
                                               "detector records to this .npz (test hook)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo only for plumbing tests)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args) -> int:
    """--gpus N > 1 without a launcher: one rank per GPU under torch.distributed.run."""
    if args.backend == "nccl":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}", file=sys.stderr,
                  flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


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


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


# ---------------------------------------------------------------------------
def cpu_reference_rate(workload: str, seconds: float, seed: int, threads: int):
    """The compiled reference (oracle/_ref) on a bounded sample of the same
    workload, through its own front door run_pipeline (config.cpp:288-321:
    run_multi_device over one host_device(threads) worker pool, energy audit)
    when the library has it, else run_group_dynamic. Returns (photons/ms, sample
    description, reference build)."""
    import oracle
    import paper_1711_03244_b200 as v
    R = oracle.ref_best()
    st = v.baseline_setup(SCENE[workload], photons=DEFAULT_PHOTONS[workload], seed=seed)
    # the reference has no gates/detectors; the continuous-wave walk is the same work
    st.config.detectors = []
    st.config.ngates = 1
    if workload == "head":  # private maps would cost threads x 134 MB plus the merge
        st.config.accumulation_mode = v.AccumulationMode.SharedAtomic
    n = 2_000 if workload == "head" else 20_000
    timed = R.time_pipeline if R.has_pipeline else R.time_group
    dt = timed(st.scene, st.config, n, threads) / 1e3
    n2 = max(n, int(n * seconds / max(dt, 1e-3)))
    ms = timed(st.scene, st.config, n2, threads)
    how = "run_pipeline(host_device(%d)) makespan" % threads if R.has_pipeline else \
        "run_group_dynamic, %d threads" % threads
    return n2 / ms, f"{n2} photons of {workload} [0,{n2}) seed {seed}, {how}", R.build


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    sample = build = ""
    for i in range(args.warmup + args.steps):
        rate, sample, build = cpu_reference_rate(args.workload, max(2.0, args.cpu_seconds / 3), args.seed, threads)
        if i >= args.warmup:
            vals.append(rate)
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": "photons/ms", "value": v, "unit": "photons/ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong" if args.workload in STRONG else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.workload], "photons_per_step": "bounded CPU sample"},
        "cpu_baseline": {"value": v, "unit": "photons/ms", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model(), "build": build},
        "e2e": {"value": v, "unit": "photons/ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_b200(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1711_03244_b200 as v
    from paper_1711_03244_b200.distributed import (gather_records, rank_ranges, reduce_to_root,
                                                   run_group_distributed)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    strong = args.workload in STRONG
    per_step = args.photons or DEFAULT_PHOTONS[args.workload]
    total = per_step if strong else per_step * world
    st = v.baseline_setup(SCENE[args.workload], photons=total, seed=args.seed)
    cfg = st.config
    if args.precision == "fp64":
        cfg.precision = v.Precision.FP64
    # contiguous range of this rank (partition_s1 over identical GPUs)
    first, mine = rank_ranges(total, world)[rank]
    if cfg.detectors:  # room for every record of this rank (~4e-3 of B3's photons reach a detector)
        cfg.det_capacity = max(1 << 16, int(mine * 1e-2))

    plan = v.Plan(st.scene, cfg, local_rank)
    cells = torch.zeros(plan.ncells, dtype=torch.int64, device=dev)
    totals = torch.zeros(4, dtype=torch.int64, device=dev)
    det = det_n = det_sorted = gathered = None
    if cfg.detectors:
        det = torch.zeros(cfg.det_capacity * plan.rec_bytes, dtype=torch.uint8, device=dev)
        det_sorted = torch.empty_like(det)
        det_n = torch.zeros(1, dtype=torch.int64, device=dev)
        if rank == 0:
            gathered = torch.empty(cfg.det_capacity * plan.rec_bytes * world, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    state = {"recs": None, "n": 0, "n_found": 0, "launches": 0}

    def step(k_ev=None):
        if k_ev is not None:
            k_ev[0].record(stream)
        plan.run_torch(first, mine, cells, totals, det, det_n, stream=stream, zero=True)
        launches = plan.launches_per_run()
        if k_ev is not None:
            k_ev[1].record(stream)
        if world > 1:  # exchange 1: int64 map + dispositions onto rank 0
            reduce_to_root(cells, totals)
        if det is not None:  # exchange 2: sorted detector records to rank 0 in rank order
            n_found = int(det_n.item())
            n = min(n_found, cfg.det_capacity)
            plan.sort_records_torch(det, n, first, mine, det_sorted, stream=stream)
            launches += 2 if n >= 2 else 0  # key extraction + gather (the radix passes are CUB's)
            recs, counts = gather_records(det_sorted, n, plan.rec_bytes, out=gathered)
            if n_found > n:
                raise RuntimeError(f"detector capacity {cfg.det_capacity} < {n_found} records")
            state.update(recs=recs, n=sum(counts), n_found=n_found)
        state["launches"] = launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # correctness guard on the warm-up result: energy audit (config.cpp:316-319)
    if rank == 0:
        tq = totals.cpu().tolist()
        q = v.quantum_for(total)
        resid = (sum(tq) * q - total) / total
        if abs(resid) > 1e-6:
            raise RuntimeError(f"energy audit failed: residual {resid}")

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    with ClockSampler(local_rank) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush between timed steps (outside the step events)
            evs[i][0].record(stream)
            step(kevs[i])
            evs[i][1].record(stream)
            launches += state["launches"]
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    kern_ms = [a.elapsed_time(b) for a, b in kevs]
    t = torch.tensor([sum(step_ms), sum(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms, kern_total = float(t[0]), float(t[1])
    ms_per_step = t_ms / args.steps
    value = total / ms_per_step  # whole-job photons per ms

    if args.dump and rank == 0:
        recs = state["recs"]
        np.savez(args.dump, cells=cells.cpu().numpy(), totals=totals.cpu().numpy(),
                 recs=(recs.cpu().numpy() if recs is not None else np.zeros(0, np.uint8)),
                 det_count=np.array([state["n"]]))

    # ---- end to end through the public API (host buffers) ----
    e2e = None
    if args.e2e_steps > 0:
        ecfg = v.baseline_setup(SCENE[args.workload], photons=total, seed=args.seed).config
        ecfg.precision = cfg.precision
        ecfg.det_capacity = cfg.det_capacity * world
        # pinned host outputs, allocated once (the step's D2H reads land here)
        pinned_cells = torch.empty(plan.ncells, dtype=torch.int64, pin_memory=True).numpy()
        pinned_det = None
        if ecfg.detectors:
            raw = torch.empty(ecfg.det_capacity * plan.rec_bytes, dtype=torch.uint8, pin_memory=True)
            pinned_det = raw.numpy().view(v.runtime._abi.det_record_dtype(plan.nmedia))
        times = []
        nrec = 0
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
                nrec = min(res.det_count, ecfg.det_capacity) if ecfg.detectors else 0
            else:  # per rank: scene upload + transport + record sort, NCCL reduce + gather, rank-0 download
                res = run_group_distributed(st.scene, ecfg, total, device=local_rank, cells_out=pinned_cells,
                                            det_out=pinned_det)
                nrec = len(res.detections) if res.detections is not None else 0
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
        d2h = plan.ncells * 8 + 4 * 8 + nrec * plan.rec_bytes  # merged map + dispositions + records, rank 0
        e2e = {"value": total / (float(tt[0]) * 1e3), "unit": "photons/ms", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "clocks": eclocks.summary(),
               "path": ("run_group_dynamic -> vmc_run_range (scene upload, kernel, on-device record sort, map + "
                        "records download into pinned host buffers), wall clock" if world == 1 else
                        "distributed.run_group_distributed per rank (scene upload, kernel, record sort, NCCL "
                        "reduce + record gather, merged map and records downloaded to rank-0 pinned host "
                        "buffers), wall clock, max over ranks")}

    if rank != 0:
        return
    peaks = measured_peaks()
    csum = clocks.summary()
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    max_mhz = csum.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    fp64 = args.precision == "fp64"
    lanes = 64 if fp64 else 128  # FP64 issues at half the FP32 rate on B200
    peak = sms * lanes * 2 * max_mhz * 1e6 / 1e12  # TFLOP/s, nominal (not in MEASURED_PEAKS.json)
    kern_ms_per = kern_total / args.steps
    achieved = FLOP_PER_PHOTON[args.workload] * mine / (kern_ms_per * 1e-3) / 1e12
    roof = {"bound": "fp64" if fp64 else "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": None, "peak_kind": "nominal",
            "kernel": plan.kernel, "kernel_ms": kern_ms_per,
            "flop_per_photon": FLOP_PER_PHOTON[args.workload],
            "peak_basis": (f"nominal SIMT {'FP64' if fp64 else 'FP32'} peak: {sms} SMs x {lanes} lanes x 2 x "
                           f"{max_mhz:.0f} MHz (MEASURED_PEAKS.json has no SIMT figure; this kernel is neither "
                           "HBM- nor tensor-core-bound)"),
            "units_per_launch": mine}
    # secondary: the HBM roofline the contract names, to show it does not bound
    # this kernel (algorithmic bytes = labels + media + fluence map, read once)
    alg_bytes = st.grid.voxel_count + len(st.grid.media) * 64 + plan.ncells * 8
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof["secondary"] = {"hbm": {"achieved": alg_bytes / (kern_ms_per * 1e-3) / 1e9, "peak": hbm_peak,
                                 "unit": "GB/s", "frac": alg_bytes / (kern_ms_per * 1e-3) / 1e9 / hbm_peak,
                                 "algorithmic_bytes": alg_bytes,
                                 "peak_basis": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}}
    pkey = "b3" if args.workload == "scale" else args.workload
    prof = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    pj = {}
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            roof["traffic"] = pj.get(pkey)
            # issue-slot roofline of the same kernel (what actually bounds it):
            # ncu IPC vs the 4 warp-instructions/cycle/SM issue peak, plus SIMT lanes
            if pkey in pj.get("issue", {}):
                roof["secondary"]["issue"] = dict(pj["issue"][pkey], source=pj.get("source", {}).get(
                    pkey, "profiles/roofline_traffic.json"))
        except Exception:
            pass
    # secondary: L2 atomics. Lanes that issued a red.global.add.u64 per photon,
    # MEASURED by ncu (l1tex red sectors; the L2 request counter reads 1.5x that
    # on B200, profiles/README.md), at this kernel's photon rate, against the
    # measured red rate of the workload's deposit-address distribution
    # (tools/atomics_bench: the B1 deposit addresses into 8 replicas; uniform
    # addresses for the head map)
    reds = pj.get("issue", {}).get(pkey, {}).get("red_lanes_per_photon")
    rate_basis = "ncu l1tex__t_sectors_pipe_lsu_mem_global_op_red per photon (profiles/roofline_traffic.json)"
    if reds is None:
        reds, rate_basis = RUNS_PER_PHOTON[args.workload], "SURVEY §8(d) deposit runs per photon (unmeasured)"
    l2 = {"achieved": reds * mine / (kern_ms_per * 1e-3), "unit": "red.add.u64 lanes/s", "per_photon": reds,
          "achieved_basis": rate_basis}
    aprof = os.path.join(ROOT, "profiles", "r1_atomics_roofline.json")
    if os.path.exists(aprof):
        try:
            with open(aprof) as f:
                aj = json.load(f)
            key = "uniform" if args.workload == "head" else "replay_rep8"
            l2.update(peak=aj[key], frac=l2["achieved"] / aj[key],
                      peak_basis=f"profiles/r1_atomics_roofline.json[{key}] (tools/atomics_bench on a B200)")
        except Exception:
            pass
    roof["secondary"]["l2_atomics"] = l2
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, sample, build = cpu_reference_rate(args.workload, args.cpu_seconds, args.seed, threads)
        cpu = {"value": rate, "unit": "photons/ms", "cores": threads, "kind": "reference", "sample": sample,
               "cpu_model": cpu_model(), "build": build}
    line = {
        "metric": "photons/ms", "value": value, "unit": "photons/ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f64" if fp64 else "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.workload], "photons_total": total,
                   "photons_per_gpu": (f"{total // world} (S1 split)" if strong else per_step),
                   "seed": args.seed, "parallelism": f"photon-split x{world} (one rank per GPU)",
                   "exchange": ("NCCL reduce of int64 maps + dispositions to rank 0, sorted detector records "
                                "gathered to rank 0" if world > 1 else "none (1 GPU); records sorted on device"),
                   "l2": "flushed between timed steps (256 MiB write); fluence map stays L2-resident within a step",
                   "accumulator": "int64 fixed point, quantum of the global photon count",
                   "detections_per_step": state["n"] if cfg.detectors else None},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": csum,
        "gpu_launches": launches,
    }
    return line


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "b200":
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks", file=sys.stderr, flush=True)
        sys.exit(2)
    if args.backend == "gloo":
        # plumbing test mode: ranks may share a GPU
        import torch
        local_rank %= max(1, torch.cuda.device_count())
    elif world > 1:
        import torch
        if torch.cuda.device_count() < world:
            print(f"bench.py: {world} ranks need {world} GPUs, this box has {torch.cuda.device_count()}",
                  file=sys.stderr, flush=True)
            sys.exit(2)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    line = None
    try:
        line = run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
    if line is not None:  # rank 0, after every rank's teardown: the JSON line is the last stdout line
        if world > 1:
            time.sleep(0.5)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
