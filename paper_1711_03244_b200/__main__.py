"""Command line front door (reference proj/tools/main.cpp subcommands).

    python -m paper_1711_03244_b200 run --config cfg.json | --benchmark b1 [--photons N] [--seed S]
                                        [--strategy s1] [--devices roster.json] [--output vol.raw]
                                        [--report report.json] [--gates G] [--precision fp32|fp64]
    python -m paper_1711_03244_b200 benchmark [--photons N]   # B1/B2/B2a photons/ms table
    python -m paper_1711_03244_b200 partition --devices roster.json --photons N
    python -m paper_1711_03244_b200 calibrate --benchmark b1 [--gpu 0] [--n1 1e6 --n2 5e6] [--cache c.json]

Exit codes as the reference (main.cpp:243-252): 0 ok, 1 validation/parse error, 2 other errors.
"""
from __future__ import annotations

import argparse
import sys

from . import pipeline as P
from . import runtime as R
from .errors import ParseError, ValidationError
from .scene import Precision, benchmark_from_name, benchmark_preset


def _setup(a) -> P.RunSetup:
    if a.config:
        s = P.parse_config(a.config)
    elif a.benchmark:
        b = benchmark_from_name(a.benchmark)
        if b is None:
            raise ValidationError(f"unknown benchmark '{a.benchmark}'")
        pre = benchmark_preset(b)
        s = P.RunSetup(pre.scene, pre.config)
    else:
        raise ValidationError("need --config or --benchmark")
    if a.photons is not None:
        if a.photons < 1:
            raise ValidationError("--photons must be >= 1")
        s.config.photon_count = a.photons
    if a.seed is not None:
        s.config.master_seed = a.seed
    if getattr(a, "gates", None):
        s.config.ngates = a.gates
    if getattr(a, "precision", None):
        s.config.precision = Precision.FP64 if a.precision == "fp64" else Precision.FP32
    if a.devices:
        s.devices = P.load_roster(a.devices)
    st = R.strategy_from_name(a.strategy)
    if st is None:
        raise ValidationError("--strategy must be one of s1, s2, s3")
    s.strategy = st
    if getattr(a, "output", None):
        s.output_path = a.output
    if getattr(a, "report", None):
        s.report_path = a.report
    s.config.validate()
    return s


def cmd_run(a) -> int:
    s = _setup(a)
    r = P.run_pipeline(s)
    print(P.report_to_json(r.report))
    return 0


def cmd_benchmark(a) -> int:
    n = a.photons or 1_000_000
    print(f"{'benchmark':10s} {'photons':>12s} {'ms':>10s} {'photons/ms':>14s}")
    for name in ("B1", "B2", "B2a"):
        pre = benchmark_preset(benchmark_from_name(name))
        pre.config.photon_count = n
        pre.config.master_seed = a.seed or 0
        res = P.run_pipeline(P.RunSetup(pre.scene, pre.config))
        print(f"{name:10s} {n:12d} {res.report.makespan_ms:10.2f} {res.report.throughput_photons_per_ms:14.0f}")
    return 0


def cmd_partition(a) -> int:
    if not a.devices:
        raise ValidationError("--devices roster is required")
    devs = P.load_roster(a.devices)
    n = a.photons or 100_000_000
    for s in R.Strategy:
        p = R.make_partition(n, devs, s)
        print(f"{s.name.lower()}: counts {p.counts} model makespan {R.model_makespan(p, devs):.3f} ms")
    return 0


def cmd_calibrate(a) -> int:
    s = _setup(a)
    dev = R.DeviceProfile(name=f"gpu{a.gpu}", kind=R.DeviceKind.CudaGpu, gpu=a.gpu)
    key = P.scene_hash(s.scene, s.config)
    if a.cache:
        hit = P.cache_lookup(a.cache, dev.name, key)
        if hit:
            print(f"{dev.name}: a={hit.a:.6e} ms/photon t0={hit.t0:.3f} ms (cached)")
            return 0
    cal = R.calibrate(dev, int(a.n1), int(a.n2), s.scene, s.config)
    if a.cache:
        P.cache_store(a.cache, dev.name, key, cal)
    print(f"{dev.name}: a={cal.a:.6e} ms/photon t0={cal.t0:.3f} ms")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1711_03244_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "benchmark", "partition", "calibrate"):
        p = sub.add_parser(name)
        p.add_argument("--config")
        p.add_argument("--benchmark")
        p.add_argument("--devices")
        p.add_argument("--strategy", default="s1")
        p.add_argument("--photons", type=lambda x: int(float(x)))
        p.add_argument("--seed", type=int)
        if name == "run":
            p.add_argument("--output")
            p.add_argument("--report")
            p.add_argument("--gates", type=int)
            p.add_argument("--precision", choices=["fp32", "fp64"])
        if name == "calibrate":
            p.add_argument("--gpu", type=int, default=0)
            p.add_argument("--n1", type=float, default=1e6)
            p.add_argument("--n2", type=float, default=5e6)
            p.add_argument("--cache")
    a = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "benchmark": cmd_benchmark, "partition": cmd_partition,
                "calibrate": cmd_calibrate}[a.cmd](a)
    except (ValidationError, ParseError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except Exception as e:  # noqa: BLE001 - CLI boundary
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
