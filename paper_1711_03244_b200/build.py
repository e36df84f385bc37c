"""Build of the native library libvoxmc_b200.so (sm_100a), in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a for every .cu; the FP64 parity
instantiation of K1 is compiled with --fmad=false. Output:
paper_1711_03244_b200/lib/libvoxmc_b200.so (git-ignored, travels with gpurun).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(OUT_DIR, "libvoxmc_b200.so")

NVCC = os.environ.get("NVCC", "nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _json_include() -> str:
    """nlohmann/json (the reference's own JSON dependency) as vendored in the
    image (cudnn_frontend/thirdparty); VMC_JSON_INCLUDE overrides."""
    env = os.environ.get("VMC_JSON_INCLUDE")
    if env:
        return env
    import glob
    import site
    roots = list(site.getsitepackages()) + [os.path.dirname(os.path.dirname(os.__file__))]
    for r in roots:
        for hit in glob.glob(os.path.join(r, "**", "nlohmann", "json.hpp"), recursive=True):
            return os.path.dirname(os.path.dirname(hit))
    raise RuntimeError("nlohmann/json.hpp not found (set VMC_JSON_INCLUDE)")


# (source, object, extra flags)
UNITS = [
    ("transport_kernels.cu", "transport_f32.o", ["-DVMC_REAL=float", "-DVMC_REAL_IS_FLOAT=1"]),
    ("transport_kernels.cu", "transport_f64.o", ["-DVMC_REAL=double", "--fmad=false"]),
    ("capi.cu", "capi.o", []),
    ("partition.cpp", "partition.o", []),
    ("voxmc_api.cpp", "voxmc_api.o", []),
    ("voxmc_config.cpp", "voxmc_config.o", None),  # flags resolved at build time (JSON include)
]

HEADERS = ["transport.cuh", "flight.cuh", "rng.cuh", "partition.hpp"]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "vmc.h")]
    deps += [os.path.join(ROOT, "include", "voxmc", f) for f in os.listdir(os.path.join(ROOT, "include", "voxmc"))]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str, obj: str, extra, verbose: bool) -> None:
    srcp = os.path.join(CSRC, src)
    objp = os.path.join(OBJ_DIR, obj)
    if not _stale(objp, srcp):
        return
    if src.endswith(".cu"):
        tune = os.environ.get("VMC_NVCC_EXTRA", "").split() if obj == "transport_f32.o" else []
        cmd = [NVCC] + ARCH + COMMON + extra + tune + ["-c", srcp, "-o", objp]
    else:  # host C++ (C++20 for the drop-in API), same visibility rules
        cmd = [CXX, "-std=c++20", "-O2", "-g", "-fPIC", "-fvisibility=hidden", "-Wall",
               "-I", os.path.join(ROOT, "include"), "-I", CSRC] + extra + ["-c", srcp, "-o", objp]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    units = [(src, obj, extra if extra is not None else ["-I", _json_include()])
             for src, obj, extra in UNITS if os.path.exists(os.path.join(CSRC, src))]
    with cf.ThreadPoolExecutor(max_workers=len(units)) as ex:
        for f in [ex.submit(_compile, s, o, e, verbose) for s, o, e in units]:
            f.result()
    objs = [os.path.join(OBJ_DIR, o) for _, o, _ in units]
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", LIB] + objs + ["-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    # L2 red.add microbenchmark (bench.py's secondary atomic roofline) and the
    # red-counter probe (what ncu's L2 red request counter counts)
    for tool in ("atomics_bench", "red_counter_probe"):
        src = os.path.join(ROOT, "tools", tool + ".cu")
        exe = os.path.join(OUT_DIR, tool)
        if os.path.exists(src) and (not os.path.exists(exe) or os.path.getmtime(src) > os.path.getmtime(exe)):
            subprocess.run([NVCC] + ARCH + ["-O3", "-lineinfo", "-o", exe, src], check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
