"""The C-ABI boundary (include/vmc.h) without a GPU: the library loads, exports
every declared entry point, the ctypes mirror matches the header layout, and
the host-only entry points (validation, quantum, partition) behave like the
reference."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1711_03244_b200 as v
from paper_1711_03244_b200 import _abi
from paper_1711_03244_b200.scene import Marshalled

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vmc.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"VMC_API\s+[\w\s\*]+?\b(vmc_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = declared_symbols()
    assert len(names) >= 17
    lib = C.CDLL(v.runtime.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_abi.EXPORTS) == names
    nm = subprocess.run(["nm", "-D", "--defined-only", v.runtime.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (vmc_\w+)", nm))
    assert exported == set(names), exported ^ set(names)


def test_struct_layout_matches_header(tmp_path):
    structs = {"vmc_scene": _abi.vmc_scene, "vmc_config": _abi.vmc_config,
               "vmc_disposition": _abi.vmc_disposition, "vmc_device_profile": _abi.vmc_device_profile,
               "vmc_photon_trace": _abi.vmc_photon_trace, "vmc_det_record_head": _abi.vmc_det_record_head}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if l)
    for name, cls in structs.items():
        assert int(out[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(out[f"{name}.{f}"]) == getattr(cls, f).offset, f"{name}.{f}"


def test_abi_version_and_no_device_here():
    lib = v.lib()
    assert lib.vmc_abi_version() == _abi.VMC_ABI_VERSION
    assert lib.vmc_device_count() >= 0


def test_quantum_matches_reference(ref):
    for n in [1, 7, 100_000, 10**6, 10**8, 10**9, 2**63]:
        assert v.quantum_for(n) == ref.quantum_for(n)


def test_det_record_bytes():
    lib = v.lib()
    for nm in [1, 2, 3, 6, 9]:
        assert lib.vmc_det_record_bytes(nm) == _abi.det_record_bytes(nm)
        assert _abi.det_record_dtype(nm).itemsize == _abi.det_record_bytes(nm)


def _validate(scene, cfg):
    m = Marshalled(scene, cfg)
    rc = v.lib().vmc_validate(C.byref(m.scene), C.byref(m.config))
    return rc, (v.lib().vmc_last_error() or b"").decode()


def test_validation_mirrors_reference():
    st = v.baseline_setup("b1", photons=10)
    assert _validate(st.scene, st.config)[0] == 0
    # SimulationConfig::validate (types.cpp:44-52)
    for field, bad in [("tmax_ns", 0.0), ("roulette_threshold", 1.0), ("roulette_multiplier", 1),
                       ("ngates", 0)]:
        cfg = v.baseline_setup("b1", photons=10).config
        setattr(cfg, field, bad)
        rc, msg = _validate(st.scene, cfg)
        assert rc == _abi.VMC_ERR_VALIDATION, field
    # launch outside the grid (transport.cpp:96-99, test_transport.cpp:77-84)
    bad = v.Scene(st.grid, v.Source((70.0, 30.0, 30.0), (0.0, 0.0, 1.0)))
    rc, msg = _validate(bad, st.config)
    assert rc == _abi.VMC_ERR_VALIDATION and "outside" in msg
    # pencil pointing out of the entry face
    bad = v.Scene(st.grid, v.Source((30.0, 30.0, 0.0), (0.0, 0.0, -1.0)))
    assert _validate(bad, st.config)[0] == _abi.VMC_ERR_VALIDATION
    # labels beyond the media table
    labels = st.grid.labels.copy()
    m = Marshalled(st.scene, st.config)
    labels[5] = 9
    m.scene.labels = labels.ctypes.data_as(C.POINTER(C.c_uint8))
    assert v.lib().vmc_validate(C.byref(m.scene), C.byref(m.config)) == _abi.VMC_ERR_VALIDATION
    # detector count above the kernel's table
    cfg = v.baseline_setup("b3", photons=10).config
    cfg.detectors = cfg.detectors * 5
    assert _validate(v.baseline_setup("b3").scene, cfg)[0] == _abi.VMC_ERR_VALIDATION


def test_host_grid_validation():
    with pytest.raises(v.ValidationError):
        v.VoxelGrid((0, 1, 1), 1.0, [], [v.OpticalProperties()])
    with pytest.raises(v.ValidationError):
        v.VoxelGrid((1, 1, 1), 1.0, [2], [v.OpticalProperties(), v.OpticalProperties()])
    with pytest.raises(v.ValidationError):
        v.VoxelGrid((1, 1, 1), 1.0, [0], [v.OpticalProperties(n=0.5)])
    with pytest.raises(v.ValidationError):
        v.VoxelGrid((2, 1, 1), 1.0, [0], [v.OpticalProperties()])


def test_compute_fails_loudly_without_gpu():
    if v.device_count() > 0:
        pytest.skip("GPU present")
    st = v.baseline_setup("b1", photons=100)
    with pytest.raises(RuntimeError):
        v.run_group_dynamic(0, 100, 1, st.scene, st.config)
    with pytest.raises(RuntimeError):
        v.rng_kat(1, 2, 3)


def test_kernel_names_demangle():
    """Plan.kernel names: the large-run K1f keeps k_flight<Real,G,D,T,U,Dep>, the
    small-run instantiation shows its trailing kSolo = 1."""
    from paper_1711_03244_b200.runtime import demangle_kernel as d
    assert d("_ZN3vmc8k_flightIfLb0ELb1ELb0ELb0ELi0ELb0EEEvNS_10KernelArgsE") == "k_flight<float,0,1,0,0,0>"
    assert d("_ZN3vmc8k_flightIfLb0ELb1ELb0ELb0ELi0ELb1EEEvNS_10KernelArgsE") == "k_flight<float,0,1,0,0,0,1>"
    assert d("_ZN3vmc8k_flightIdLb1ELb0ELb0ELb1ELi0ELb0EEEvNS_10KernelArgsE") == "k_flight<double,1,0,0,1,0>"
    assert d("_ZN3vmc11k_transportIfLb0ELb1ELb0ELb0EEEvNS_10KernelArgsE") == "k_transport<float,0,1,0,0>"
