"""Test configuration.

Markers: `gpu` = needs a CUDA device (run on the B200 with -m gpu); everything
else runs on CPU. The oracle package (oracle/) is the checker for both."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1711_03244_b200", "lib", "libvoxmc_b200.so")
    if not os.path.exists(lib):
        from paper_1711_03244_b200 import build
        build.build()
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle_c.so")) or (
            os.path.isdir("/root/reference/proj") and
            not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libvoxmc_ref.so"))):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True,
                       stdout=subprocess.DEVNULL)


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ref():
    import oracle
    return oracle.ref()


@pytest.fixture(scope="session")
def corc():
    import oracle
    return oracle.corc()


@pytest.fixture(scope="session")
def gpu():
    import paper_1711_03244_b200 as v
    n = v.device_count()
    if n < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 (there is no CPU fallback)")
    return v
