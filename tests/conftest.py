import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def _ensure_oracle():
    so = os.path.join(ROOT, "oracle", "_build", "libhlf_oracle.so")
    fma = os.path.join(ROOT, "oracle", "_build", "libhlf_oracle_fma.so")
    if not os.path.exists(so) or not os.path.exists(fma):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    ref = os.path.join(ROOT, "oracle", "_ref", "libhlf_refc.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


_ensure_oracle()


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "reference_1d.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def have_ref():
    import oracle
    return oracle.ref_available()
