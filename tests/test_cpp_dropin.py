"""The C++ drop-ins (include/hlf/b200/stepper1d.hpp, stepper2d.hpp) driven by
the reference's own Stepper1d test cases (tests/cpp/test_b200_stepper1d.cpp)
and by the stepper2d module's checks over the reference's 2D types
(tests/cpp/test_b200_stepper2d.cpp), on the GPU."""
import os
import subprocess

import pytest

import oracle as O

EXE = os.path.join(O.HERE, "_ref", "test_b200_stepper1d")
EXE2D = os.path.join(O.HERE, "_ref", "test_b200_stepper2d")
EXESLABS = os.path.join(O.HERE, "_ref", "test_b200_slabs")


@pytest.mark.gpu
def test_cpp_dropin_stepper1d_suite():
    if not os.path.exists(EXE):
        pytest.skip("drop-in test binary not built (needs /root/reference at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout


def test_cpp_dropin_rejects_unsupported_features_without_gpu():
    # the configuration checks run before any device call
    if not os.path.exists(EXE):
        pytest.skip("drop-in test binary not built")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert "unsupported problem features" not in r.stderr


@pytest.mark.gpu
def test_cpp_dropin_stepper2d_suite():
    if not os.path.exists(EXE2D):
        pytest.skip("2D drop-in test binary not built (needs /root/reference at build time)")
    r = subprocess.run([EXE2D], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_host_slab_group():
    # the multi-GPU z-slab path driven from C++ through the C-ABI only
    if not os.path.exists(EXESLABS):
        pytest.skip("slab-group test binary not built")
    r = subprocess.run([EXESLABS], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout
