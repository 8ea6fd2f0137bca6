"""CPU-side checks of the product library and its host mirror: the C-ABI
library loads and exports every entry point include/hlf_b200.h declares, the
host operator builder matches the reference, and configuration errors follow
the reference's exception mapping (no compute without a GPU)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1808_10481_b200 as H
from paper_1808_10481_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "hlf_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(hlf_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.hlf_abi_version() == 1


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.parametrize("m", range(9))
def test_interp_operator_matches_fixture(golden, m):
    op = H.build_interp_operator(m)
    assert op.n == 2 * m + 2
    ref = np.array(golden["M"][str(m)]["M"]).reshape(op.n, op.n)
    # same Gauss-Jordan elimination as the shimmed reference: bit-identical
    assert np.array_equal(op.M, ref)
    assert op.condition == pytest.approx(golden["M"][str(m)]["condition"], rel=1e-12)


def test_interp_operator_order_zero_by_hand():
    # test_interpolation.cpp:28-43
    op = H.build_interp_operator(0)
    assert op.M.ravel().tolist() == [0.5, 0.5, -1.0, 1.0]


def test_interp_operator_bad_order():
    for m in (-1, 9):
        with pytest.raises(H.ConfigError):
            H.build_interp_operator(m)


def test_parity_split_symmetry_of_M():
    # M[s][n1+l] = (-1)^{s+l} M[s][l] (xi -> -xi symmetry)
    for m in range(9):
        op = H.build_interp_operator(m)
        n1 = m + 1
        L, R = op.M[:, :n1], op.M[:, n1:]
        sgn = np.array([[(-1) ** (s + l) for l in range(n1)] for s in range(op.n)])
        assert np.abs(R - sgn * L).max() <= 1e-12 * np.abs(op.M).max()


def test_scheme_config_guards():
    # test_jet.cpp:166-187
    cfg = H.SchemeConfig(m=3, cfl=0.9)
    cfg.validate()
    for m in (9, -1):
        with pytest.raises(H.ConfigError):
            H.SchemeConfig(m=m).validate()
    H.SchemeConfig(m=8).validate()
    for cfl in (0.0, -0.5, float("nan")):
        with pytest.raises(H.ConfigError):
            H.SchemeConfig(m=3, cfl=cfl).validate()
    assert H.step_count(1.0, 0.3) == 4
    assert H.step_count(1.2, 0.3) == 4
    with pytest.raises(H.ConfigError):
        H.step_count(-1.0, 0.3)
    assert cfg.dt_nominal_2d(0.1, 1.0) == pytest.approx(0.9 * 0.1 / np.sqrt(2.0))


def test_grid_guards():
    g = H.Grid1d.over(-1.0, 1.0, 8)
    assert g.h == 0.25 and g.K == (8,)
    with pytest.raises(H.ConfigError):
        H.Grid1d.over(-1.0, 1.0, 1)
    with pytest.raises(H.ConfigError):
        H.Grid1d.over(1.0, -1.0, 4)
    with pytest.raises(H.ConfigError):
        H.Grid.over([0, 0], [1, 2], [4, 4])  # non-square (grid.cpp:25-26)


def test_create_rejects_bad_configs_before_touching_the_device():
    g = H.Grid1d.over(-1.0, 1.0, 8)
    with pytest.raises(H.ConfigError):
        H.Stepper(g, 9)
    desc = _lib.HlfDesc()
    desc.dim = 3
    desc.m = 5
    desc.K[:] = [4, 4, 4]
    desc.h = 0.5
    h = ctypes.c_void_p()
    assert _lib.lib().hlf_create(ctypes.byref(desc), ctypes.byref(h)) == _lib.HLF_CONFIG_ERROR
    assert b"m <= 4" in _lib.lib().hlf_last_error(None)
    desc.dim = 4
    assert _lib.lib().hlf_create(ctypes.byref(desc), ctypes.byref(h)) == _lib.HLF_CONFIG_ERROR


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.CudaError):
        H.Stepper(H.Grid1d.over(-1.0, 1.0, 8), 2)


def test_missing_extension_fails_loudly(tmp_path):
    # no CPU fallback: without the CUDA library the product path raises
    import subprocess
    import sys
    code = ("import paper_1808_10481_b200 as H\n"
            "H.Stepper(H.Grid1d.over(-1.0, 1.0, 8), 2)\n")
    env = dict(os.environ, HLF_B200_LIB_OVERRIDE=str(tmp_path / "absent.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=300)
    assert r.returncode != 0
    assert "absent.so" in r.stderr and "missing" in r.stderr


@pytest.mark.parametrize("T,dtn", [(1.0, 0.9 * 2.0 / 256), (4.13, 0.9 * 2.0 / 20), (3.2, 0.07), (0.5, 0.5)])
def test_plan_steps_is_the_reference_caller_rule(T, dtn):
    # step_count (config.cpp:34-38) and dt = T / n (tests/test_stepper1d.cpp:33-35)
    n, dt = H.plan_steps(T, dtn)
    assert n == math.ceil(T / dtn)
    assert dt == T / n
    if O.ref_available():
        assert n == O.ref_step_count(T, dtn)


def test_plan_steps_guards():
    with pytest.raises(H.ConfigError):
        H.plan_steps(0.0, 0.1)
    with pytest.raises(H.ConfigError):
        H.plan_steps(1.0, -0.1)
