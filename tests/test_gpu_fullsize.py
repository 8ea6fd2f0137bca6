"""Size-independent properties at the bench's full size: 3D m = 3,
512 x 512 x 256 cells (128 GiB of state, the BASELINE workload on one B200),
checked with the on-device accessors only (no 128 GiB download).

* accuracy: the periodic standing mode p = cos(wt t) sin(pi x) sin(pi y)
  sin(2 pi z) (the z extent is 1) after 6 steps matches the exact jets at
  roundoff / truncation level;
* time reversal (tests/test_stepper1d.cpp:276-299): 4 steps forward, 4 back
  with dt -> -dt return the initial state."""
import math

import pytest

import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu

K = (512, 512, 256)


W = (math.pi, math.pi, 2 * math.pi)  # periodic on [-1, 1] x [-1, 1] x [-1, 0]
WT = math.sqrt(sum(w * w for w in W))


def vel_phase(c):
    return [math.pi / 2 if a == c - 1 else 0.0 for a in range(3)]


def mode_stepper():
    import torch

    free, _ = torch.cuda.mem_get_info()
    if free < 140 * 2 ** 30:
        pytest.skip("needs ~140 GiB of free device memory")
    d, m = 3, 3
    h = 2.0 / K[0]
    g = H.Stepper(H.Grid([-1.0] * d, h, K), m)
    assert g.kernel_variant == 1
    dt = 0.9 * h / math.sqrt(d)
    g.fill_separable(0, 1.0, list(W), [0.0] * d)
    # v_c = -(w_c / wt) sin(wt t) cos(w_c x_c) prod_{a != c} sin(w_a x_a), at t = dt / 2
    for c in range(1, d + 1):
        g.fill_separable(c, -W[c - 1] / WT * math.sin(WT * dt / 2), list(W), vel_phase(c))
    g.set_times(0.0, dt / 2, dt)
    return g, dt


def test_fullsize_mode_accuracy():
    g, dt = mode_stepper()
    try:
        g.advance_n(6)
        t_p, t_v, _ = g.times()
        rms, mx = g.error_separable(0, math.cos(WT * t_p), list(W), [0.0] * 3)
        assert rms < 1e-10 and mx < 1e-9, (rms, mx)
        for c in range(1, 4):
            rms, mx = g.error_separable(c, -W[c - 1] / WT * math.sin(WT * t_v), list(W), vel_phase(c))
            assert rms < 1e-10 and mx < 1e-9, (c, rms, mx)
    finally:
        del g


def test_fullsize_time_reversal():
    g, dt = mode_stepper()
    try:
        for i in range(4):
            g.step_system(i)
        g.dt = -dt
        for _ in range(4):
            g.advance_v()
            g.advance_p()
        _, mx = g.error_separable(0, 1.0, list(W), [0.0] * 3)
        assert mx < 1e-12, mx
        for c in range(1, 4):
            _, mx = g.error_separable(c, -W[c - 1] / WT * math.sin(WT * dt / 2), list(W), vel_phase(c))
            assert mx < 1e-12, (c, mx)
        assert abs(g.t_p) <= 1e-12
    finally:
        del g
