"""The stepping API at the drop-in boundary, on the GPU: advance-to-T and the
non-finite flag.

* advance_to(T) is the reference's caller loop (tests/test_stepper1d.cpp:29-41:
  n = step_count(T, dt_nominal), dt = T / n, init_leapfrog(dt), n x
  step_system): it must land on the same state, time stamps and step count as
  the compiled reference running that loop, continue from the current t_p,
  run backwards with a negative dt, and refuse a dt that does not divide the
  remaining time.
* check_finite (stepper1d.cpp:121-129) looks only at the current state: after
  an InstabilityError a re-initialised state must step without a stale error
  (hlf_step / hlf_advance_n reset the device flag)."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu


def rel_err(got, ref):
    scale = np.abs(ref).max()
    return np.abs(got - ref).max() / (scale if scale > 0 else 1.0)


def ref_and_gpu(problem, m, K, T, cfl=0.9):
    r = O.RefStepper1d(problem, m, K)
    n, dt = H.plan_steps(T, H.SchemeConfig(m=m, cfl=cfl).dt_nominal_1d(r.h, r.c_max))
    r.init_leapfrog(dt)
    p, v, times = r.get()
    g = H.Stepper1d(H.Grid1d.over(r.x_min, r.x_max, K), m)
    g.set_field(0, p)
    g.set_field(1, v)
    g.set_times(*times)
    return r, g, n, dt


@pytest.mark.parametrize("m,K", [(2, 20), (3, 256), (1, 40)])
def test_advance_to_is_the_reference_caller_loop(have_ref, m, K):
    if not have_ref:
        pytest.skip("compiled reference (oracle/_ref) not built")
    T = 4.13 if m == 2 else 1.0
    r, g, n, dt = ref_and_gpu("standing-wave", m, K, T)
    assert g.advance_to(T) == n
    assert r.steps(n) == -1
    p, v, times = r.get()
    assert g.times() == times
    assert rel_err(g.get_field(0), p) <= 1e-12
    assert rel_err(g.get_field(1), v) <= 1e-12
    assert abs(g.t_p - T) <= 1e-12 * T


def test_advance_to_continues_from_t_p_and_runs_backwards(have_ref):
    if not have_ref:
        pytest.skip("compiled reference (oracle/_ref) not built")
    m, K, T = 2, 40, 2.0
    r, g, n, dt = ref_and_gpu("standing-wave", m, K, T)
    half = n // 2
    T1 = half * dt
    assert g.advance_to(T1, first_step=0) == half
    assert g.advance_to(T, first_step=half) == n - half
    r.steps(n)
    p, v, times = r.get()
    assert rel_err(g.get_field(0), p) <= 1e-12
    # a negative dt runs backwards in time (test_stepper1d.cpp:288 sets
    # st.dt = -dt); advance_to counts the steps towards an earlier T
    g.dt = -dt
    assert g.advance_to(T1, first_step=n) == n - half
    assert abs(g.t_p - T1) <= 1e-12
    with pytest.raises(H.ConfigError):
        g.advance_to(T)  # ahead of t_p for a negative dt


def test_advance_to_rejects_a_dt_that_does_not_divide():
    g = H.Stepper1d(H.Grid1d.over(-1.0, 1.0, 16), 2)
    g.zero_field(0)
    g.zero_field(1)
    g.set_times(0.0, 0.05, 0.1)
    with pytest.raises(H.ConfigError):
        g.advance_to(0.25)
    with pytest.raises(H.ConfigError):
        g.advance_to(-1.0)  # behind t_p for a positive dt
    assert g.advance_to(0.3) == 3


@pytest.mark.parametrize("d", [1, 3])
def test_instability_flag_is_not_sticky(d):
    # blow up, re-initialise, step again: no stale InstabilityError
    K = 16 if d == 1 else 8
    m = 2
    grid = H.Grid([-1.0] * d, 2.0 / K, (K,) * d)
    g = H.Stepper(grid, m)
    pi = math.pi

    def init(dt):
        for f in range(d + 1):
            g.zero_field(f)
        g.fill_separable(0, 1.0, [pi] * d, [0.0] * d)
        g.set_times(0.0, dt / 2, dt)

    init(3.0 * grid.h)
    with pytest.raises(H.InstabilityError) as ei:
        g.advance_n(4000, 7)
    assert ei.value.step >= 7
    init(0.2 * grid.h)
    g.advance_n(5, 0)        # hlf_advance_n starts from a clean flag
    g.step_system(5)         # and so does hlf_step
    assert g.poll_finite() == -1
