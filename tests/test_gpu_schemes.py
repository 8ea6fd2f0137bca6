"""The reference Stepper1d's alternative time schemes on the GPU (SURVEY.md
sec. 8(f) items 2 and 4): the modified Hermite-leapfrog step (step_modified,
stepper1d.cpp:174-232) and the classic two-half-step Hermite baseline
(step_dual_hermite, stepper1d.cpp:235-272), against the compiled reference
driven through oracle/ref_capi.cpp on identical initial states.  The 1D kernels
keep the reference's operation order, so the states must agree bit for bit."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu


def _coeffs(r):
    # constant problems: ap / av jets are [c, 0, ...] at every node
    return float(r.coeff(0, False)[0][0]), float(r.coeff(1, False)[0][0])


@pytest.mark.parametrize("problem", ["standing-wave", "random-wave"])
@pytest.mark.parametrize("m", [0, 1, 2, 3, 5])
@pytest.mark.parametrize("chunk", [0, 8])  # 8: advance_n replays CUDA graphs of 8 steps
def test_modified_scheme_matches_reference(have_ref, problem, m, chunk):
    if not have_ref:
        pytest.skip("compiled reference (oracle/_ref) not built")
    K = 40
    r = O.RefStepper1d(problem, m, K)
    dt = O.ref_dt_nominal(1, 0.9, 2.0 / K, 1.0)
    r.init_modified(dt)
    (pp, vp, pd, vd), (t, dt) = r.get_modified()
    ap, av = _coeffs(r)
    g = H.Stepper(H.Grid1d.over(-1.0, 1.0, K), m, ap=ap, av=av, scheme=H.SCHEME_MODIFIED)
    g.set_graph_steps(chunk)
    for f, a in ((0, pp), (1, vd), (2, vp), (3, pd)):
        g.set_field(f, a)
    g.set_times(t, t + dt / 2, dt)
    steps = 37
    g.advance_n(steps)
    assert r.steps_modified(steps) == -1
    (pp1, vp1, pd1, vd1), (t1, _) = r.get_modified()
    for f, ref in ((0, pp1), (1, vd1), (2, vp1), (3, pd1)):
        assert np.array_equal(g.get_field(f), ref), f
    assert g.times()[0] == t1


@pytest.mark.parametrize("problem", ["standing-wave", "random-wave"])
@pytest.mark.parametrize("m", [0, 1, 2, 3, 5])
@pytest.mark.parametrize("chunk", [0, 8])  # 8: advance_n replays CUDA graphs of 8 steps
def test_dual_hermite_scheme_matches_reference(have_ref, problem, m, chunk):
    if not have_ref:
        pytest.skip("compiled reference (oracle/_ref) not built")
    K = 40
    r = O.RefStepper1d(problem, m, K)
    dt = O.ref_dt_nominal(1, 0.9, 2.0 / K, 1.0)
    r.init_dual(dt)
    (p, v), (t, dt) = r.get_dual()
    ap, av = _coeffs(r)
    g = H.Stepper(H.Grid1d.over(-1.0, 1.0, K), m, ap=ap, av=av, scheme=H.SCHEME_DUAL_HERMITE)
    g.set_graph_steps(chunk)
    g.set_field(0, p)
    g.set_field(2, v)
    g.set_times(t, t, dt)
    steps = 29
    g.advance_n(steps)
    assert r.steps_dual(steps) == -1
    (p1, v1), (t1, _) = r.get_dual()
    assert np.array_equal(g.get_field(0), p1)
    assert np.array_equal(g.get_field(2), v1)
    assert g.times()[0] == t1


def test_alternative_schemes_reject_leapfrog_half_steps_and_non_1d():
    g = H.Stepper(H.Grid1d.over(-1.0, 1.0, 16), 2, scheme=H.SCHEME_MODIFIED)
    with pytest.raises(H.ConfigError):
        g.advance_p()
    with pytest.raises(H.ConfigError):
        H.Stepper(H.Grid([-1.0] * 2, 0.25, (8, 8)), 2, scheme=H.SCHEME_MODIFIED)
    with pytest.raises(H.ConfigError):
        H.Stepper(H.Grid1d.over(-1.0, 1.0, 16), 2, boundary=[H.REFLECTIVE], scheme=H.SCHEME_DUAL_HERMITE)
