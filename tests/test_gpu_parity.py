"""Parity of the sm_100a kernels (through the C-ABI) against the oracle.

Bar (north star): ||gpu - cpu||_inf / ||cpu||_inf <= 1e-12 per field, FP64,
identical inputs and step counts.  1D is also checked against the compiled
reference's committed fixture (tests/golden/reference_1d.json)."""
import math

import numpy as np
import pytest

import oracle as O
import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel_err(got, ref):
    scale = np.abs(ref).max()
    return np.abs(got - ref).max() / (scale if scale > 0 else 1.0)


def make_pair(d, m, K, boundary=None, ap=-1.0, av=-1.0, variable=False, h=None, seed=0):
    K = [K] * d if not hasattr(K, "__len__") else list(K)
    boundary = boundary or [0] * d
    h = h or 2.0 / K[0]
    grid = H.Grid([-1.0] * d, h, tuple(K))
    g = H.Stepper(grid, m, boundary=boundary, ap=ap, av=av, variable_ap=variable)
    o = O.OracleStepper(d, m, K, h, boundary=boundary, ap=ap, av=av)
    rng = np.random.default_rng(seed)
    for f in range(d + 1):
        n = g.field_nodes(f)
        # decaying coefficients, like scaled jets of smooth data
        scale = 0.6 ** np.arange(g.F)
        a = rng.standard_normal((n, g.F)) * scale
        g.set_field(f, a)
        o.set_field(f, a)
    return g, o


def compare(g, o, d, tol=TOL):
    errs = []
    for f in range(d + 1):
        e = rel_err(g.get_field(f), o.get_field(f))
        errs.append(e)
        assert e <= tol, (f, e)
    assert g.times() == pytest.approx(o.get_times(), abs=0, rel=0)
    return errs


def run_both(g, o, steps, dt):
    g.set_times(0.0, dt / 2, dt)
    o.set_times(0.0, dt / 2, dt)
    g.advance_n(steps)
    assert o.advance_n(steps) == -1


def test_config1_matches_reference_fixture(golden):
    c1 = golden["config1"]
    grid = H.Grid1d.over(-1.0, 1.0, c1["K"])
    g = H.Stepper(grid, c1["m"])
    g.set_field(0, np.array(c1["p0"]))
    g.set_field(1, np.array(c1["v0"]))
    g.set_times(*c1["times0"])
    for i in range(c1["steps"]):
        g.step_system(i)
    assert g.times() == tuple(c1["times1"])
    assert rel_err(g.get_field(0).ravel(), np.array(c1["p1"])) <= TOL
    assert rel_err(g.get_field(1).ravel(), np.array(c1["v1"])) <= TOL


def test_set_get_roundtrip_is_exact():
    g, _ = make_pair(3, 2, [5, 6, 7], boundary=[1, 0, 1])
    rng = np.random.default_rng(1)
    for f in range(4):
        a = rng.standard_normal((g.field_nodes(f), g.F))
        g.set_field(f, a)
        assert np.array_equal(g.get_field(f), a)


@pytest.mark.parametrize("m", range(9))
@pytest.mark.parametrize("boundary", [0, 1])
def test_parity_1d(m, boundary):
    g, o = make_pair(1, m, 24, boundary=[boundary], seed=m)
    run_both(g, o, 30, 0.4 * g.grid.h)
    compare(g, o, 1)


@pytest.mark.parametrize("m", range(5))
@pytest.mark.parametrize("boundary", [[0, 0], [1, 1], [1, 0]])
def test_parity_2d(m, boundary):
    g, o = make_pair(2, m, [12, 10], boundary=boundary, seed=10 + m)
    run_both(g, o, 8, 0.3 * g.grid.h)
    compare(g, o, 2)


@pytest.mark.parametrize("m", range(5))
@pytest.mark.parametrize("boundary", [[0, 0, 0], [1, 1, 1], [0, 1, 0]])
def test_parity_3d_generic(m, boundary):
    K = [6, 5, 7] if m < 4 else [4, 4, 5]
    g, o = make_pair(3, m, K, boundary=boundary, seed=20 + m)
    g.kernel_variant = 0
    run_both(g, o, 3, 0.25 * g.grid.h)
    compare(g, o, 3)


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("boundary", [[0, 0, 0], [1, 1, 1], [1, 0, 0], [0, 1, 1]])
def test_parity_3d_tiled_kernel(m, boundary):
    # K crosses a partial 32-cell x tile and three 64-layer z chunks
    g, o = make_pair(3, m, [36, 2, 133], boundary=boundary, seed=40 + m)
    assert g.kernel_variant == 1
    run_both(g, o, 3, 0.25 * g.grid.h)
    compare(g, o, 3)


def test_custom_M_falls_back_to_generic_kernel():
    # the tiled kernel has M baked in; a caller-supplied M that differs must
    # still be honoured (generic kernel), matching the oracle run with that M
    m, K = 3, [18, 4, 5]
    h = 2.0 / K[0]
    M = H.build_interp_operator(m).M * (1.0 + 2.0 ** -40)
    g = H.Stepper(H.Grid([-1.0] * 3, h, tuple(K)), m, M=M)
    o = O.OracleStepper(3, m, K, h)
    o.set_M(M)
    rng = np.random.default_rng(4)
    for f in range(4):
        a = rng.standard_normal((g.field_nodes(f), g.F)) * 0.6 ** np.arange(g.F)
        g.set_field(f, a)
        o.set_field(f, a)
    run_both(g, o, 2, 0.25 * h)
    compare(g, o, 3)


def test_tiled_equals_generic_long_run():
    # the tiled kernel reorders the arithmetic (parity split, FMA); over a long
    # run the two GPU kernels differ by the reconstruction's roundoff floor only
    ga, _ = make_pair(3, 3, [32, 8, 8], seed=77)
    gb, _ = make_pair(3, 3, [32, 8, 8], seed=77)
    gb.kernel_variant = 0
    for s in (ga, gb):
        s.set_times(0, 0.02, 0.04)
        s.advance_n(50)
    for f in range(4):
        assert rel_err(ga.get_field(f), gb.get_field(f)) <= 1e-10


def c2_jets(d, K, h, n, boundary, dual):
    """ap = -c^2 with c^2 = 1 + sin(pi x) sin(pi y) / 2 (SURVEY.md sec. 8(d) cfg 3)."""
    N = [k + 1 if (b == 1 and not dual) else k for k, b in zip(K, boundary)]
    jets = np.zeros((int(np.prod(N)), n ** d))
    O.add_separable(d, N, [-1.0] * d, h, 0.5 if dual else 0.0, n, 0.5, [math.pi] * d, [0.0] * d, jets)
    jets[:, 0] += 1.0
    return -jets


@pytest.mark.parametrize("d,m,boundary", [(1, 3, [0]), (1, 2, [1]), (2, 1, [0, 0]), (2, 3, [1, 1]), (3, 1, [1, 1, 1])])
def test_parity_variable_speed(d, m, boundary):
    K = [10] * d if d < 3 else [5, 4, 6]
    g, o = make_pair(d, m, K, boundary=boundary, variable=True, seed=60 + m)
    n = 2 * m + 2
    for grid, dual in ((0, False), (1, True)):
        jets = c2_jets(d, K, g.grid.h, n, boundary, dual)
        g.set_coeff(grid, jets)
        o.set_coeff(grid, 0, jets)
    run_both(g, o, 5, 0.2 * g.grid.h)
    compare(g, o, d)


def set_both_coeff(g, o, jets_of):
    for grid, dual in ((0, False), (1, True)):
        jets = jets_of(grid, dual)
        g.set_coeff(grid, jets)
        o.set_coeff(grid, 0, jets)


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("boundary", [[0, 0], [1, 1], [1, 0]])
def test_parity_2d_variable_kernel(m, boundary):
    # var2d (per-node ap jets): K = 13 x 11 leaves a partial CTA and, at m = 2
    # and 4, idle lanes; the c^2 jets of config 3
    K = [13, 11]
    g, o = make_pair(2, m, K, boundary=boundary, variable=True, seed=80 + m)
    assert g.kernel_variant == 1
    set_both_coeff(g, o, lambda grid, dual: c2_jets(2, K, g.grid.h, 2 * m + 2, boundary, dual))
    run_both(g, o, 4, 0.2 * g.grid.h)
    compare(g, o, 2)


@pytest.mark.parametrize("m", [1, 3, 4])
def test_parity_2d_variable_kernel_random_jets(m):
    # dense random ap jets: every entry of the truncated products contributes,
    # so a wrong region (rows / columns skipped) cannot hide
    K, boundary = [9, 12], [1, 1]
    g, o = make_pair(2, m, K, boundary=boundary, variable=True, seed=90 + m)
    rng = np.random.default_rng(7 + m)
    n = 2 * m + 2

    def jets(grid, dual):
        a = rng.standard_normal((g.field_nodes(1 if dual else 0), n * n)) * 0.3
        a *= 0.7 ** np.add.outer(np.arange(n), np.arange(n)).ravel()
        a[:, 0] -= 1.0
        return a

    set_both_coeff(g, o, jets)
    run_both(g, o, 4, 0.2 * g.grid.h)
    compare(g, o, 2)


def test_variable_kernel_equals_generic_long_run():
    # var2d reorders the arithmetic (FMA, sum/difference M, Lap instead of
    # grad-then-div); over a long run it stays at the roundoff floor of the
    # faithful generic kernel
    K, boundary, m = [70, 45], [1, 1], 3
    runs = []
    for variant in (1, 0):
        g, _ = make_pair(2, m, K, boundary=boundary, variable=True, seed=11)
        for grid, dual in ((0, False), (1, True)):
            g.set_coeff(grid, c2_jets(2, K, g.grid.h, 2 * m + 2, boundary, dual))
        g.kernel_variant = variant
        g.set_times(0.0, 0.005, 0.01)
        g.advance_n(40)
        runs.append([g.get_field(f) for f in range(3)])
    for a, b in zip(*runs):
        assert rel_err(a, b) <= 1e-10


def test_asymmetric_M_disables_fast_kernels():
    # the fast kernels apply M through its left half (the mirror symmetry of
    # A); a caller-supplied M without it must run on the generic kernel
    m, K = 2, [12, 10]
    M = H.build_interp_operator(m).M.copy()
    M[1, 2 * m + 1] *= 1.0 + 1e-9
    for variable in (False, True):
        g = H.Stepper(H.Grid([-1.0] * 2, 2.0 / K[0], tuple(K)), m, M=M, variable_ap=variable)
        assert g.kernel_variant == 0
        with pytest.raises(H.ConfigError):
            g.kernel_variant = 1


def test_1d_variable_coefficients_vs_compiled_reference():
    if not O.ref_available():
        pytest.skip("compiled reference not present")
    m, K = 3, 40
    r = O.RefStepper1d("pv", m, K)
    r.init_leapfrog(0.9 * r.h)
    p0, v0, t0 = r.get()
    g = H.Stepper(H.Grid1d.over(r.x_min, r.x_max, K), m, variable_ap=True, av=-1.0)
    g.set_coeff(0, r.coeff(0, False))
    g.set_coeff(1, r.coeff(0, True))
    g.set_field(0, p0)
    g.set_field(1, v0)
    g.set_times(*t0)
    g.advance_n(25)
    assert r.steps(25) == -1
    p1, v1, t1 = r.get()
    assert rel_err(g.get_field(0), p1) <= TOL and rel_err(g.get_field(1), v1) <= TOL
    assert g.times() == t1


def forced_run(r, g, steps):
    """advance the device solver with the reference problem's forcing tables:
    advance_p at (primary x_j, t_v), advance_v at (dual x_j, t_p after the
    pressure half step), as Stepper1d::advance_p/v (stepper1d.cpp:147-166)"""
    for _ in range(steps):
        _, t_v, _ = g.times()
        g.set_forcing(H.PRIMARY, r.forcing(False, t_v))
        g.advance_p()
        t_p, _, _ = g.times()
        g.set_forcing(H.DUAL, r.forcing(True, t_p))
        g.advance_v()


def forced_pair(m, K, dt):
    r = O.RefStepper1d("variable-speed", m, K)
    assert r.has_forcing()
    r.init_leapfrog(dt)
    p0, v0, t0 = r.get()
    g = H.Stepper(H.Grid1d.over(r.x_min, r.x_max, K), m, variable_ap=True, av=-1.0)
    g.set_coeff(0, r.coeff(0, False))
    g.set_coeff(1, r.coeff(0, True))
    g.set_field(0, p0)
    g.set_field(1, v0)
    g.set_times(*t0)
    return r, g


@pytest.mark.parametrize("m", [1, 2, 3])
def test_1d_forcing_bit_identical_to_compiled_reference(m):
    # variable_speed_problem (problems.cpp:37-61): c^2(x) jets AND a forcing
    # provider; the faithful 1D kernel with the forcing tables runs the full
    # coupled recurrence and must reproduce the reference bit for bit
    if not O.ref_available():
        pytest.skip("compiled reference not present")
    K = 32
    r, g = forced_pair(m, K, 0.9 * (2 * math.pi / K) / math.sqrt(1.5))
    forced_run(r, g, 30)
    assert r.steps(30) == -1
    p1, v1, t1 = r.get()
    assert np.array_equal(g.get_field(0), p1) and np.array_equal(g.get_field(1), v1)
    assert g.times() == t1


def test_1d_forcing_golden_convergence():
    # tests/test_stepper1d.cpp:341-353: variable speed, Hermite-leapfrog m = 2,
    # T = 3.2, cfl 0.9, L2(p) at K = 10/20/40/80 within 2 % of the pinned values
    if not O.ref_available():
        pytest.skip("compiled reference not present")
    m, T, cfl = 2, 3.2, 0.9
    expect = [5.3628e-06, 8.0000e-08, 1.2426e-09, 1.9781e-11]
    for K, e_ref in zip([10, 20, 40, 80], expect):
        h = 2 * math.pi / K
        n = math.ceil(T / (cfl * h / math.sqrt(1.5)))  # step_count (config.cpp:34-38)
        r, g = forced_pair(m, K, T / n)
        forced_run(r, g, n)
        r.set(g.get_field(0), g.get_field(1), g.times())
        assert r.l2_p() == pytest.approx(e_ref, rel=0.02), (K, r.l2_p())


def test_forcing_mode_needs_a_table_per_half_step():
    if not O.ref_available():
        pytest.skip("compiled reference not present")
    r, g = forced_pair(2, 16, 0.01)
    forced_run(r, g, 1)
    with pytest.raises(H.ConfigError):
        g.advance_p()  # no fresh table
    with pytest.raises(H.ConfigError):
        g.advance_n(2)
    g.clear_forcing()
    g.advance_n(2)
    g2 = H.Stepper(H.Grid([-1.0] * 2, 0.2, (10, 10)), 2)
    with pytest.raises(ValueError):
        g2.set_forcing(H.PRIMARY, np.zeros((100, 5, 6)))  # 2D tables hold n^2 jets
    g2.set_forcing(H.PRIMARY, np.zeros((100, 5, 36)))
    g3 = H.Stepper(H.Grid([-1.0], 0.2, (10,)), 2, scheme=H.SCHEME_MODIFIED)
    with pytest.raises(H.ConfigError):
        g3.set_forcing(H.PRIMARY, np.zeros((10, 5, 6)))  # leapfrog scheme only


@pytest.mark.parametrize("d", [1, 2, 3])
def test_time_reversal(d):
    # tests/test_stepper1d.cpp:276-299, in d dimensions
    m = 2
    g, _ = make_pair(d, m, [10] * d if d < 3 else [8, 8, 8], seed=5)
    p0 = g.get_field(0).copy()
    v0 = [g.get_field(c).copy() for c in range(1, d + 1)]
    dt = 0.07 * g.grid.h / 0.2
    g.set_times(0.0, dt / 2, dt)
    for i in range(20):
        g.step_system(i)
    g.dt = -dt
    for _ in range(20):
        g.advance_v()
        g.advance_p()
    assert rel_err(g.get_field(0), p0) <= 1e-11
    for c in range(1, d + 1):
        assert rel_err(g.get_field(c), v0[c - 1]) <= 1e-11
    assert abs(g.t_p) <= 1e-12


def test_linearity_3d():
    # tests/test_stepper1d.cpp:242-274
    m = 3
    ga, _ = make_pair(3, m, [8, 8, 8], seed=1)
    gb, _ = make_pair(3, m, [8, 8, 8], seed=2)
    gab, _ = make_pair(3, m, [8, 8, 8], seed=3)
    al, be = 0.6, -1.3
    for f in range(4):
        gab.set_field(f, al * ga.get_field(f) + be * gb.get_field(f))
    for s in (ga, gb, gab):
        s.set_times(0, 0.02, 0.04)
        s.step_system(0)
    for f in range(4):
        ref = al * ga.get_field(f) + be * gb.get_field(f)
        assert rel_err(gab.get_field(f), ref) <= 1e-12


def test_zero_stays_zero():
    g = H.Stepper(H.Grid([-1.0] * 3, 0.25, (8, 8, 8)), 3)
    g.set_times(0, 0.05, 0.1)
    g.advance_n(5)
    for f in range(4):
        assert np.abs(g.get_field(f)).max() == 0.0


def test_instability_raises_with_step_index():
    # tests/test_stepper1d.cpp:301-321: cfl 2.5 on the standing wave blows up
    golden_grid = H.Grid1d.over(-1.0, 1.0, 16)
    g = H.Stepper(golden_grid, 2)
    o = O.OracleStepper(1, 2, [16], golden_grid.h)
    p = np.zeros((16, 3))
    v = np.zeros((16, 3))
    O.add_separable(1, [16], [-1.0], golden_grid.h, 0.0, 3, 1.0, [2 * math.pi], [0.0], p)
    g.set_field(0, p)
    g.set_field(1, v)
    o.set_field(0, p)
    o.set_field(1, v)
    dt = 2.5 * golden_grid.h
    g.set_times(0, dt / 2, dt)
    o.set_times(0, dt / 2, dt)
    expected = o.advance_n(5000)
    assert expected > 0
    with pytest.raises(H.InstabilityError) as ei:
        for i in range(5000):
            g.step_system(i)
    assert ei.value.step == expected
    assert str(expected) in str(ei.value)
    # advance_n reports the same first bad step
    g2 = H.Stepper(golden_grid, 2)
    g2.set_field(0, p)
    g2.set_field(1, v)
    g2.set_times(0, dt / 2, dt)
    with pytest.raises(H.InstabilityError) as ei2:
        g2.advance_n(expected + 10)
    assert ei2.value.step == expected


@pytest.mark.parametrize("d", [1, 2, 3])
def test_fill_separable_matches_host_jets(d):
    m = 3
    K = [9, 7, 5][:d]
    grid = H.Grid([-1.0] * d, 0.3, tuple(K))
    g = H.Stepper(grid, m, boundary=[1] + [0] * (d - 1))
    w = [1.3, -0.7, 2.1][:d]
    ph = [0.2, 1.1, -0.4][:d]
    for f, off in ((0, 0.0), (1, 0.5)):
        g.fill_separable(f, 0.8, w, ph)
        ref = np.zeros((g.field_nodes(f), g.F))
        O.add_separable(d, list(g.node_shape(f)), [-1.0] * d, 0.3, off, m + 1, 0.8, w, ph, ref)
        assert np.abs(g.get_field(f) - ref).max() <= 1e-14


def test_advance_n_equals_step_loop():
    ga, _ = make_pair(2, 3, [16, 16], seed=9)
    gb, _ = make_pair(2, 3, [16, 16], seed=9)
    for s in (ga, gb):
        s.set_times(0, 0.01, 0.02)
    ga.advance_n(7, 3)
    for i in range(7):
        gb.step_system(3 + i)
    for f in range(3):
        assert np.array_equal(ga.get_field(f), gb.get_field(f))


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("m", [1, 3])
def test_z_slabs_on_one_gpu_match_single_domain(m, overlap):
    """Two z-slab solvers (z_slab=True) on one GPU, halos copied through the
    hlf_halo_send/recv_ptr device views exactly as the NCCL exchanger does;
    the result equals one periodic solver on the whole box.  With `overlap`
    the slabs advance in layer ranges in distributed.slab_step's order: the
    interior layers before the halo lands, the boundary layer after."""
    import torch
    from paper_1808_10481_b200.distributed import device_view
    K = [36, 4, 8]
    h = 2.0 / K[0]
    full = H.Stepper(H.Grid([-1.0] * 3, h, tuple(K)), m)
    kz = K[2] // 2
    slabs = [H.Stepper(H.Grid([-1.0, -1.0, -1.0 + r * kz * h], h, (K[0], K[1], kz)), m, z_slab=True)
             for r in range(2)]
    rng = np.random.default_rng(8)
    F = (m + 1) ** 3
    for f in range(4):
        a = rng.standard_normal((K[0] * K[1] * K[2], F)) * 0.6 ** np.arange(F)
        full.set_field(f, a)
        a4 = a.reshape(K[0], K[1], K[2], F)
        for r in range(2):
            slabs[r].set_field(f, a4[:, :, r * kz:(r + 1) * kz, :].reshape(-1, F))
    dt = 0.25 * h
    for s in [full] + slabs:
        s.set_times(0.0, dt / 2, dt)

    def view(s, kind, comp, send):
        ptr, cnt = s.halo_ptr(kind, comp, send)
        return device_view(ptr, cnt)

    def v_halo():  # my ghost z=-1 <- previous rank's last layer
        for s in slabs:
            s.synchronize()
        for r in range(2):
            for c in range(3):
                view(slabs[r], 1, c, False).copy_(view(slabs[(r - 1) % 2], 1, c, True))
        torch.cuda.synchronize()

    def p_halo():  # my layer Kz <- next rank's layer 0
        for s in slabs:
            s.synchronize()
        for r in range(2):
            view(slabs[r], 0, 0, False).copy_(view(slabs[(r + 1) % 2], 0, 0, True))
        torch.cuda.synchronize()

    for i in range(3):
        if overlap:
            for s in slabs:
                s.advance_layers(0, i, 1, kz)
            v_halo()
            for s in slabs:
                s.advance_layers(0, i, 0, 1)
                s.commit_half(0)
                s.advance_layers(1, i, 0, kz - 1)
            p_halo()
            for s in slabs:
                s.advance_layers(1, i, kz - 1, kz)
                s.commit_half(1)
                s.synchronize()
        else:
            v_halo()
            for s in slabs:
                s.advance_p_indexed(i)
            p_halo()
            for s in slabs:
                s.advance_v_indexed(i)
                s.synchronize()
        full.step_system(i)
    for s in slabs:
        assert s.times() == full.times()
    for f in range(4):
        ref = full.get_field(f).reshape(K[0], K[1], K[2], F)
        for r in range(2):
            got = slabs[r].get_field(f).reshape(K[0], K[1], kz, F)
            assert np.array_equal(got, ref[:, :, r * kz:(r + 1) * kz, :]), (f, r)


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("boundary", [[0, 0], [1, 1], [0, 1], [1, 0]])
def test_parity_2d_tiled_kernel(m, boundary):
    # crosses a partial 32-cell x tile and three 32-row y chunks
    g, o = make_pair(2, m, [40, 70], boundary=boundary, seed=90 + m)
    assert g.kernel_variant == 1
    run_both(g, o, 5, 0.3 * g.grid.h)
    compare(g, o, 2)


@pytest.mark.parametrize("d,m,K,boundary", [(1, 3, [256], [0]), (2, 2, [40, 33], [1, 0]), (2, 3, [20, 20], [1, 1]),
                                            (3, 3, [36, 4, 6], [0, 0, 0]), (3, 2, [8, 6, 5], [1, 1, 1])])
def test_graph_replay_is_bit_identical(d, m, K, boundary):
    # hlf_advance_n replays chunks of steps as a captured CUDA graph; the
    # fields, time stamps and launch sequence must equal direct launches
    runs = []
    for chunk in (4, 0):
        g, _ = make_pair(d, m, K, boundary=boundary, seed=31)
        g.set_graph_steps(chunk)
        dt = 0.25 * g.grid.h
        g.set_times(0.0, dt / 2, dt)
        g.advance_n(23, 5)
        g.advance_n(9, 28)  # cached graph, new step base
        runs.append(([g.get_field(f) for f in range(d + 1)], g.times()))
    (fa, ta), (fb, tb) = runs
    assert ta == tb
    for a, b in zip(fa, fb):
        assert np.array_equal(a, b)


def test_graph_replay_reports_the_first_bad_step():
    # the step index of a blow-up inside a replayed chunk (graph step base)
    grid = H.Grid1d.over(-1.0, 1.0, 16)
    p = np.zeros((16, 3))
    O.add_separable(1, [16], [-1.0], grid.h, 0.0, 3, 1.0, [2 * math.pi], [0.0], p)
    idx = []
    for chunk in (0, 4):
        g = H.Stepper(grid, 2)
        g.set_graph_steps(chunk)
        g.set_field(0, p)
        g.zero_field(1)
        dt = 2.5 * grid.h
        g.set_times(0, dt / 2, dt)
        with pytest.raises(H.InstabilityError) as ei:
            g.advance_n(5000, 3)
        idx.append(ei.value.step)
    assert idx[0] == idx[1] and idx[0] > 3
