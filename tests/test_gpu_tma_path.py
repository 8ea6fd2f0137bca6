"""Oracle parity on the code path the bench runs: the TMA box loads.

The tiled kernels load a CTA's raw source rows with one TMA tensor box only
when the row needs no x wrap / mirror (pressure launches: x0 >= 2 and
x0 + 32 <= sNx, so K_x >= 64 for an interior x tile; kernels_tiled3d.cu
tma_rows, kernels_tiled2d.cu tma_rows); edge CTAs load node by node.  These
tests use grids with interior x tiles (K_x = 96: tiles at x0 = 0, 32, 64), run
>= 10 steps against the oracle at the 1e-12 bar, and read the kernels' path
counters (hlf_enable_path_counters) to prove that TMA CTAs ran in both half
steps.  The long runs (100 steps) compare the tiled
kernels' drift with the drift of the same oracle compiled with contracted FMAs
(oracle/_build/libhlf_oracle_fma.so: the identical algorithm, another valid
rounding): the GPU must stay within 1e-12, or at worst within 4x that
yardstick when the yardstick itself exceeds 2.5e-13.
Reference path: Stepper1d::advance_p / advance_v / step_system
(/root/reference/proj/src/stepper1d.cpp:147-172), generalised per SURVEY.md
App. A.3."""
import numpy as np
import pytest

import oracle as O
import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel_err(got, ref):
    scale = np.abs(ref).max()
    return np.abs(got - ref).max() / (scale if scale > 0 else 1.0)


def setup(d, m, K, boundary, seed, fma_oracle=False):
    h = 2.0 / K[0]
    grid = H.Grid([-1.0] * d, h, tuple(K))
    g = H.Stepper(grid, m, boundary=boundary)
    o = O.OracleStepper(d, m, K, h, boundary=boundary)
    of = O.OracleStepper(d, m, K, h, boundary=boundary, fma=True) if fma_oracle else None
    rng = np.random.default_rng(seed)
    for f in range(d + 1):
        a = rng.standard_normal((g.field_nodes(f), g.F)) * 0.6 ** np.arange(g.F)
        g.set_field(f, a)
        o.set_field(f, a)
        if of is not None:
            of.set_field(f, a)
    return g, o, of


def run(steppers, steps, dt, first=0):
    for s in steppers:
        if s is None:
            continue
        s.set_times(0.0, dt / 2, dt)
        r = s.advance_n(steps, first)
        if isinstance(r, int) and not isinstance(s, H.Stepper):
            assert r == -1


def assert_tma_ran(g, K, boundary):
    """TMA boxes need 16 B aligned rows: an even node count along x.  The
    primary grid has K_x + 1 nodes along a walled x axis, so with x walls one
    of the two half steps loads per node (for K_x = 96: the velocity half step
    reads p rows of 97 nodes and writes 96-node v rows; the pressure half step
    the reverse)."""
    c = g.path_counters()
    nx_primary = K[0] + (1 if boundary[0] == 1 else 0)
    nx_dual = K[0]
    expect = {"vel": (nx_primary % 2 == 0, nx_dual % 2 == 0), "pre": (nx_dual % 2 == 0, nx_primary % 2 == 0)}
    for kind in ("vel", "pre"):
        rows, tgts = expect[kind]
        assert c[kind]["ctas"] > 0, c
        if rows:
            assert c[kind]["tma_rows"] > 0, (kind, c)
        if tgts:
            assert c[kind]["tma_targets"] > 0, (kind, c)
    assert c["pre"]["tma_rows"] + c["vel"]["tma_rows"] > 0
    return c


# (boundary, K_x): with x walls an odd K_x gives the velocity half step
# aligned (K_x + 1)-node source rows instead
BND3 = [([0, 0, 0], 96), ([1, 1, 1], 96), ([1, 0, 1], 95), ([0, 1, 0], 96)]


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("boundary,kx", BND3)
def test_tma_path_3d_parity(m, boundary, kx):
    K = [kx, 6, 70]  # interior x tiles + a 64-layer z chunk boundary
    g, o, _ = setup(3, m, K, boundary, seed=300 + 7 * m)
    assert g.kernel_variant == 1
    g.enable_path_counters()
    run([g, o], 10, 0.25 * g.grid.h)
    assert_tma_ran(g, K, boundary)
    for f in range(4):
        e = rel_err(g.get_field(f), o.get_field(f))
        assert e <= TOL, (f, e)
    assert g.times() == o.get_times()


@pytest.mark.parametrize("raster", ["8", "3", "0"])
@pytest.mark.parametrize("boundary,kx", [([0, 0, 0], 96), ([1, 1, 1], 95)])
def test_tma_path_3d_raster_groups(raster, boundary, kx, monkeypatch):
    """CTA row groups (kernels_tiled3d.cu TParams.raster, default 8 at m = 3)
    with a partial last group (K_y = 13 = 8 + 5; 3 + 3 + 3 + 3 + 1) cover
    every CTA exactly once: oracle parity over 6 steps for each grouping."""
    monkeypatch.setenv("HLF_RASTER", raster)  # read by the host at every launch
    K = [kx, 13, 20]
    g, o, _ = setup(3, 3, K, boundary, seed=700 + int(raster))
    assert g.kernel_variant == 1
    run([g, o], 6, 0.25 * g.grid.h)
    for f in range(4):
        e = rel_err(g.get_field(f), o.get_field(f))
        assert e <= TOL, (raster, f, e)


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("boundary,kx", [([0, 0], 96), ([1, 1], 96), ([1, 0], 95), ([0, 1], 96)])
def test_tma_path_2d_parity(m, boundary, kx):
    K = [kx, 80]
    g, o, _ = setup(2, m, K, boundary, seed=400 + 5 * m)
    assert g.kernel_variant == 1
    g.enable_path_counters()
    run([g, o], 12, 0.3 * g.grid.h)
    assert_tma_ran(g, K, boundary)
    for f in range(3):
        e = rel_err(g.get_field(f), o.get_field(f))
        assert e <= TOL, (f, e)


def long_run_bound(yardstick: float) -> float:
    return TOL if yardstick <= 2.5e-13 else 4.0 * yardstick


@pytest.mark.parametrize("m", [1, 2, 3])
def test_tma_path_3d_long_run(m):
    # 100 steps at 3D 32^3 (x doubled to 64 so one x
    # tile is interior and takes the TMA path in both half steps)
    K = [64, 32, 32]
    g, o, of = setup(3, m, K, [0, 0, 0], seed=500 + m, fma_oracle=True)
    g.enable_path_counters()
    run([g, o, of], 100, 0.3 * g.grid.h)
    assert_tma_ran(g, K, [0, 0, 0])
    for f in range(4):
        ref = o.get_field(f)
        yard = rel_err(of.get_field(f), ref)
        e = rel_err(g.get_field(f), ref)
        assert e <= long_run_bound(yard), (f, e, yard)


@pytest.mark.parametrize("m", [1, 2, 3, 4])
def test_tma_path_2d_long_run(m):
    # 100 steps at 2D 64^2, with walls on y
    K = [64, 64]
    g, o, of = setup(2, m, K, [0, 1], seed=600 + m, fma_oracle=True)
    g.enable_path_counters()
    run([g, o, of], 100, 0.35 * g.grid.h)
    assert_tma_ran(g, K, [0, 1])
    for f in range(3):
        ref = o.get_field(f)
        yard = rel_err(of.get_field(f), ref)
        e = rel_err(g.get_field(f), ref)
        assert e <= long_run_bound(yard), (f, e, yard)


def test_path_counters_off_by_default_and_resettable():
    g, _, _ = setup(3, 3, [64, 2, 4], [0, 0, 0], seed=1)
    g.advance_n(1)
    assert g.path_counters()["vel"]["ctas"] == 0
    g.enable_path_counters()
    g.advance_n(1)
    c1 = g.path_counters()
    assert c1["vel"]["ctas"] == 2 * 2 * 1 and c1["pre"]["ctas"] == 2 * (2 * 2 * 1)  # two pressure launches
    g.enable_path_counters()
    assert g.path_counters()["pre"]["ctas"] == 0
    g.enable_path_counters(False)
    g.advance_n(1)
    assert g.path_counters()["vel"]["ctas"] == 0
