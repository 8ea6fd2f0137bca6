"""3D variable coefficients on the var3d kernel (csrc/kernels_var3d.cu):
ap = -(c0 + c1 prod sin(w x + phase)) generated on the fly at every node
(hlf_set_coeff_separable), against the oracle running the reference's
iterated truncated CK recurrence (ck_recurrence_variable, stepper1d.cpp:22-38;
tensor_multiply, jet.cpp:109-121) with the same coefficient as stored per-node
jets (the reference's sin_jet, jet.cpp:65-74, in outer product).
Bar: 1e-12 relative max-norm per field."""
import math
import time

import numpy as np
import pytest

import oracle as O
import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu
TOL = 1e-12


def sin_jets(x, h, n, w, ph):
    k = np.arange(n)
    fac = np.cumprod(np.concatenate(([1.0], (w * h) / np.arange(1, n))))
    return fac[None, :] * np.sin(w * x[:, None] + ph + k[None, :] * math.pi / 2)


def sep_jets(K, h, n, boundary, dual, c0, c1, w, ph):
    """[nodes][n^3] x-major: -(c0 e_0 + c1 s_x (x) s_y (x) s_z) at the nodes of one grid"""
    N = [k if (dual or b == 0) else k + 1 for k, b in zip(K, boundary)]
    off = 0.5 * h if dual else 0.0
    s = [sin_jets(-1.0 + off + h * np.arange(N[a]), h, n, w[a], ph[a]) for a in range(3)]
    jets = -c1 * np.einsum("xi,yj,zk->xyzijk", s[0], s[1], s[2])
    jets[:, :, :, 0, 0, 0] -= c0
    return jets.reshape(N[0] * N[1] * N[2], n ** 3)


def pair(m, K, boundary, seed):
    h = 2.0 / K[0]
    g = H.Stepper(H.Grid([-1.0] * 3, h, tuple(K)), m, boundary=boundary, variable_ap=True)
    o = O.OracleStepper(3, m, K, h, boundary=boundary)
    rng = np.random.default_rng(seed)
    for f in range(4):
        a = rng.standard_normal((g.field_nodes(f), g.F)) * 0.6 ** np.arange(g.F)
        g.set_field(f, a)
        o.set_field(f, a)
    return g, o


def rel_err(got, ref):
    return np.abs(got - ref).max() / np.abs(ref).max()


CASES = [(1.0, 0.5, [math.pi] * 3, [0.0] * 3),                            # cfg 3's c^2, extended to 3D
         (1.3, -0.4, [math.pi, 2 * math.pi, math.pi], [0.3, 0.1, 0.7])]   # a general separable c^2


@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("boundary", [[0, 0, 0], [1, 1, 1], [1, 0, 1]])
@pytest.mark.parametrize("case", [0, 1])
def test_var3d_matches_oracle(m, boundary, case):
    K = [7, 6, 5]
    c0, c1, w, ph = CASES[case]
    g, o = pair(m, K, boundary, seed=700 + 10 * m + case)
    g.set_coeff_separable(c0, c1, w, ph)
    assert g.kernel_variant == 1
    n = 2 * m + 2
    for grid, dual in ((0, False), (1, True)):
        o.set_coeff(grid, 0, sep_jets(K, g.grid.h, n, boundary, dual, c0, c1, w, ph))
    dt = 0.2 * g.grid.h
    for s in (g, o):
        s.set_times(0.0, dt / 2, dt)
    g.advance_n(6)
    assert o.advance_n(6) == -1
    for f in range(4):
        e = rel_err(g.get_field(f), o.get_field(f))
        assert e <= TOL, (f, e)


def test_separable_2d_equals_stored_jets():
    # 2D: hlf_set_coeff_separable runs var2d with the jets generated in the
    # kernel and separable products; the stored-jet var2d path with the same
    # coefficient (host jets) must agree to roundoff
    m, K, bnd = 3, [16, 12], [1, 1]
    h = 2.0 / K[0]
    outs = []
    for mode in ("sep", "stored"):
        g = H.Stepper(H.Grid([-1.0] * 2, h, tuple(K)), m, boundary=bnd, variable_ap=True)
        rng = np.random.default_rng(5)
        for f in range(3):
            g.set_field(f, rng.standard_normal((g.field_nodes(f), g.F)) * 0.6 ** np.arange(g.F))
        if mode == "sep":
            g.set_coeff_separable(1.0, 0.5, [math.pi] * 2, [0.0] * 2)
        else:
            n = 2 * m + 2
            for grid, dual in ((0, False), (1, True)):
                N = [k if (dual or b == 0) else k + 1 for k, b in zip(K, bnd)]
                off = 0.5 * h if dual else 0.0
                sx = sin_jets(-1.0 + off + h * np.arange(N[0]), h, n, math.pi, 0.0)
                sy = sin_jets(-1.0 + off + h * np.arange(N[1]), h, n, math.pi, 0.0)
                jets = -0.5 * np.einsum("xi,yj->xyij", sx, sy)
                jets[:, :, 0, 0] -= 1.0
                g.set_coeff(grid, jets.reshape(N[0] * N[1], n * n))
        g.set_times(0.0, 0.01, 0.02)
        g.advance_n(5)
        outs.append([g.get_field(f) for f in range(3)])
    for a, b in zip(*outs):
        assert rel_err(a, b) <= 1e-12


def test_var3d_throughput_against_the_generic_kernel():
    # the generic (faithful) kernel with stored jets vs var3d with on-the-fly jets
    m, K = 3, [24, 24, 24]
    h = 2.0 / K[0]
    rates = {}
    for mode in ("var3d", "generic"):
        g = H.Stepper(H.Grid([-1.0] * 3, h, tuple(K)), m, variable_ap=True)
        g.fill_separable(0, 1.0, [math.pi] * 3, [0.0] * 3)
        if mode == "var3d":
            g.set_coeff_separable(1.0, 0.5, [math.pi] * 3, [0.0] * 3)
        else:
            n = 2 * m + 2
            for grid, dual in ((0, False), (1, True)):
                g.set_coeff(grid, sep_jets(K, h, n, [0, 0, 0], dual, 1.0, 0.5, [math.pi] * 3, [0.0] * 3))
            g.kernel_variant = 0
        g.set_times(0.0, 0.01, 0.02)
        g.advance_n(1)
        g.synchronize()
        t0 = time.perf_counter()
        g.advance_n(3)
        g.synchronize()
        sec = (time.perf_counter() - t0) / 3
        rates[mode] = 4 * 64 * 24 ** 3 / sec
    print("DOF-updates/s", rates)
    assert rates["var3d"] > 3 * rates["generic"], rates


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("boundary", [[0, 0], [1, 1], [1, 0]])
def test_var2d_separable_matches_oracle(m, boundary):
    # config 3's coefficient generated in the var2d kernel vs the oracle with stored jets
    K = [13, 11]
    h = 2.0 / K[0]
    g = H.Stepper(H.Grid([-1.0] * 2, h, tuple(K)), m, boundary=boundary, variable_ap=True)
    o = O.OracleStepper(2, m, K, h, boundary=boundary)
    rng = np.random.default_rng(900 + m)
    for f in range(3):
        a = rng.standard_normal((g.field_nodes(f), g.F)) * 0.6 ** np.arange(g.F)
        g.set_field(f, a)
        o.set_field(f, a)
    w, ph = [math.pi, 2 * math.pi], [0.3, -0.2]
    g.set_coeff_separable(1.1, 0.45, w, ph)
    n = 2 * m + 2
    for grid, dual in ((0, False), (1, True)):
        N = [k if (dual or b == 0) else k + 1 for k, b in zip(K, boundary)]
        off = 0.5 * h if dual else 0.0
        sx = sin_jets(-1.0 + off + h * np.arange(N[0]), h, n, w[0], ph[0])
        sy = sin_jets(-1.0 + off + h * np.arange(N[1]), h, n, w[1], ph[1])
        jets = -0.45 * np.einsum("xi,yj->xyij", sx, sy)
        jets[:, :, 0, 0] -= 1.1
        o.set_coeff(grid, 0, jets.reshape(N[0] * N[1], n * n))
    dt = 0.2 * h
    for s_ in (g, o):
        s_.set_times(0.0, dt / 2, dt)
    g.advance_n(8)
    assert o.advance_n(8) == -1
    for f in range(3):
        e = rel_err(g.get_field(f), o.get_field(f))
        assert e <= TOL, (f, e)
