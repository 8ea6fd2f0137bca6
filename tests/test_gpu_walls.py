"""Reflective walls keep Eq. (80)'s conditions after every step (SPEC.md:325:
"boundary conditions of Eq. (80) hold at quadrature points on every wall after
every step, to 1e-10"; mirror rules SPEC.md:303-311).

Walls lie on primary-grid lines and p is odd across them, so p = 0 on a wall.
The cell polynomial restricted to a wall is the 1D Hermite interpolant (M,
interpolation.cpp:53-61) of the wall nodes' normal-index-0 jets, so the check
is (1) p evaluated at the Gauss points of every wall segment, in 2D literally
from the downloaded wall jets, and (2) in 2D and 3D every even-normal
coefficient of every wall node (the jets that interpolant and all even normal
derivatives read) <= 1e-10 relative, after each of 20 steps, on the kernels
the configs run with walls: tiled2d (TMA rows, K_x >= 64), var2d with the
separable c^2 generated in the kernel, tiled3d and var3d.  The velocity
conditions (normal velocity even, tangential odd) hold by construction of
the mirrored ghosts, which the parity tests pin against the oracle."""
import math

import numpy as np
import pytest

import paper_1808_10481_b200 as H

pytestmark = pytest.mark.gpu
TOL = 1e-10


def cavity(g, d, dt):
    # box [-1, -1 + L_a]: p = prod sin(w_a (x_a + 1)), w_a = pi / L_a (zero on
    # every wall), v_c = -(w_c / wt) sin(wt dt/2) cos(w_c (x_c + 1)) prod_{a != c} sin
    w = [math.pi / (k * g.grid.h) for k in g.grid.K]
    wt = math.sqrt(sum(x * x for x in w))
    g.fill_separable(0, 1.0, w, w)
    for c in range(d):
        ph = list(w)
        ph[c] += math.pi / 2
        g.fill_separable(1 + c, -(w[c] / wt) * math.sin(wt * dt / 2), w, ph)
    g.set_times(0.0, dt / 2, dt)


def wall_even_max(g, d):
    N = g.node_shape(0)
    n1 = g.m + 1
    p = g.get_field(0).reshape(tuple(N) + (n1,) * d)
    worst = 0.0
    for a in range(d):
        for side in (0, N[a] - 1):
            sl = [slice(None)] * (2 * d)
            sl[a] = side
            sl[d + a] = slice(0, n1, 2)  # even normal index
            worst = max(worst, np.abs(p[tuple(sl)]).max())
    return worst / np.abs(p).max(), p


def wall_gauss_max_2d(g, p):
    # 1D Hermite interpolant along each wall from consecutive wall nodes'
    # normal-index-0 jets, evaluated at the 2m+2 Gauss points of each segment
    m, n1 = g.m, g.m + 1
    M = H.build_interp_operator(m).M
    s, _ = np.polynomial.legendre.leggauss(2 * m + 2)
    s = s / 2  # segment [-1/2, 1/2] in units of h around its midpoint
    V = np.vander(s, 2 * m + 2, increasing=True)
    worst = 0.0
    N = p.shape[:2]
    for a in range(2):
        t = 1 - a  # tangential axis
        for side in (0, N[a] - 1):
            sl = [slice(None)] * 4
            sl[a] = side
            sl[2 + a] = 0
            wall = p[tuple(sl)]  # [tangential node][tangential coef]
            stacked = np.concatenate([wall[:-1], wall[1:]], axis=1)  # [segment][2 n1]
            ext = stacked @ M.T
            worst = max(worst, np.abs(ext @ V.T).max())
    return worst / np.abs(p).max()


CASES = [
    # (d, m, K, variable c^2)
    (2, 3, [80, 40], False),   # tiled2d, TMA rows
    (2, 2, [72, 36], False),
    (2, 3, [80, 40], True),    # var2d, separable c^2 in the kernel (config 3's kernel)
    (3, 3, [70, 6, 8], False), # tiled3d
    (3, 2, [24, 8, 8], True),  # var3d
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_walls_hold_after_every_step(case):
    d, m, K, var = CASES[case]
    h = 2.0 / K[0]
    g = H.Stepper(H.Grid([-1.0] * d, h, tuple(K)), m, boundary=[H.REFLECTIVE] * d, variable_ap=var)
    if var:
        # c^2 = 1 + 1/2 prod cos(w_a (x_a + 1)): even across every wall, as the
        # image principle needs (A.5: "variable c^2: mirror even").  Config 3's
        # 1 + 1/2 sin(pi x) sin(pi y) is odd across x, y = -1, so its product
        # with the odd divergence leaves p = 0 on the wall only to
        # discretisation error (2.5e-6 after one step at K = 80, m = 3; the
        # oracle does the same arithmetic, tests/test_gpu_var3d.py)
        w = [math.pi / (k * h) for k in K]
        g.set_coeff_separable(1.0, 0.5, w, [x + math.pi / 2 for x in w])
    assert g.kernel_variant == 1
    dt = 0.9 * h / (math.sqrt(1.5) * math.sqrt(d))
    cavity(g, d, dt)
    for step in range(20):
        g.advance_n(1, step)
        rel, p = wall_even_max(g, d)
        assert rel <= TOL, (step, rel)
        if d == 2:
            assert wall_gauss_max_2d(g, p) <= TOL, step
    assert np.isfinite(p).all() and np.abs(p).max() > 0.1
