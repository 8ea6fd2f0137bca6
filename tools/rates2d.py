"""Explore the 2D acoustics convergence rates:
p = sin(pi x) sin(pi y) cos(sqrt2 pi t) on [-1,1]^2 periodic, CFL 0.9,
Gauss-quadrature L2 of p on the device (hlf_l2_error_separable), rates by the
reference's least-squares rule (convergence_rate, analysis.cpp)."""
import math
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1808_10481_b200 as H


def l2_err(m, K, T, cfl=0.9, field=0):
    h = 2.0 / K
    n, dt = H.plan_steps(T, H.SchemeConfig(m=m, cfl=cfl).dt_nominal_2d(h, 1.0))
    g = H.Stepper(H.Grid([-1.0] * 2, h, (K, K)), m)
    pi = math.pi
    wt = math.sqrt(2) * pi
    g.fill_separable(0, 1.0, [pi] * 2, [0.0] * 2)
    amp = -pi / wt * math.sin(wt * dt / 2)
    for c in range(1, 3):
        g.fill_separable(c, amp, [pi] * 2, [pi / 2 if a == c - 1 else 0.0 for a in range(2)])
    g.set_times(0.0, dt / 2, dt)
    g.advance_to(T)
    return g.l2_error_separable(0, math.cos(wt * g.t_p), [pi] * 2, [0.0] * 2)


def rate(hs, es, floor=2.220446049250313e-14):
    pts = [(math.log(h), math.log(e)) for h, e in zip(hs, es) if e > floor]
    x = np.array([p[0] for p in pts]); y = np.array([p[1] for p in pts])
    return np.polyfit(x, y, 1)[0]


if __name__ == "__main__":
    for T in (1.0, 2.0, 4.13):
        for Ks in ([10, 20, 40, 80], [20, 40, 80, 160], [10, 20, 40, 80, 160]):
            out = []
            for m in range(4):
                es = [l2_err(m, K, T) for K in Ks]
                out.append(rate([2.0 / K for K in Ks], es))
            print(f"T={T} Ks={Ks} rates={[round(r, 2) for r in out]}", flush=True)
