"""Experiment harness (the reference specification's `harness` module,
SPEC.md:452-508, which the reference itself does not implement): the paper's
convergence studies run on the B200 stepper and written as CSV.

    python -m paper_1808_10481_b200.harness list
    python -m paper_1808_10481_b200.harness run standing-wave-1d --m 2 --cfl 0.9 \
        --resolutions 10,20,40,80 --final-time 4.13 --out results/
    python -m paper_1808_10481_b200.harness conserve --m 3 --cfl 0.5

Experiments (SPEC.md "Built-in experiment catalog", problems.cpp):
  standing-wave-1d      p = cos(2 pi t) sin(2 pi x) on [-1,1]; variants leapfrog, dual-hermite, modified
  variable-speed-1d     p = v = sin(x - t) on [0,2pi], c^2 = 1 + sin(x)/2, forced (leapfrog)
  advection-modified-1d u = sin(3 pi (x - t)), single field (modified)
  pv-modified-1d        p = cos(3 pi t) sin(3 pi x) (modified, leapfrog)
  acoustics-2d          p = sin(pi x) sin(pi y) cos(sqrt2 pi t), periodic (leapfrog)
  maxwell-tm-2d         TM cavity mode, omega = 8 pi, PEC walls (leapfrog)
  gaussian-reflect-2d   Gaussian pulse at (0.3, 0.3), walls: stability only
Every simulation runs on the device; L2 errors are the Gauss-quadrature
accessor (hlf_l2_error_separable, the reference's l2_error_1d/_2d) on the
final state.  CSV (SPEC.md emit_csv): errors.csv (experiment, variant, m, cfl,
K, h, field, l2_error, steps, wall_seconds) and rates.csv (experiment,
variant, m, cfl, rate, points_used), least-squares slope of log L2 against
log h over the errors above 100 eps (convergence_rate, analysis.cpp).
Exit codes: 0 ok, 1 configuration error, 2 numerical failure (instability).
"""
from __future__ import annotations

import argparse
import csv
import math
import os
import sys
import time

import numpy as np

from . import solver as S

PI = math.pi
RATE_FLOOR = 2.220446049250313e-14  # analysis.hpp rate_floor (100 eps)

CATALOG = {
    "standing-wave-1d": dict(dim=1, lo=-1.0, hi=1.0, T=4.13, variants=("leapfrog", "dual-hermite", "modified"),
                             Ks=(10, 20, 40, 80)),
    "variable-speed-1d": dict(dim=1, lo=0.0, hi=2 * PI, T=3.2, variants=("leapfrog",), Ks=(10, 20, 40, 80)),
    "advection-modified-1d": dict(dim=1, lo=-1.0, hi=1.0, T=4.13, variants=("modified",), Ks=(10, 20, 40)),
    "pv-modified-1d": dict(dim=1, lo=-1.0, hi=1.0, T=4.13, variants=("modified", "leapfrog"), Ks=(10, 20, 40, 80)),
    "acoustics-2d": dict(dim=2, lo=-1.0, hi=1.0, T=4.13, variants=("leapfrog",), Ks=(10, 20, 40, 80)),
    "maxwell-tm-2d": dict(dim=2, lo=-1.0, hi=1.0, T=0.25, variants=("leapfrog",), Ks=(16, 32, 64)),
    "gaussian-reflect-2d": dict(dim=2, lo=-1.0, hi=1.0, T=2.0, variants=("leapfrog",), Ks=(64,)),
}


class HarnessError(Exception):
    pass


def convergence_rate(hs, es, floor=RATE_FLOOR):
    """Least-squares slope of log e against log h over e > floor; (rate, points)
    (convergence_rate, analysis.cpp); rate None below 3 points."""
    pts = [(math.log(h), math.log(e)) for h, e in zip(hs, es) if e > floor and math.isfinite(e)]
    if len(pts) < 3:
        return None, len(pts)
    x = np.array([p[0] for p in pts])
    y = np.array([p[1] for p in pts])
    return float(np.polyfit(x, y, 1)[0]), len(pts)


# ------------------------------------------------------------- single runs


def _plan(T, dt_nominal):
    return S.plan_steps(T, dt_nominal)


def run_1d(name, variant, m, cfl, K, T):
    """One 1D run; returns ({field: L2}, steps)."""
    spec = CATALOG[name]
    lo, hi = spec["lo"], spec["hi"]
    grid = S.Grid1d.over(lo, hi, K)
    h = grid.h
    c_max = math.sqrt(1.5) if name == "variable-speed-1d" else 1.0
    n, dt = _plan(T, S.SchemeConfig(m=m, cfl=cfl).dt_nominal_1d(h, c_max))
    w = {"standing-wave-1d": 2 * PI, "pv-modified-1d": 3 * PI, "advection-modified-1d": 3 * PI,
         "variable-speed-1d": 1.0}[name]
    scheme = {"leapfrog": S.SCHEME_LEAPFROG, "dual-hermite": S.SCHEME_DUAL_HERMITE,
              "modified": S.SCHEME_MODIFIED_ADVECTION if name == "advection-modified-1d" else S.SCHEME_MODIFIED}
    if variant not in scheme:
        raise HarnessError(f"unknown variant {variant}")
    if name == "variable-speed-1d":
        g = S.Stepper(grid, m, variable_ap=True)
        g.set_coeff_separable(1.0, 0.5, [1.0], [0.0])  # ap = -(1 + sin(x)/2)  (problems.cpp:45-49)
    else:
        g = S.Stepper(grid, m, scheme=scheme[variant])

    def fill(f, t, pvf):
        # the problem's exact jets at (field f's nodes, t), problems.cpp
        if name == "advection-modified-1d":
            g.fill_separable(f, 1.0, [w], [-w * t])
        elif name == "variable-speed-1d":
            g.fill_separable(f, 1.0, [w], [-t])
        elif pvf == 0:
            g.fill_separable(f, math.cos(w * t), [w], [0.0])
        else:
            g.fill_separable(f, -math.sin(w * t), [w], [PI / 2])

    nf = 2 if variant == "leapfrog" or name == "advection-modified-1d" else 4
    for f in range(nf):
        g.zero_field(f)
    if variant == "leapfrog":
        fill(0, 0.0, 0)
        fill(1, dt / 2, 1)
        g.set_times(0.0, dt / 2, dt)
    elif name == "advection-modified-1d":
        fill(0, 0.0, 0)
        fill(1, dt / 2, 0)
        g.set_times(0.0, dt / 2, dt)
    elif variant == "modified":  # fields: p prim (t), v dual (t+dt/2), v prim (t), p dual (t+dt/2)
        fill(0, 0.0, 0)
        fill(1, dt / 2, 1)
        fill(2, 0.0, 1)
        fill(3, dt / 2, 0)
        g.set_times(0.0, dt / 2, dt)
    else:  # dual-hermite: p, v at primary nodes, fields 1/3 scratch
        fill(0, 0.0, 0)
        fill(2, 0.0, 1)
        g.set_times(0.0, 0.0, dt)
    if name == "variable-speed-1d":
        _run_forced_1d(g, grid, m, n)
    else:
        g.advance_n(n)
    t = g.t_p
    if name == "advection-modified-1d":
        e = g.l2_error_separable(0, 1.0, [w], [-w * t])
    elif name == "variable-speed-1d":
        e = g.l2_error_separable(0, 1.0, [w], [-t])
    else:
        e = g.l2_error_separable(0, math.cos(w * t), [w], [0.0])
    return {"p" if name != "advection-modified-1d" else "u": e}, n


def _forcing_table(grid, m, t, dual):
    """forcing_at(x_j, t)(r) of variable_speed_problem (problems.cpp:52-57):
    z_r = sin_jet(0.25, 2, -t - r pi/2) + 0.25 sin(t + r pi/2) e_0, r = 0..2m"""
    n = 2 * m + 2
    K = grid.K[0]
    x = grid.x_min[0] + grid.h * (np.arange(K) + (0.5 if dual else 0.0))
    out = np.zeros((K, n - 1, n))
    k = np.arange(n)
    fac = np.cumprod(np.concatenate(([1.0], (2.0 * grid.h) / np.arange(1, n))))
    for r in range(n - 1):
        ph = -t - r * PI / 2
        out[:, r, :] = 0.25 * fac[None, :] * np.sin(2.0 * x[:, None] + ph + k[None, :] * PI / 2)
        out[:, r, 0] += 0.25 * math.sin(t + r * PI / 2)
    return out


def _run_forced_1d(g, grid, m, steps):
    """the forced leapfrog loop: tables for p at (primary, t_v), for v at (dual, t_p + dt)
    (stepper1d.cpp:152, 162)"""
    for i in range(steps):
        t_p, t_v, dt = g.times()
        g.set_forcing(S.PRIMARY, _forcing_table(grid, m, t_v, False))
        g.set_forcing(S.DUAL, _forcing_table(grid, m, t_p + dt, True))
        g.step_system(i)


def _gauss_jets(centre, delta, x, h, n):
    """gaussian_jet (jet.cpp:76-85) at the points x: [len(x), n]"""
    d = x - centre
    raw = np.zeros((len(x), n))
    raw[:, 0] = np.exp(-d * d / delta)
    if n > 1:
        raw[:, 1] = -2.0 / delta * d * raw[:, 0]
    for i in range(1, n - 1):
        raw[:, i + 1] = -2.0 / delta * (d * raw[:, i] + i * raw[:, i - 1])
    fac = np.cumprod(np.concatenate(([1.0], h / np.arange(1, n))))
    return raw * fac[None, :]


def run_2d(name, variant, m, cfl, K, T):
    if variant != "leapfrog":
        raise HarnessError("2D experiments run the Hermite-leapfrog scheme")
    grid = S.Grid2d.over(-1.0, 1.0, -1.0, 1.0, K)
    h = grid.h
    n, dt = _plan(T, S.SchemeConfig(m=m, cfl=cfl).dt_nominal_2d(h, 1.0))
    walls = name in ("maxwell-tm-2d", "gaussian-reflect-2d")
    g = S.Stepper(grid, m, boundary=[S.REFLECTIVE if walls else S.PERIODIC] * 2)
    for f in range(3):
        g.zero_field(f)
    if name == "gaussian-reflect-2d":
        N = K + 1
        x = -1.0 + h * np.arange(N)
        gx = _gauss_jets(0.3, 0.002, x, h, m + 1)
        jets = np.einsum("xi,yj->xyij", gx, gx).reshape(N * N, (m + 1) ** 2)
        g.set_field(0, jets)
        g.set_times(0.0, dt / 2, dt)
        p0 = np.abs(jets).max()
        g.advance_n(n)
        pmax = float(np.abs(g.get_field(0)).max())
        return {"p_max_over_initial": float(pmax / p0)}, n
    wx = PI if name == "acoustics-2d" else 8 * PI
    wt = math.sqrt(2.0) * wx
    # p (or Ez) = cos(wt t) sin(wx x) sin(wx y); velocities at t = dt/2 (problems.cpp:140-183;
    # Maxwell: v = -Hy, u = Hx on the device, the same acoustic mode)
    g.fill_separable(0, 1.0, [wx, wx], [0.0, 0.0])
    amp = -wx / wt * math.sin(wt * dt / 2)
    g.fill_separable(1, amp, [wx, wx], [PI / 2, 0.0])
    g.fill_separable(2, amp, [wx, wx], [0.0, PI / 2])
    g.set_times(0.0, dt / 2, dt)
    g.advance_n(n)
    e = g.l2_error_separable(0, math.cos(wt * g.t_p), [wx, wx], [0.0, 0.0])
    return {"Ez" if name == "maxwell-tm-2d" else "p": e}, n


def run_experiment(name, variant, ms, cfls, Ks, T):
    """The sweep; returns (error rows, rate rows) (ExperimentReport)."""
    if name not in CATALOG:
        raise HarnessError(f"unknown experiment {name}")
    spec = CATALOG[name]
    if not Ks:
        raise HarnessError("empty resolution list")
    if list(Ks) != sorted(set(Ks)):
        raise HarnessError("resolutions must be strictly increasing")
    if not T > 0:
        raise HarnessError("final time must be positive")
    if variant not in spec["variants"]:
        raise HarnessError(f"{name} supports variants {spec['variants']}")
    errs, rates = [], []
    for m in ms:
        for cfl in cfls:
            by_field = {}
            for K in Ks:
                t0 = time.perf_counter()
                try:
                    if spec["dim"] == 1:
                        res, steps = run_1d(name, variant, m, cfl, K, T)
                    else:
                        res, steps = run_2d(name, variant, m, cfl, K, T)
                except S.InstabilityError as exc:
                    res, steps = {"p": float("nan")}, exc.step
                sec = time.perf_counter() - t0
                h = (spec["hi"] - spec["lo"]) / K
                for fld, e in res.items():
                    errs.append(dict(experiment=name, variant=variant, m=m, cfl=cfl, K=K, h=h, field=fld,
                                     l2_error=e, steps=steps, wall_seconds=sec))
                    by_field.setdefault(fld, []).append((h, e))
            if name != "gaussian-reflect-2d":
                for fld, pts in by_field.items():
                    r, used = convergence_rate([p[0] for p in pts], [p[1] for p in pts])
                    if r is not None:
                        rates.append(dict(experiment=name, variant=variant, m=m, cfl=cfl, rate=r, points_used=used))
    return errs, rates


def emit_csv(errs, rates, out):
    os.makedirs(out, exist_ok=True)
    ecols = ["experiment", "variant", "m", "cfl", "K", "h", "field", "l2_error", "steps", "wall_seconds"]
    rcols = ["experiment", "variant", "m", "cfl", "rate", "points_used"]
    for fname, cols, rows in (("errors.csv", ecols, errs), ("rates.csv", rcols, rates)):
        with open(os.path.join(out, fname), "w", newline="") as f:
            w = csv.writer(f, lineterminator="\n")
            w.writerow(cols)
            for r in rows:
                w.writerow([repr(float(r[c])) if isinstance(r[c], (float, np.floating)) else r[c] for c in cols])


def conserve(m, cfl, steps=100, K=16, out=None):
    """The conservation trace (SPEC.md acceptance 6) on the device: Q^h / R^h of
    random periodic data (random_wave_problem's p_t = v_x, v_t = p_x form with
    four trig modes) over `steps` steps; returns the max relative drift."""
    grid = S.Grid1d.over(-1.0, 1.0, K)
    g = S.Stepper(grid, m, ap=1.0, av=1.0)
    dt = S.SchemeConfig(m=m, cfl=cfl).dt_nominal_1d(grid.h, 1.0)
    rng = np.random.default_rng(1234)
    for f in range(2):
        g.zero_field(f)
    for k in range(4):
        wk = (k + 1) * PI
        fade = 1.0 / (k + 1) ** 2
        a, b = rng.standard_normal(2) * fade
        g.fill_separable(0, a, [wk], [0.0])
        g.fill_separable(0, b, [wk], [PI / 2])
        c, d = rng.standard_normal(2) * fade
        g.fill_separable(1, c, [wk], [0.0])
        g.fill_separable(1, d, [wk], [PI / 2])
    g.set_times(0.0, dt / 2, dt)
    g.advance_v()  # R(0) pairs v(t + dt/2) with p(t)
    g.set_times(0.0, dt / 2, dt)
    r0 = g.energy_1d(1)
    trace = [r0]
    for _ in range(steps):
        g.advance_p()
        trace.append(g.energy_1d(0))
        g.advance_v()
        trace.append(g.energy_1d(1))
    drift = max(abs(q / r0 - 1.0) for q in trace)
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "conservation.csv"), "w", newline="") as f:
            w = csv.writer(f, lineterminator="\n")
            w.writerow(["half_step", "energy", "relative_drift"])
            for i, q in enumerate(trace):
                w.writerow([i, repr(q), repr(q / r0 - 1.0)])
    return drift


def _floats(s):
    return [float(x) for x in s.split(",") if x]


def _ints(s):
    return [int(x) for x in s.split(",") if x]


def cli_main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1808_10481_b200.harness")
    sub = ap.add_subparsers(dest="cmd")
    sub.add_parser("list")
    r = sub.add_parser("run")
    r.add_argument("experiment")
    r.add_argument("--m", default="2")
    r.add_argument("--cfl", default="0.9")
    r.add_argument("--resolutions", default=None)
    r.add_argument("--variant", default=None)
    r.add_argument("--final-time", type=float, default=None)
    r.add_argument("--out", default="harness_out")
    c = sub.add_parser("conserve")
    c.add_argument("--m", type=int, default=2)
    c.add_argument("--cfl", type=float, default=0.9)
    c.add_argument("--steps", type=int, default=100)
    c.add_argument("--out", default=None)
    sub.add_parser("dispersion")
    args = ap.parse_args(argv)
    if args.cmd == "list":
        for name, spec in CATALOG.items():
            print(f"{name:24s} d={spec['dim']} variants={','.join(spec['variants'])} T={spec['T']} K={spec['Ks']}")
        return 0
    if args.cmd == "dispersion":
        print("dispersion analysis is out of scope (DESIGN.md sec. 7: offline Fourier analysis, dispersion.cpp)")
        return 1
    try:
        if args.cmd == "conserve":
            drift = conserve(args.m, args.cfl, args.steps, out=args.out)
            print(f"max relative drift of Q/R over {args.steps} steps: {drift:.3e}")
            return 0 if drift < 1e-10 else 2
        if args.cmd != "run":
            ap.print_help()
            return 1
        if args.experiment not in CATALOG:
            print(f"unknown experiment {args.experiment}; catalog: {', '.join(CATALOG)}", file=sys.stderr)
            return 1
        spec = CATALOG[args.experiment]
        Ks = _ints(args.resolutions) if args.resolutions is not None else list(spec["Ks"])
        variant = args.variant or spec["variants"][0]
        T = args.final_time if args.final_time is not None else spec["T"]
        errs, rates = run_experiment(args.experiment, variant, _ints(args.m), _floats(args.cfl), Ks, T)
        emit_csv(errs, rates, args.out)
        for row in rates:
            print(f"{row['experiment']} {row['variant']} m={row['m']} cfl={row['cfl']}: rate "
                  f"{row['rate']:.2f} ({row['points_used']} points)")
        if any(not math.isfinite(e["l2_error"]) for e in errs):
            return 2
        return 0
    except (HarnessError, S.ConfigError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(cli_main())
