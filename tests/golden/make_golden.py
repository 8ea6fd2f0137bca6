"""Generate tests/golden/reference_1d.json by running the COMPILED REFERENCE
(/root/reference/proj/src built unchanged by oracle/Makefile into oracle/_ref).

Run here (where /root/reference exists):   python tests/golden/make_golden.py
The fixture pins the oracle and the CUDA path on machines without the
reference sources (the GPU box).  Contents:
  * M for m = 0..8 and its condition (build_interp_operator, interpolation.cpp:21-51)
  * the L2 goldens of proj/tests/test_stepper1d.cpp:323-355 recomputed
  * config 1 (standing wave, m = 3, K = 256, T = 1, cfl 0.9): step count, dt,
    the full initial and final staggered state, L2(p)
  * the random-wave energy setup of test_stepper1d.cpp:389-417 (initial state,
    state after 100 steps, max relative drift of Q/R) for m = 0..3
  * reconstruct_cell_2d outputs for fixed corner data (interpolation.cpp:77-113)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle as O  # noqa: E402


def leapfrog_l2(problem, m, cfl, K, T):
    r = O.RefStepper1d(problem, m, K)
    n = O.ref_step_count(T, O.ref_dt_nominal(1, cfl, r.h, r.c_max))
    r.init_leapfrog(T / n)
    assert r.steps(n) == -1
    return r.l2_p()


def main():
    out = {"source": "oracle/_ref (reference proj/src compiled with oracle/shim)"}
    out["M"] = {}
    for m in range(9):
        M, cond = O.ref_build_interp(m)
        out["M"][str(m)] = {"M": M.ravel().tolist(), "condition": cond}

    conv = {}
    for name, T, Ks, pinned in (
        ("standing-wave", 4.13, [10, 20, 40, 80], [1.5081e-04, 2.3521e-06, 3.6708e-08, 5.7460e-10]),
        ("variable-speed", 3.2, [10, 20, 40, 80], [5.3628e-06, 8.0000e-08, 1.2426e-09, 1.9781e-11]),
    ):
        conv[name] = {"m": 2, "cfl": 0.9, "T": T, "K": Ks, "pinned": pinned,
                      "l2": [leapfrog_l2(name, 2, 0.9, K, T) for K in Ks]}
    out["convergence"] = conv

    m, K, T = 3, 256, 1.0
    r = O.RefStepper1d("standing-wave", m, K)
    n = O.ref_step_count(T, O.ref_dt_nominal(1, 0.9, r.h, r.c_max))
    r.init_leapfrog(T / n)
    p0, v0, t0 = r.get()
    assert r.steps(n) == -1
    p1, v1, t1 = r.get()
    out["config1"] = {"problem": "standing-wave", "m": m, "K": K, "T": T, "cfl": 0.9, "steps": n,
                      "h": r.h, "x_min": r.x_min, "times0": list(t0), "times1": list(t1),
                      "p0": p0.ravel().tolist(), "v0": v0.ravel().tolist(),
                      "p1": p1.ravel().tolist(), "v1": v1.ravel().tolist(), "l2_p": r.l2_p()}

    energy = {}
    for m in range(4):
        r = O.RefStepper1d("random-wave", m, 16, seed=1234)
        dt = O.ref_dt_nominal(1, 0.9, r.h, 1.0)
        r.init_leapfrog(dt)
        p0, v0, t0 = r.get()
        q0 = r.conserved_r(1.0)
        drift = 0.0
        for _ in range(100):
            r.advance_p()
            drift = max(drift, abs(r.conserved_q(1.0) / q0 - 1.0))
            r.advance_v()
            drift = max(drift, abs(r.conserved_r(1.0) / q0 - 1.0))
        p1, v1, t1 = r.get()
        energy[str(m)] = {"K": 16, "cfl": 0.9, "dt": dt, "steps": 100, "q0": q0, "max_drift": drift,
                          "times0": list(t0), "times1": list(t1),
                          "p0": p0.ravel().tolist(), "v0": v0.ravel().tolist(),
                          "p1": p1.ravel().tolist(), "v1": v1.ravel().tolist()}
    out["energy"] = energy

    rng = np.random.default_rng(7)
    rec = []
    for m in (1, 2, 3):
        cs = [rng.standard_normal((m + 1) ** 2) for _ in range(4)]
        ext = O.ref_reconstruct_2d(m, *cs)
        rec.append({"m": m, "corners": [c.tolist() for c in cs], "ext": ext.ravel().tolist()})
    out["reconstruct_2d"] = rec

    path = os.path.join(os.path.dirname(__file__), "reference_1d.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path)


if __name__ == "__main__":
    main()
