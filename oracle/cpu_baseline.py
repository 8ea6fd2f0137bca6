"""ORACLE TEST INFRASTRUCTURE -- the CPU baseline legs of bench.py (not product code).

The CPU measurements BASELINE.md sec. 4 asks for, taken on the host the GPU
numbers come from:
  1. the reference's own Stepper1d (oracle/_ref: /root/reference/proj/src
     compiled unchanged against the dependency shims), 1 thread, config 1
     (standing wave, m = 3, K = 256) and K = 2^20, m = 3;
  2. the same as `nproc` concurrent independent instances (the reference's
     concurrency model: distinct states may step concurrently),
     aggregate DOF-updates/s;
  3. the oracle restatement (oracle/hlf_oracle.cpp) on the bench's own 3D m = 3
     periodic mode at 64^3 (out of cache: 4 x 134 MB of state) and 2D 1024^2
     with OpenMP over every host thread, and at 32^3 / 512^2 with 1 thread.
Each leg is bounded (a few seconds of CPU work) so bench.py stays within
minutes.  A DOF-update is one coefficient of one field at one node advanced
one full step: 1D 2 (m+1) K, 3D 4 (m+1)^3 K^3 per step.
"""
from __future__ import annotations

import math
import multiprocessing as mp
import os
import platform
import subprocess
import time

import numpy as np

from . import OracleStepper, RefStepper1d, add_separable, ref_available


def host_info() -> dict:
    model = platform.processor() or "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count() or 1}


def ref1d_rate(K: int, m: int = 3, min_seconds: float = 1.0, max_steps: int = 1000) -> dict:
    """The reference's Stepper1d::step_system (stepper1d.cpp:168-172) on the
    standing wave, 1 thread: DOF-updates/s = 2 (m+1) K steps / s."""
    r = RefStepper1d("standing-wave", m, K)
    dt = 0.9 * r.h / r.c_max
    r.init_leapfrog(dt)
    r.steps(1)  # warm-up
    steps, sec = 0, 0.0
    t0 = time.perf_counter()
    while sec < min_seconds and steps < max_steps:
        r.steps(1, steps)
        steps += 1
        sec = time.perf_counter() - t0
    return {"K": K, "m": m, "steps": steps, "seconds": sec, "dof_per_s": 2 * (m + 1) * K * steps / sec}


def _ref1d_worker(args):
    K, m, steps = args
    r = RefStepper1d("standing-wave", m, K)
    r.init_leapfrog(0.9 * r.h / r.c_max)
    t0 = time.perf_counter()
    r.steps(steps)
    return time.perf_counter() - t0


def ref1d_instances(K: int, m: int, steps: int, procs: int) -> dict:
    """`procs` concurrent independent reference Stepper1d instances (one
    process each); aggregate rate over the slowest instance's wall time."""
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        t0 = time.perf_counter()
        secs = pool.map(_ref1d_worker, [(K, m, steps)] * procs)
        wall = time.perf_counter() - t0
    return {"K": K, "m": m, "steps": steps, "instances": procs, "wall_seconds": wall,
            "max_instance_seconds": max(secs),
            "dof_per_s": procs * 2 * (m + 1) * K * steps / max(secs)}


def oracle_rate(d: int, K: int, m: int, steps: int, threads: int) -> dict:
    """The restatement on the periodic standing mode (the bench's workload in
    3D): DOF-updates/s = (d+1) (m+1)^d K^d steps / s."""
    h = 2.0 / K
    o = OracleStepper(d, m, [K] * d, h, threads=threads)
    F = (m + 1) ** d
    p = np.zeros((K ** d, F))
    add_separable(d, [K] * d, [-1.0] * d, h, 0.0, m + 1, 1.0, [math.pi] * d, [0.0] * d, p)
    o.set_field(0, p)
    dt = 0.9 * h / math.sqrt(d)
    o.set_times(0.0, dt / 2, dt)
    t0 = time.perf_counter()
    o.advance_n(steps)
    sec = time.perf_counter() - t0
    dof = (d + 1) * F * K ** d
    return {"d": d, "K": K, "m": m, "steps": steps, "threads": threads, "seconds": sec,
            "dof_per_s": dof * steps / sec}


def full_plan(quick: bool = False) -> dict:
    """Every leg of BASELINE.md sec. 4 (quick: smaller samples, for tests)."""
    info = host_info()
    n = info["nproc"]
    out = {"host": info}
    if ref_available():
        out["ref_stepper1d_config1_1thread"] = ref1d_rate(256, 3, min_seconds=0.2 if quick else 1.0)
        out["ref_stepper1d_K2^20_1thread"] = ref1d_rate(1 << (12 if quick else 20), 3,
                                                         min_seconds=0.2 if quick else 2.0, max_steps=3)
        out["ref_stepper1d_K2^20_nproc_instances"] = ref1d_instances(1 << (12 if quick else 20), 3,
                                                                      1 if quick else 2, min(n, 4) if quick else n)
    # 1 thread on 32^3 / 512^2 (bounded time; still out of L2), every thread on 64^3 / 1024^2
    out["oracle_3d_m3_32^3_1thread"] = oracle_rate(3, 12 if quick else 32, 3, 1, 1)
    out["oracle_3d_m3_64^3_all_threads"] = oracle_rate(3, 16 if quick else 64, 3, 1 if quick else 2, n)
    out["oracle_2d_m3_512^2_1thread"] = oracle_rate(2, 32 if quick else 512, 3, 1, 1)
    out["oracle_2d_m3_1024^2_all_threads"] = oracle_rate(2, 64 if quick else 1024, 3, 1, n)
    return out
