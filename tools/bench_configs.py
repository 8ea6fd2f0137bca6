"""Device throughput of every SURVEY.md sec. 8(d) configuration through the
public Python API (CUDA events on the solver stream, warm-up steps first).
The headline 3D line is bench.py's; this script records the others:

  cfg1   1D m=3 standing wave, K=256 (143 steps) and K=2^24
  cfg2   2D periodic acoustics mode, K=1024, m=1..4 (+ 4096^2 m=3)
  cfg3   2D walls, K=4096, m=3, c^2 = 1 + sin(pi x) sin(pi y)/2 generated in the
         var2d kernel (hlf_set_coeff_separable; and as stored jets, hlf_set_coeff;
         separable data instead of the Gaussian pulse: same arithmetic)
  cfg4   3D periodic, 512x512x256, m=1..3 (bench.py's workload)
  cfg3-3D  3D periodic, 192^3, m=1..3, c^2 = 1 + sin(pi x) sin(pi y) sin(pi z)/2
         generated in the var3d kernel

Every line carries the nvidia-smi clocks sampled while it ran (bench.py's
ClockSampler).  Usage: python tools/bench_configs.py [out.json]"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1808_10481_b200 as H

ROOT_ = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT_)
from bench import ClockSampler  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HBM = 6551.4e9  # MEASURED_PEAKS.json hbm_gbs


def timed(g, stream, steps, warm=3):
    # advance_n captures its CUDA graph (runs of >= 64 steps) on the first call
    # with a given dt: warm up with the timed step count there
    warm = steps if steps >= 64 else warm
    g.advance_n(warm)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    g.advance_n(steps, warm)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def sin_jets(x, h, n, w=math.pi):
    """scaled jets of sin(w x) at the points x: [len(x), n] (sin_jet, jet.cpp)"""
    k = np.arange(n)
    fac = np.cumprod(np.concatenate(([1.0], (w * h) / np.arange(1, n))))
    return fac[None, :] * np.sin(w * x[:, None] + k[None, :] * math.pi / 2)


def c2_jets_2d(K, h, n, boundary, dual):
    """-(1 + sin(pi x) sin(pi y) / 2) jets, [nodes][n * n] x-major (nodes x-slowest)"""
    N = [K if dual or b == 0 else K + 1 for b in boundary]
    off = 0.5 * h if dual else 0.0
    sx = sin_jets(-1.0 + off + h * np.arange(N[0]), h, n)
    sy = sin_jets(-1.0 + off + h * np.arange(N[1]), h, n)
    jets = -0.5 * np.einsum("xi,yj->xyij", sx, sy)
    jets[:, :, 0, 0] -= 1.0
    return jets.reshape(N[0] * N[1], n * n)


def kernel_name(d, variable, variant):
    if d == 1:
        return "faithful1d"  # half_1d: register-resident, bit-identical to the reference
    if variant != 1:
        return "generic"
    if variable:
        return "var2d" if d == 2 else "var3d"
    return f"tiled{d}d"


def run(name, d, m, K, boundary=None, variable=False, steps=20, separable=False):
    stream = torch.cuda.Stream()
    Ks = list(K)
    g = H.Stepper(H.Grid([-1.0] * d, 2.0 / Ks[0], tuple(Ks)), m, boundary=boundary, variable_ap=variable,
                  stream=stream.cuda_stream)
    pi = math.pi
    g.fill_separable(0, 1.0, [pi] * d, [0.0] * d)
    if variable and separable:
        # c^2 = 1 + prod sin(pi x_a) / 2 through hlf_set_coeff_separable
        # (3D: generated in the var3d kernel; 2D: expanded into jets on the device)
        g.set_coeff_separable(1.0, 0.5, [pi] * d, [0.0] * d)
    elif variable:
        # config 3's ap = -c^2, c^2 = 1 + sin(pi x) sin(pi y) / 2, as scaled jets
        # (n entries per axis) at the nodes of both grids
        for grid in (0, 1):
            g.set_coeff(grid, c2_jets_2d(Ks[0], g.grid.h, 2 * m + 2, boundary or [0, 0], dual=grid == 1))
    c_max = math.sqrt(1.5) if variable else 1.0
    dt = 0.9 * g.grid.h / (math.sqrt(d) * c_max)
    g.set_times(0.0, dt / 2, dt)
    with ClockSampler(g.device) as clk:
        ms = timed(g, stream, steps)
    dof = (d + 1) * (m + 1) ** d * math.prod(Ks)
    rate = dof / (ms * 1e-3)
    line = {"config": name, "d": d, "m": m, "K": Ks, "boundary": boundary or [0] * d, "variable_c2": variable,
            "kernel": kernel_name(d, variable, g.kernel_variant), "ms_per_step": ms,
            "dof_updates_per_s": rate, "hbm_frac_24B": 24 * rate / HBM, "clocks": clk.summary()}
    if variable and not (separable and d == 3):
        # + the ap jets of both grids (n^d doubles per node, read once per half step)
        alg = 24 + 2 * (2 * m + 2) ** d * 8 / ((d + 1) * (m + 1) ** d)
        line["alg_bytes_per_dof"] = alg
        line["hbm_frac_alg"] = alg * rate / HBM
    print(json.dumps(line), flush=True)
    del g
    torch.cuda.empty_cache()
    return line


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2", "configs.json")
    res = [run("cfg1", 1, 3, [256], steps=143), run("cfg1 large", 1, 3, [1 << 24], steps=20)]
    for m in (1, 2, 3, 4):
        res.append(run("cfg2", 2, m, [1024, 1024], steps=100))
    res.append(run("cfg2 large", 2, 3, [4096, 4096], steps=20))
    res.append(run("cfg3", 2, 3, [4096, 4096], boundary=[1, 1], variable=True, separable=True, steps=3))
    res.append(run("cfg3 stored jets", 2, 3, [4096, 4096], boundary=[1, 1], variable=True, steps=3))
    for m in (1, 2, 3):
        res.append(run("cfg4", 3, m, [512, 512, 256], steps=5))
    for m in (1, 2, 3):
        res.append(run("cfg3-3D", 3, m, [192, 192, 192], variable=True, separable=True, steps=3))
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
