"""Benchmark driver: 3D acoustic Hermite-leapfrog step, order m = 3, FP64.

Workload (BASELINE.json configs[3]/[4]): 3D acoustic tensor-product
Hermite-leapfrog, m = 3, periodic.  512^3 (256 GiB of state) does not fit one
B200, so each GPU holds a 512 x 512 x 256 z-slab (128 GiB);
with N GPUs the global grid is 512 x 512 x (256 N) (weak scaling, NCCL z halos).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One JSON line on rank 0.  `value` = DOF-updates/s of the whole job, device-timed
with CUDA events on the solver stream, max over ranks.  A DOF-update is one
FP64 scaled coefficient of one field at one node advanced one full leapfrog
step: DOF/step = 4 (m+1)^3 K^3.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = 3
NX, NY, NZ_PER_GPU = 512, 512, 256
CFL = 0.9
FLOP_PER_DOF = 166.5          # SURVEY.md sec. 8(d) / App. B, minimal formulation, 3D m=3
FLOP_VEL_PER_CELL = 14976.0   # App. B: R + d(2 T_v + F)
FLOP_PRE_PER_CELL = 27648.0   # App. B: d R + (d-1) n^d + 2 T_p + F (pressure half step)
BYTES_PER_DOF = 24.0          # read twice + written once per full step
METRIC = "DOF-updates/sec (FP64, order m)"
UNIT = "DOF-updates/s"


def peaks():
    out = {"hbm_gbs": 6551.4, "hbm_src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        out["hbm_gbs"] = float(mp["hbm_gbs"])
        out["hbm_src"] = "MEASURED_PEAKS.json"
    except Exception:
        pass
    # FP64 is not in MEASURED_PEAKS.json; tools/fp64_peak.cu measured it on this pool
    out["fp64_tflops"] = 34.23
    out["fp64_src"] = "profiles/fp64_peak.json (tools/fp64_peak.cu DFMA loop, B200)"
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            fp = json.load(f)
        out["fp64_tflops"] = float(fp["dfma_tflops_best"])
    except Exception:
        pass
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_reference_arm(args, steps, warmup):
    """The reference's own CPU path for this workload.  The reference ships no
    3D stepper, so this is the oracle port (oracle/hlf_oracle.cpp,
    the d-dim restatement that is bit-identical to the compiled reference in 1D),
    run with every host thread on a bounded sample of the same 3D m=3 periodic
    mode.  Returns (DOF-updates/s, sample description, threads, ms per sample step)."""
    import numpy as np
    import oracle as O
    threads = os.cpu_count() or 1
    K = 24
    h = 2.0 / K
    o = O.OracleStepper(3, M, [K, K, K], h, threads=threads)
    pi = math.pi
    F = (M + 1) ** 3
    p = np.zeros((K ** 3, F))
    O.add_separable(3, [K] * 3, [-1.0] * 3, h, 0.0, M + 1, 1.0, [pi] * 3, [0.0] * 3, p)
    o.set_field(0, p)
    dt = CFL * h / math.sqrt(3.0)
    o.set_times(0.0, dt / 2, dt)
    for _ in range(warmup):
        o.advance_n(1)
    t0 = time.perf_counter()
    o.advance_n(steps)
    sec = time.perf_counter() - t0
    dof = 4 * F * K ** 3
    return (dof * steps / sec, f"oracle port, 3D m=3 periodic {K}^3 cells, {steps} steps after {warmup} warm-up",
            threads, sec / steps * 1e3)


def run_reference_impl(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    value, sample, threads, sample_ms = cpu_reference_arm(args, steps, warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        # one step = one leapfrog step of the bounded 24^3 sample (the metric is a rate)
        "steps": steps, "warmup": warmup, "ms_per_step": sample_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "3D acoustic Hermite-leapfrog m=3 periodic (CPU sample of the 512x512x256-per-GPU job)",
                   "m": M},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200")
    ap.add_argument("--nz", type=int, default=NZ_PER_GPU, help="z cells per GPU (default 256)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_impl(args)
        return
    if args.warmup < 3:
        args.warmup = 3

    import torch
    import torch.distributed as dist
    from paper_1808_10481_b200.distributed import SlabStepper

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nz = args.nz
    Kg = (NX, NY, nz * world)
    h = 2.0 / NX
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        st = SlabStepper(Kg, h, M, rank=rank, world=world, device=local, stream=stream)
        st.init_mode(CFL)
        dof_local = 4 * (M + 1) ** 3 * NX * NY * nz
        dof_total = dof_local * world
        # warm-up
        for i in range(args.warmup):
            st.step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches0 = st.launch_count()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            e0.record(stream)
            for i in range(args.steps):
                st.step(args.warmup + i)
            e1.record(stream)
            e1.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        launches = st.launch_count() - launches0
        bad = st.poll_finite()
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        value = dof_total / (ms * 1e-3)

        # per-kernel device times (separate instrumented pass, same stream)
        kt = st.kernel_times(2)
        pk = peaks()
        cells = NX * NY * nz
        pre_ms = kt["pre_ms"]
        vel_ms = kt["vel_ms"]
        # dominant single launch: the velocity half step (one tiled3d<3,3> launch,
        # 14976 algorithmic flop per cell); the pressure half step is two launches
        # (V_x+V_y merged, V_z) and is reported beside it
        vel_flops = FLOP_VEL_PER_CELL * cells
        achieved = vel_flops / (vel_ms * 1e-3) / 1e12
        pre_flops = FLOP_PRE_PER_CELL * cells
        step_flops = FLOP_PER_DOF * dof_local
        roofline = {
            "bound": "fp64", "unit": "TFLOP/s",
            "kernel": "tiled3d<3,3> (velocity half step, one launch per step)",
            "achieved": achieved, "peak": pk["fp64_tflops"], "frac": achieved / pk["fp64_tflops"],
            "peak_src": pk["fp64_src"], "traffic": None,
            "algorithmic_flop_per_launch": vel_flops,
            "share_of_step": vel_ms / (pre_ms + vel_ms),
            "pressure_half_step": {"launches": 2, "ms": pre_ms, "algorithmic_flop": pre_flops,
                                   "achieved_tflops": pre_flops / (pre_ms * 1e-3) / 1e12,
                                   "frac_fp64": pre_flops / (pre_ms * 1e-3) / 1e12 / pk["fp64_tflops"]},
            "step": {"achieved_tflops": step_flops / (ms * 1e-3) / 1e12,
                     "frac_fp64": step_flops / (ms * 1e-3) / 1e12 / pk["fp64_tflops"],
                     "hbm_gbs_algorithmic": BYTES_PER_DOF * dof_local / (ms * 1e-3) / 1e9,
                     "frac_hbm": BYTES_PER_DOF * dof_local / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                     "hbm_peak_gbs": pk["hbm_gbs"], "hbm_src": pk["hbm_src"]},
        }
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tr = json.load(f)
            roofline["traffic"] = tr.get("vel_dram_bytes_per_launch")
            roofline["traffic_src"] = tr.get("source")
        except Exception:
            pass

        # end to end through the C-ABI with pinned host buffers
        e2e = None
        if not args.no_e2e and world == 1:
            e2e = st.e2e(args.e2e_steps, dof_local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample, threads, _ = cpu_reference_arm(args, 2, 1)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"3D acoustic Hermite-leapfrog m={M}, periodic, {NX}x{NY}x{nz} cells per GPU "
                                   f"(global {Kg[0]}x{Kg[1]}x{Kg[2]}; 512^3 needs 256 GiB and does not fit one B200)",
                       "m": M, "cells_per_gpu": [NX, NY, nz], "global_cells": list(Kg),
                       "dof_per_step": dof_total, "parallelism": f"z-slab x{world}",
                       "l2": "state (128 GiB per GPU) far larger than L2; no flush needed",
                       "init": "standing mode of the periodic box, p = cos(wt t) prod sin(2 pi x_a / L_a) (512x512x256, h = 1/256: sin(pi x) sin(pi y) sin(2 pi z)), exact jets on device"},
            "gpu_launches": launches,
            "roofline": roofline,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "finite": bad < 0,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
