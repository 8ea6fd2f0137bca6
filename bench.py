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
              "clocks_event_reasons.sw_power_cap,power.draw,power.limit")

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
                if len(parts) == 8:
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
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        pw = [x for x in (num(s[6]) for s in self.samples) if x is not None]
        pl = [x for x in (num(s[7]) for s in self.samples) if x is not None]
        # board power next to the clocks: the 3D m = 3 launches run at the
        # power limit (profiles/r2b/launch_power.json)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_median": statistics.median(pw) if pw else None, "power_limit_w": max(pl) if pl else None}


# Algorithmic work per cell of the three launches of one 3D m = 3 step
# (DESIGN.md sec. 4).  Bytes are the compulsory
# HBM traffic of the bulk-synchronous contract (each coefficient read once per
# launch that needs it, targets read and written once), flops the minimal
# sum-factorised formulation.  The pressure half step's algorithm (one CK of
# the divergence, one read-modify-write of p: 27648 flop, 2560 B per cell) is
# split over its two launches so that they sum to the half step.
R3 = 8064.0   # one reconstruction (L = 112 lines x (n + n^2))
LAUNCHES = {
    "vel": [{"kernel": "tiled3d<3,3> velocity (p -> v_x, v_y, v_z)",
             "bytes": 512.0 + 3 * 1024.0, "flops": FLOP_VEL_PER_CELL}],
    "pre": [{"kernel": "tiled3d<3,2> pressure, V_x + V_y merged (-> p)",
             "bytes": 2 * 512.0 + 1024.0, "flops": 2 * R3 + 512.0 + 2 * 1184.0 + 64.0},
            {"kernel": "tiled3d<3,1> pressure, V_z (-> p)",
             "bytes": 512.0, "flops": R3 + 512.0}],
}


def roofline_block(kt, pk, cells, step_ms, dof_local):
    """Per-launch and per-half-step rooflines: each bound = max(bytes / HBM,
    flops / FP64) (whichever takes longer binds); `frac` = that ceiling time
    over the measured time.  The top level describes the dominant launch."""
    hbm = pk["hbm_gbs"] * 1e9
    fp = pk["fp64_tflops"] * 1e12
    launches = []
    half = {}
    for kind, specs in LAUNCHES.items():
        tms = kt[kind]
        hb = sum(x["bytes"] for x in specs) * cells
        hf = sum(x["flops"] for x in specs) * cells
        t_meas = sum(tms[: len(specs)]) * 1e-3
        t_ceil = max(hb / hbm, hf / fp)
        half[kind] = {"launches": len(specs), "ms": t_meas * 1e3, "algorithmic_bytes": hb,
                      "algorithmic_flop": hf, "bound": "hbm" if hb / hbm >= hf / fp else "fp64",
                      "ceiling_ms": t_ceil * 1e3, "frac": t_ceil / t_meas,
                      "hbm_gbs": hb / t_meas / 1e9, "fp64_tflops": hf / t_meas / 1e12}
        for spec, t in zip(specs, tms):
            b, f = spec["bytes"] * cells, spec["flops"] * cells
            tb, tf = b / hbm, f / fp
            sec = t * 1e-3
            bound = "hbm" if tb >= tf else "fp64"
            launches.append({
                "kernel": spec["kernel"], "half_step": kind, "ms": t,
                "algorithmic_bytes": b, "algorithmic_flop": f,
                "intensity_flop_per_byte": f / b, "ridge_flop_per_byte": fp / hbm,
                "bound": bound, "achieved_gbs": b / sec / 1e9, "achieved_tflops": f / sec / 1e12,
                "frac_hbm": tb / sec, "frac_fp64": tf / sec, "frac": max(tb, tf) / sec})
    dom = max(launches, key=lambda x: x["ms"])
    hbm_bound = dom["bound"] == "hbm"
    top = {
        "bound": "hbm" if hbm_bound else "tensor",  # FP64 runs on the DFMA pipe; "tensor" = compute-bound
        "compute_pipe": None if hbm_bound else "fp64 (DFMA)",
        "kernel": dom["kernel"],
        "unit": "GB/s" if hbm_bound else "TFLOP/s",
        "achieved": dom["achieved_gbs"] if hbm_bound else dom["achieved_tflops"],
        "peak": pk["hbm_gbs"] if hbm_bound else pk["fp64_tflops"],
        "frac": dom["frac"],
        "peak_src": pk["hbm_src"] if hbm_bound else pk["fp64_src"],
        "algorithmic_per_launch": dom["algorithmic_bytes"] if hbm_bound else dom["algorithmic_flop"],
        "per_unit": "3584 B/cell (read p, read+write v_x,v_y,v_z: 7 x 512 B)" if hbm_bound else "flop/cell",
        "share_of_step": dom["ms"] / step_ms,
        "traffic": None,
        "launches": launches,
        "half_steps": half,
    }
    ceil_ms = sum(h["ceiling_ms"] for h in half.values())
    top["step"] = {
        "ms": step_ms,
        "ceiling_ms_per_half_step_sum": ceil_ms, "frac_per_half_step_ceiling": ceil_ms / step_ms,
        "ceiling_ms_aggregate": max(BYTES_PER_DOF * dof_local / hbm, FLOP_PER_DOF * dof_local / fp) * 1e3,
        "frac_aggregate": max(BYTES_PER_DOF * dof_local / hbm, FLOP_PER_DOF * dof_local / fp) * 1e3 / step_ms,
        "achieved_tflops": FLOP_PER_DOF * dof_local / (step_ms * 1e-3) / 1e12,
        "hbm_gbs_algorithmic": BYTES_PER_DOF * dof_local / (step_ms * 1e-3) / 1e9,
        "hbm_peak_gbs": pk["hbm_gbs"], "fp64_peak_tflops": pk["fp64_tflops"],
    }
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        per = {x["kernel"].split("tiled3d<")[-1].split(">")[0].replace(" ", ""): x["bytes_per_cell"] for x in tr["launches"]}
        key = dom["kernel"].split("tiled3d<")[-1].split(">")[0]
        if key in per:
            top["traffic"] = per[key] * cells
            top["traffic_src"] = tr.get("source", "") + "; per-cell DRAM bytes x cells"
    except Exception:
        pass
    return top


def cpu_reference_arm(quick: bool = False):
    """The reference's own CPU path, timed on this host:
    the compiled reference's Stepper1d (oracle/_ref, /root/reference/proj/src
    unchanged) is the only stepper the reference implements (1D), run as
    `nproc` concurrent independent instances at K = 2^20, m = 3 (its
    concurrency model); the oracle port (oracle/hlf_oracle.cpp)
    runs the bench's own 3D m = 3 periodic mode at 64^3 with every host thread
    (same config, out of cache).  Returns (value, cpu_baseline dict)."""
    from oracle import cpu_baseline as B
    plan = B.full_plan(quick=quick)
    host = plan["host"]
    if "ref_stepper1d_K2^20_nproc_instances" in plan:
        leg = plan["ref_stepper1d_K2^20_nproc_instances"]
        value = leg["dof_per_s"]
        cb = {"value": value, "unit": UNIT, "cores": leg["instances"], "kind": "reference",
              "sample": f"the reference's own Stepper1d::step_system (oracle/_ref), 1D m=3 K=2^20, "
                        f"{leg['instances']} concurrent instances x {leg['steps']} steps (the reference has no 2D/3D "
                        f"stepper, so its config differs from the 3D bench workload)",
              "same_config": False}
    else:
        leg = plan["oracle_3d_m3_64^3_all_threads"]
        value = leg["dof_per_s"]
        cb = {"value": value, "unit": UNIT, "cores": leg["threads"], "kind": "port",
              "sample": f"oracle port, 3D m=3 periodic 64^3, {leg['steps']} steps", "same_config": True}
    port = plan["oracle_3d_m3_64^3_all_threads"]
    cb["port_3d_same_config"] = {"value": port["dof_per_s"], "cores": port["threads"], "kind": "port",
                                 "sample": f"oracle port (bit-identical to the reference in 1D), 3D m=3 periodic "
                                           f"64^3 = 4 x 134 MB of state, {port['steps']} steps, OpenMP"}
    cb["cpu_model"] = host["cpu_model"]
    cb["nproc"] = host["nproc"]
    cb["plan"] = plan
    return value, cb


def run_reference_impl(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    value, cb = cpu_reference_arm()
    plan = cb["plan"]
    leg = plan.get("ref_stepper1d_K2^20_nproc_instances")
    sec_per_step = leg["max_instance_seconds"] / leg["steps"] if leg else plan["oracle_3d_m3_64^3_all_threads"]["seconds"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        # one step = one leapfrog step of the bounded CPU sample (the metric is a rate)
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec_per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "3D acoustic Hermite-leapfrog m=3 periodic (CPU: the reference's own 1D Stepper1d, "
                               "and the oracle port on 64^3 of the same 3D mode)", "m": M},
        "cpu_baseline": cb,
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
    ap.add_argument("--configs", action="store_true",
                    help="instead of the headline line: one JSON line (with clocks) per SURVEY.md sec. 8(d) "
                         "configuration, tools/bench_configs.py")
    args = ap.parse_args()
    if args.configs:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_configs
        sys.argv = [sys.argv[0]]
        bench_configs.main()
        return
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

        # per-launch device times (separate instrumented pass on the solver
        # stream: hlf_time_launches records CUDA events around every kernel)
        kt = st.kernel_times(2)
        pk = peaks()
        cells = NX * NY * nz
        roofline = roofline_block(kt, pk, cells, ms, dof_local)

        # end to end through the C-ABI with pinned host buffers (every rank
        # its slab; N > 1 only when the node's host memory holds all ranks'
        # pinned states, 128 GiB each at the default size)
        e2e = None
        e2e_note = None
        if not args.no_e2e:
            ok = True
            if world > 1:
                need = world * dof_local * 8 * 1.15
                try:
                    with open("/proc/meminfo") as f:
                        avail = next(int(l.split()[1]) * 1024 for l in f if l.startswith("MemAvailable:"))
                except (OSError, StopIteration, ValueError):
                    avail = 0
                flag = torch.tensor([1 if avail >= need else 0], device="cuda")
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                ok = bool(flag.item())
                if not ok:
                    e2e_note = (f"e2e skipped: {world} ranks x {dof_local * 8 / 2**30:.0f} GiB of pinned host state "
                                f"exceed the node's available host memory ({avail / 2**30:.0f} GiB)")
                else:
                    dist.barrier()
            if ok:
                e2e = st.e2e(args.e2e_steps, dof_local)
                if world > 1:
                    t = torch.tensor([e2e["job"]["seconds"]], device="cuda")
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the slowest rank ends the job
                    sec = float(t.item())
                    e2e["job"]["seconds"] = sec
                    e2e["value"] = dof_total * args.e2e_steps / sec
                    e2e["h2d_bytes_per_step"] *= world
                    e2e["d2h_bytes_per_step"] *= world
                    e2e["job"]["h2d_bytes"] *= world
                    e2e["job"]["d2h_bytes"] *= world
                    e2e["job"]["ranks"] = world

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        _, cpu = cpu_reference_arm()

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
            **({"e2e_note": e2e_note} if e2e_note else {}),
            "cpu_baseline": cpu,
            "finite": bad < 0,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
