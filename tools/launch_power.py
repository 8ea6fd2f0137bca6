"""SM clock and board power while one half step runs back to back (3D m = 3,
512x512x256 unless given): is a launch power-capped, and at what clock?
Each half step alone for ~4 s under nvidia-smi sampling (200 ms).
Usage: python tools/launch_power.py [m] [KxKyKz]"""
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1808_10481_b200 as H

m = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "512x512x256").split("x"))
KINDS = sys.argv[3].split(",") if len(sys.argv) > 3 else ["vel", "pre", "step"]


class Smi:
    def __init__(self):
        self.rows, self._stop = [], threading.Event()

    def run(self):
        while not self._stop.is_set():
            out = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
            p = [x.strip() for x in out.strip().split(",")]
            if len(p) == 3:
                self.rows.append(p)
            self._stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()


stream = torch.cuda.Stream()
g = H.Stepper(H.Grid([-1.0] * 3, 2.0 / K[0], K), m, stream=stream.cuda_stream)
pi = math.pi
g.fill_separable(0, 1.0, [pi] * 3, [0.0] * 3)
for c in range(1, 4):
    g.fill_separable(c, -0.1, [pi] * 3, [pi / 2 if a == c - 1 else 0.0 for a in range(3)])
dt = 0.9 * g.grid.h / math.sqrt(3)
res = {"m": m, "K": K}
for name in KINDS:
    # forward then backward in time keeps the data bounded (dt -> -dt)
    g.set_times(0, dt / 2, dt)
    raw = {"vel": g.advance_v, "pre": g.advance_p, "step": lambda: g.step_system(0)}[name]

    def fn(raw=raw):
        try:  # ablation builds (HLF_EXP_*) produce garbage: time them anyway
            raw()
        except H.InstabilityError:
            g.clear_finite()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    with Smi() as s:
        t0 = time.time()
        e0.record(stream)
        while time.time() - t0 < 4.0:
            for _ in range(4):
                fn()
                n += 1
            torch.cuda.synchronize()
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    load = [r for r in s.rows[2:] if float(r[1]) > 200]
    res[name] = {"ms": round(ms, 3), "sm_mhz_median": statistics.median(float(r[0]) for r in load) if load else None,
                 "power_w_median": statistics.median(float(r[1]) for r in load) if load else None,
                 "power_cap_frac": round(sum(r[2] == "Active" for r in load) / max(1, len(load)), 2),
                 "joules": round(ms * 1e-3 * statistics.median(float(r[1]) for r in load), 2) if load else None,
                 "samples": len(load)}
print(json.dumps(res))
