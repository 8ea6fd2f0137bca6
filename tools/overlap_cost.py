"""Cost of the z-slab overlap split at world = 1: the
same 512x512x256 m = 3 box stepped (a) by one plain solver (3 launches per
step) and (b) as one slab of the C++ host group with its halo exchanged
through the library (hlf_slabs_*: pressure interior + boundary layer,
velocity interior + boundary layer = 6 launches per step, plus the self
copies of the halo layers), device-timed with CUDA events.
Usage: python tools/overlap_cost.py [nz] [steps]"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1808_10481_b200 as H
from paper_1808_10481_b200.distributed import TRANSPORT_COPY, TRANSPORT_NCCL, SlabGroup

nz = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
K = (512, 512, nz)
h = 2.0 / 512
m = 3
dt = 0.9 * h / math.sqrt(3.0)
out = {"K": K, "m": m, "steps": steps}


def mode(s):
    w = [2 * math.pi / (k * h) for k in K]
    for f in range(4):
        s.zero_field(f)
    s.fill_separable(0, 1.0, w, [0.0] * 3)


def timed(fn):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


g = H.Stepper(H.Grid([-1.0] * 3, h, K), m)
mode(g)
g.set_times(0.0, dt / 2, dt)
g.advance_n(2)
out["plain_ms_per_step"] = timed(lambda: g.advance_n(steps))
out["plain_launches_per_step"] = 3
del g
torch.cuda.empty_cache()
for name, tr in (("slab_copy", TRANSPORT_COPY), ("slab_nccl", TRANSPORT_NCCL)):
    sg = SlabGroup(K, h, m, [0], transport=tr)
    s = sg._solver(0)
    for f in range(4):
        sg._L.hlf_zero_field(s, f)
    # the same mode as the plain solver (zero data would run at other clocks)
    import ctypes as C
    w3 = (C.c_double * 3)(*[2 * math.pi / (k * h) for k in K])
    p3 = (C.c_double * 3)(0.0, 0.0, 0.0)
    assert sg._L.hlf_fill_separable(s, 0, 1.0, w3, p3) == 0
    sg.set_times(0.0, dt / 2, dt)
    sg.advance_n(2)
    out[f"{name}_ms_per_step"] = timed(lambda: sg.advance_n(steps))
    sg.close()
    del sg
    torch.cuda.empty_cache()
out["slab_launches_per_step"] = 6
out["overhead_copy"] = out["slab_copy_ms_per_step"] / out["plain_ms_per_step"] - 1.0
out["overhead_nccl"] = out["slab_nccl_ms_per_step"] / out["plain_ms_per_step"] - 1.0
print(json.dumps(out))
