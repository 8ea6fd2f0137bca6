"""Quick device timing of the half-step kernels (CUDA events via torch on the
solver's stream). Usage: python tools/time_kernel.py d m K [steps] [variant]"""
import sys, os, math, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1808_10481_b200 as H

d, m = int(sys.argv[1]), int(sys.argv[2])
Ks = [int(x) for x in sys.argv[3].split("x")]
Ks = Ks if len(Ks) == d else Ks * d
K = Ks[0]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
variant = int(sys.argv[5]) if len(sys.argv) > 5 else -1
stream = torch.cuda.Stream()
var = os.environ.get("HLF_VAR_SEP") is not None  # variable c^2 = 1 + prod sin / 2 (var2d / var3d)
g = H.Stepper(H.Grid([-1.0] * d, 2.0 / K, tuple(Ks)), m, stream=stream.cuda_stream, variable_ap=var)
if var:
    g.set_coeff_separable(1.0, 0.5, [math.pi] * d, [0.0] * d)
if variant >= 0:
    g.kernel_variant = variant
pi = math.pi
g.fill_separable(0, 1.0, [pi] * d, [0.0] * d)
for c in range(1, d + 1):
    g.fill_separable(c, -0.1, [pi] * d, [pi / 2 if a == c - 1 else 0.0 for a in range(d)])
dt = 0.9 * g.grid.h / math.sqrt(d)
g.set_times(0, dt / 2, dt)
# HLF_EXP_* ablation builds produce garbage: time them without the finite check
check = os.environ.get("HLF_NOCHECK") is None
def run(k):
    try:
        g.advance_n(k)
    except H.InstabilityError:
        if check:
            raise
run(2)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(stream)
run(steps)
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / steps
dof = (d + 1) * (m + 1) ** d * math.prod(Ks)
tl = g.time_launches(2, 1000) if d > 1 else {}
lt = " ".join(f"{k}=" + "/".join(f"{x:.2f}" for x in v) for k, v in tl.items())
print(f"d={d} m={m} K={Ks} variant={g.kernel_variant} ms/step={ms:.3f} DOF/s={dof / ms * 1e3:.3e} "
      f"GB/s(24B/DOF)={24 * dof / ms / 1e6:.1f} launches_ms: {lt}")
