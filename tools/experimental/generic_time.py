"""Device timing of the generic (faithful) kernel: python generic_time.py d m K [variable]"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1808_10481_b200 as H
d, m, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
variable = len(sys.argv) > 4 and sys.argv[4] == "1"
g = H.Stepper(H.Grid([-1.0] * d, 2.0 / K, (K,) * d), m, variable_ap=variable)
g.kernel_variant = 0
pi = math.pi
g.fill_separable(0, 1.0, [pi] * d, [0.0] * d)
if variable:
    for grid in (0, 1):
        jets = np.zeros((g.num_nodes(grid), g.E))
        jets[:, 0] = -1.0
        jets[:, 1] = -0.01
        g.set_coeff(grid, jets)
dt = 0.5 * g.grid.h / math.sqrt(d)
g.set_times(0.0, dt / 2, dt)
g.advance_n(1)
torch.cuda.synchronize()
t0 = time.perf_counter()
steps = 3
g.advance_n(steps)
ms = (time.perf_counter() - t0) / steps * 1e3
dof = (d + 1) * (m + 1) ** d * K ** d
print(f"generic d={d} m={m} K={K} var={variable} ms/step={ms:.2f} DOF/s={dof / ms * 1e3:.3e}")
