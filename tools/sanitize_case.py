"""Smallest grids on the TMA box path of the tiled kernels, for
compute-sanitizer racecheck / synccheck / memcheck runs:
  3D m = 3, K = [64, 2, 4]: both x tiles load their rows as TMA boxes (the
  x0 = 0 pressure tile and the last velocity tile through the one-node patch),
  the targets arrive as TMA boxes; merged V_x + V_y and V_z pressure launches
  and the velocity launch, 2 steps;
  2D m = 3, K = [64, 8], 2 steps.
Prints the path counters so the log shows which loaders ran."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1808_10481_b200 as H

for d, K in ((3, [64, 2, 4]), (2, [64, 8])):
    g = H.Stepper(H.Grid([-1.0] * d, 2.0 / K[0], tuple(K)), 3)
    rng = np.random.default_rng(0)
    for f in range(d + 1):
        g.set_field(f, rng.standard_normal((g.field_nodes(f), g.F)))
    g.enable_path_counters()
    g.set_times(0.0, 0.005, 0.01)
    g.advance_n(2)
    g.synchronize()
    print(d, K, g.path_counters(), flush=True)
