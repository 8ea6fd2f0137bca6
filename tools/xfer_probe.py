"""Host<->device transfer rates of hlf_set_field / hlf_get_field (pinned host AoS, one 34 GB field)."""
import time, torch, numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1808_10481_b200 as H
g = H.Stepper(H.Grid([-1.0]*3, 2/512, (512, 512, 256)), 3)
n = g.field_nodes(0) * g.F
buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.set_field_ptr(0, buf.data_ptr()); t1 = time.perf_counter()
    g.get_field_ptr(0, buf.data_ptr()); t2 = time.perf_counter()
    print(f"H2D {n*8/(t1-t0)/1e9:.1f} GB/s  D2H {n*8/(t2-t1)/1e9:.1f} GB/s  ({n*8/1e9:.1f} GB)")
