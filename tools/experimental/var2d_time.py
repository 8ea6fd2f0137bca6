"""Device timing of the config-3 variable-coefficient step (var2d kernel).
Usage: python tools/experimental/var2d_time.py m [K] [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_configs as B
m = int(sys.argv[1]); K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
import io, contextlib
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    r = B.run("cfg3", 2, m, [K, K], boundary=[1, 1], variable=True, steps=steps)
print(f"m={m} K={K} ms/step={r['ms_per_step']:.3f} DOF/s={r['dof_updates_per_s']:.3e}")
