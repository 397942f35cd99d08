"""Stability / speed probe of a bench configuration: max |omega| coefficient per step and steps/s.
  python tools/ns_probe.py SIZE VMAX STEPS"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2206_04827_b200 as P  # noqa: E402

size, vmax, steps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
cfg = dict(bench.CONFIGS[size])
t0 = time.time()
ctx = P.Context(cfg["m"], cfg["n"], cfg["p"])
wl, wg, v0 = bench.initial_vorticity(ctx, cfg, vmax)
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
print(f"setup {time.time() - t0:.1f} s, unscaled max|v| {v0:.3e}, max|omega0| {np.abs(wl).max():.3e} {np.abs(wg).max():.3e}",
      flush=True)
for k in range(steps):
    try:
        st.step(1)
    except P.CCFError as e:
        print("step", k + 1, "failed:", e)
        break
    if k < 5 or (k + 1) % 5 == 0:
        l, g = st.omega()
        print(f"step {k + 1}: max|lam| {np.abs(l).max():.4e} max|gam| {np.abs(g).max():.4e}", flush=True)
torch.cuda.synchronize()
t0 = time.time()
st.step(10)
torch.cuda.synchronize()
print(f"{10 / (time.time() - t0):.1f} steps/s (wall, graph replay)")
