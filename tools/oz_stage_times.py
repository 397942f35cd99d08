"""Diagnostics: per-stage times (CUDA events between stages, median of 5 eager profiled steps) of the
256^3 bench step. Used with CCF_OZ_MODE (oz_gemm diagnostic modes: bit 0 no epilogue math, bit 1 no
MMAs, bit 3 no stores) to see which part of the INT8 product kernel binds; results are wrong under any
mode != 0, only the timings mean something."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2206_04827_b200 as P  # noqa: E402

cfg = bench.CONFIGS[256]
ctx = P.Context(256, 256, 256)
wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
try:
    st.step(10)
except Exception as e:  # (diagnostic modes produce garbage; the step's non-finite guard may fire)
    print("step:", e)
runs = []
for _ in range(5):
    try:
        runs.append(st.profile_step())
    except Exception as e:
        print("profile:", e)
        break
if runs:
    keys = runs[0].keys()
    med = {k[:12]: round(statistics.median(r[k] for r in runs), 4) for k in keys}
    print("mode", os.environ.get("CCF_OZ_MODE", "0"), "total", round(sum(med.values()), 4), med)
