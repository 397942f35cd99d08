import sys, ctypes
sys.path.insert(0, "/root/repo")
import bench, paper_2206_04827_b200 as P
cfg = bench.CONFIGS[256]
ctx = P.Context(256, 256, 256)
wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
st.step(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
ctx.synchronize()
P.lib().ccf_debug_oz_trace_dump()
