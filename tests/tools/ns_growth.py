"""Step the NS solver (GPU) and print max|omega| per step + ADI iterations; optionally compare with the oracle."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', '..'))
import numpy as np
import paper_2206_04827_b200 as P
from bench import CONFIGS, initial_vorticity
from tests.inputs import rel_err
size = int(sys.argv[1]); nsteps = int(sys.argv[2]); oracle_steps = int(sys.argv[3]) if len(sys.argv) > 3 else 0
vt = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
cfg = CONFIGS[size]
ctx = P.Context(cfg["m"], cfg["n"], cfg["p"])
wl, wg, vmax = initial_vorticity(ctx, cfg, vt)
print('vmax target', vt)
print(f"size {size} vmax {vmax:.3e} |wl| {np.abs(wl).max():.3e} |wg| {np.abs(wg).max():.3e}", flush=True)
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
st.set_graphs(False)
ons = None
if oracle_steps:
    from oracle import pyoracle as O
    O.set_threads(os.cpu_count())
    ons = O.NSStepper(wl, wg, cfg["reynolds"], cfg["h"])
for s in range(1, nsteps + 1):
    ctx.reset_stats()
    try:
        st.step(1)
    except P.CCFError as e:
        print(f"step {s}: GPU FAIL {type(e).__name__}: {e} hist {e.residual_history}", flush=True)
        break
    l, g = st.omega()
    it = ctx.stats()["adi_iterations"]
    line = f"step {s}: max|lam| {np.abs(l).max():.3e} max|gam| {np.abs(g).max():.3e} adi_iters {it}"
    if ons is not None and s <= oracle_steps:
        t0 = time.time()
        try:
            ons.step(1)
            rl, rg = ons.omega()
            line += f" | oracle {time.time()-t0:.1f}s rel {rel_err(l, rl):.2e} {rel_err(g, rg):.2e} max|lam| {np.abs(rl).max():.3e}"
        except Exception as e:
            line += f" | oracle FAIL {e}"
            ons = None
    print(line, flush=True)
