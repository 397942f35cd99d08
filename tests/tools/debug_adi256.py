import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', '..'))
import numpy as np
import paper_2206_04827_b200 as P
from oracle import pyoracle as O
from bench import CONFIGS, initial_vorticity
from tests.inputs import rel_err
m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = dict(CONFIGS[256]); cfg.update(m=m, n=m, p=m)
ctx = P.Context(m, m, m)
wl, wg, vmax = initial_vorticity(ctx, cfg)
print("vmax", vmax, "max|wl|", np.abs(wl).max(), "max|wg|", np.abs(wg).max(), flush=True)
half = m // 2
for wsel in [0, 1, 2, 5]:
    f = np.zeros_like(wl)
    f[half + wsel] = -wl[half + wsel]
    if wsel: f[half - wsel] = -wl[half - wsel]
    try:
        u = ctx.solve_poisson_3d(f); ok = "ok"
    except P.CCFError as e:
        u = None; ok = f"FAIL {e} hist {e.residual_history}"
    t0 = time.time()
    try:
        uo = O.poisson3d(f); ook = "ok"
    except O.OracleError as e:
        uo = None; ook = f"FAIL {e}"
    st = O.adi_stats()
    print(f"w={wsel}: gpu {ok}; oracle {ook} ({time.time()-t0:.1f}s) stats {st}", flush=True)
    if u is not None and uo is not None:
        print(f"   rel_err {rel_err(u, uo):.3e}", flush=True)
    O.adi_stats_reset()
# Helmholtz (BDF1 scale) on the same data
sc = 1.0 * cfg["h"] / cfg["reynolds"]
for wsel in [0, 1]:
    f = np.zeros_like(wl)
    f[half + wsel] = wl[half + wsel]
    if wsel: f[half - wsel] = wl[half - wsel]
    try:
        u = ctx.helmholtz_step([f], 1, 1.0 / cfg["reynolds"], cfg["h"]); ok = "ok"
    except P.CCFError as e:
        u = None; ok = f"FAIL {e} hist {e.residual_history}"
    try:
        uo = O.helmholtz_step([f], 1, 1.0 / cfg["reynolds"], cfg["h"]); ook = "ok"
    except O.OracleError as e:
        uo = None; ook = f"FAIL {e}"
    print(f"helm w={wsel}: gpu {ok}; oracle {ook} stats {O.adi_stats()}", flush=True)
    if u is not None and uo is not None:
        print(f"   rel_err {rel_err(u, uo):.3e}", flush=True)
    O.adi_stats_reset()
