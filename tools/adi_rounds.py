"""Per-slot ADI round counts / residual histories of the NS Poisson and Helmholtz solves at 256^3."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    import paper_2206_04827_b200 as P
    size = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    cfg = bench.CONFIGS[size]
    m, n, p = cfg["m"], cfg["n"], cfg["p"]
    ctx = P.Context(m, n, p, device=0)
    wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
    ctx.velocity_from_vorticity(wl, wg)
    r, h = ctx.adi_last_rounds()
    print("velocity_from_vorticity Poisson rounds histogram:", np.bincount(r.ravel(), minlength=5)[1:])
    for s in range(r.shape[1]):
        if r[0, s] > 1:
            print(f"  slot {s:4d} w {s - p // 2:5d} rounds {r[0, s]} hist {h[0, s, :r[0, s]]}")
    st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
    st.set_graphs(False)
    ctx.adi_keep_history(True)
    for k in range(8):
        st.step(1)
        for which, name in ((1, "Poisson"), (2, "Helmholtz")):
            r, h = ctx.adi_last_rounds(which)
            print(f"step {k} NS {name} rounds histogram:", np.bincount(r.ravel(), minlength=5)[1:],
                  "worst first-round residual", h[:, :, 0].max())
            for t in range(r.shape[0]):
                for s in range(r.shape[1]):
                    if r[t, s] > 1:
                        print(f"    tensor {t} slot {s:4d} rounds {r[t, s]} hist {h[t, s, :r[t, s]]}")


if __name__ == "__main__":
    main()
