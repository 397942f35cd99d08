"""Where the e2e time of a fresh NSStepper goes (creation, ramp, graph captures, transfers)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    import paper_2206_04827_b200 as P
    cfg = bench.CONFIGS[256]
    ctx = P.Context(cfg["m"], cfg["n"], cfg["p"], device=0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
    st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
    st.step(12)
    torch.cuda.synchronize()
    hl = torch.from_numpy(np.ascontiguousarray(wl)).pin_memory()
    hg = torch.from_numpy(np.ascontiguousarray(wg)).pin_memory()
    pl = torch.empty_like(hl).pin_memory()
    pg = torch.empty_like(hg).pin_memory()
    for rep in range(2):
        t0 = time.perf_counter()
        s2 = P.NSStepper(ctx, hl.numpy(), hg.numpy(), reynolds=cfg["reynolds"], h=cfg["h"], order=4)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        for k in range(10):
            s2.step(1)
            torch.cuda.synchronize()
            print(f"  rep {rep} step {k}: {1e3 * (time.perf_counter() - t1):.1f} ms cumulative", flush=True)
        t2 = time.perf_counter()
        s2.step(40)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        ol, og = s2.omega(pl.numpy(), pg.numpy())
        t4 = time.perf_counter()
        print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, first 10 steps {1e3*(t2-t1):.1f} ms, next 40 {1e3*(t3-t2):.1f} ms, omega D2H {1e3*(t4-t3):.1f} ms", flush=True)
        s2.close()


if __name__ == "__main__":
    main()
