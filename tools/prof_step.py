"""Profile exactly one NS step (graph-replayed, as in bench.py) between cudaProfilerStart/Stop.

Use with `ncu --profile-from-start off ...`. Not a bench: numbers printed under ncu are not timings.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_2206_04827_b200 as P
    cfg = bench.CONFIGS[args.size]
    ctx = P.Context(cfg["m"], cfg["n"], cfg["p"], device=0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
    st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
    st.step(args.warmup)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    st.step(args.steps)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled", args.steps, "step(s) at", args.size)


if __name__ == "__main__":
    main()
