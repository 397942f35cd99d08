"""Profiling target: one graph-replayed steady-state NS step (bench configuration) between
cudaProfilerStart/Stop, for ncu --profile-from-start off (launch lists and --set full captures
of exactly one step, without setup, warm-up or the BDF ramp).

  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file launches.csv python tools/ncu_step.py [size]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2206_04827_b200 as P  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = bench.CONFIGS[size]
ctx = P.Context(cfg["m"], cfg["n"], cfg["p"])
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
st.step(12)  # BDF ramp + the five ring-phase graph captures
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
st.step(1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("launches per step:", st.launches_per_step())
