#!/bin/bash
# Diagnostics: per-stage times of the bench step under the oz_gemm kernel's diagnostic modes
# (CCF_OZ_MODE bit 0: no epilogue math, bit 1: no MMAs, bit 3: no stores). Results are wrong
# under any mode != 0; only the timings mean something. Run under gpurun from the repo root.
for mode in 0 1 2 3 8 9 11; do
  CCF_OZ_MODE=$mode python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/mode$mode.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/mode$mode.json').read().strip().splitlines()[-1]);print('mode $mode', round(d['ms_per_step'],4),{k:round(x,4) for k,x in d['stage_ms'].items()})" 2>&1 | tail -1
done
