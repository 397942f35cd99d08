#!/bin/bash
# Quick GPU-box check used between changes: NS parity against the oracle (tests/tools/gpu_check_ns.py)
# and one short bench line with the per-stage times. Run under gpurun from the repo root.
python tests/tools/gpu_check_ns.py > gpurun_out/ns.log 2>&1; echo "gpu_check_ns rc=$?"; grep "NS step" gpurun_out/ns.log | tail -4
python bench.py --steps 30 --warmup 10 --no-cpu-baseline > gpurun_out/bench.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1),round(d['ms_per_step'],4),d['gpu_launches'],{k[:3]:round(x,4) for k,x in d['stage_ms'].items()})"
