python tools/gpu_check_ns.py > gpurun_out/ns.log 2>&1; echo rc=$?; grep "NS step" gpurun_out/ns.log | tail -4
python bench.py --steps 30 --warmup 5 > gpurun_out/bench.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['gpu_launches'],d['stage_ms'])"
