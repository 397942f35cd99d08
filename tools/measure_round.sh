# Full GPU check of HEAD: GPU test suite, smoke, bench line, ncu launch list of one graph-replayed step and
# one --set full capture of that step (run under gpurun from the repo root; outputs in gpurun_out/)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1), d['gpu_launches'], d['roofline']['frac'])"
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/ncu_step.py > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
[ -n "$FULL" ] && { ncu --profile-from-start off --set full --import-source on --clock-control none -f -o gpurun_out/step_full python tools/ncu_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"; }
true
