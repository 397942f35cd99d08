# per-stage times of the 256^3 step, three independent runs (noise check)
for i in 1 2 3; do timeout 300 python tools/oz_stage_times.py 2>&1 | grep -E "^mode"; done
