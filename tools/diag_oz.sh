set -x
for mode in 0 1 2 3 8 9; do CCF_OZ_MODE=$mode timeout 300 python tools/oz_stage_times.py 2>&1 | grep -E "^mode|step:|profile:"; done
for tag in X3 X1 H C; do echo "== trace $tag"; CCF_OZ_MODE=4 CCF_OZ_TRACE=$tag timeout 300 python tools/oz_trace_ns.py 2>&1 | tail -60; done
timeout 900 ncu --profile-from-start off -k regex:oz_gemm --set full --import-source on --clock-control none -f -o gpurun_out/oz_full python tools/ncu_step.py > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
