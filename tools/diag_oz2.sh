# quick INT8-GEMM iteration check: Ozaki unit tests, per-stage times, block-0 traces of X3 and X1
python -m pytest tests/test_gpu_ozaki.py -x -q 2>&1 | tail -3
CCF_OZ_MODE=0 timeout 300 python tools/oz_stage_times.py 2>&1 | grep -E "^mode|step:|profile:"
for m in ${OZ_MODES:-}; do CCF_OZ_MODE=$m timeout 300 python tools/oz_stage_times.py 2>&1 | grep -E "^mode|step:|profile:"; done
for tag in ${OZ_TAGS:-X3 X1}; do echo "== trace $tag"; CCF_OZ_MODE=4 CCF_OZ_TRACE=$tag timeout 300 python tools/oz_trace_ns.py 2>&1 | tail -${OZ_TAIL:-20}; done
