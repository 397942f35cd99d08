# CTA-pair INT8 GEMM checks + timings (tools/cpp/oz_pair_check)
B=tools/cpp/oz_pair_check
for a in "1 1 0 0 0.9" "1 1 1 0 0.9" "1 3 0 0 0.9" "1 1 0 1 0.9" "1 2 1 1 0.9" "74 1 0 0 0.9" "300 2 0 0 0.8" "300 2 1 1 0.8"; do timeout 60 $B $a | grep -v "^ "; done
echo "== timings"
timeout 60 $B 1290 1 2 0 0.9 20 | grep pair     # X3-like: 2580 single-term panel tiles
timeout 60 $B 1548 1 2 0 0.9 20 | grep pair    # H-like: 3096 single-term panel tiles
timeout 60 $B 1548 2 1 1 0.9 20 | grep pair    # X1-like: 3096 tiles of 2 terms, MN-major A, transposed fp64
for m in ${OZ_MODES:-1 2 3 35}; do echo "mode $m"; CCF_OZ_MODE=$m timeout 60 $B 1290 1 2 0 0.9 20 | grep pair; CCF_OZ_MODE=$m timeout 60 $B 1548 2 1 1 0.9 20 | grep pair; done
[ -n "$OZ_TRACE" ] && CCF_OZ_MODE=4 timeout 60 $B $OZ_TRACE
