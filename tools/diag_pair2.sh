B=tools/cpp/oz_pair_check
for a in "1 1 0 0 0.9" "74 1 0 0 0.9" "300 1 1 1 0.8" "1 1 0 1 0.9"; do CCF_OZ_BRES=1 timeout 60 $B $a | grep -v "^ "; done
for a in "1 3 0 0 0.9" "300 2 1 1 0.8"; do timeout 60 $B $a | grep -v "^ "; done
for m in 0 1 2 3 32 35; do echo "mode $m"; CCF_OZ_MODE=$m timeout 60 $B 1290 1 2 0 0.9 20 | grep pair; CCF_OZ_BRES=1 CCF_OZ_MODE=$m timeout 60 $B 1290 1 2 0 0.9 20 | grep pair; done
