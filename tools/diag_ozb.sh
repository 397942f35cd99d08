# INT8 GEMM microbenchmark (tools/cpp/oz_check) at the NS-step shapes under the kernel's diagnostic modes
# (bit 0 no epilogue math, bit 1 no MMAs, bit 3 no fp64 stores, bit 5 no panel stores); timing only
B=tools/cpp/oz_check
for m in ${OZ_MODES:-0 1 2 3 32 34 35}; do
  echo "mode $m X3-like (2580 single-term panel tiles, shared B):"; CCF_OZ_NOCHECK=1 CCF_OZ_PANEL=1 CCF_OZ_MODE=$m $B 128 128 128 2580 1 0.9 20 2 | grep split
  echo "mode $m X1-like (1548 x 2 tiles of 2 terms, fp64 out, MN-major B):"; CCF_OZ_NOCHECK=1 CCF_OZ_MN=1 CCF_OZ_MODE=$m $B 128 256 128 1548 2 0.9 20 | grep split
done
