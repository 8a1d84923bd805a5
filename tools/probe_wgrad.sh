# MN-major-operand rate probe: the same 8192^3 contraction as fwd (A K-major, B MN-major),
# dgrad (both K-major) and wgrad (both MN-major); then the ViT-S wgrad shapes, cluster on/off
for op in fwd dgrad wgrad; do python tools/gemm_one.py 8192 8192 8192 $op 5; done
for s in "8320 384 1152" "8320 384 1536" "8320 1536 384" "8320 384 384"; do
  PPLL_GEMM_VERBOSE=1 python tools/gemm_one.py $s wgrad 20 2>&1 | sort -u | tail -2
  PPLL_GEMM_CLUSTER=0 python tools/gemm_one.py $s wgrad 20
done
