# tcgen05 engine throughput by operand layout at large sizes (is MN-major A slower?)
for op in fwd dgrad wgrad; do python tools/gemm_one.py 8192 8192 8192 $op 5 2>&1 | head -1; done
PPLL_GEMM_CLUSTER=0 python tools/gemm_one.py 8192 8192 8192 wgrad 5 2>&1 | head -1
# ViT-S wgrad shapes: cluster vs plain split-K
for sh in "8320 384 1152" "8320 384 1536" "8320 1536 384" "8320 384 384"; do python tools/gemm_one.py $sh wgrad 20 | head -1; PPLL_GEMM_CLUSTER=0 python tools/gemm_one.py $sh wgrad 20 | head -1; done
