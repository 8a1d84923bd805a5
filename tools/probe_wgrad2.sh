# fixed cost vs K of the cluster split-K weight gradient (ViT-S qkv / fc1 / proj shapes)
for m in 1040 2080 4160 8320 16640 33280; do
  PPLL_GEMM_VERBOSE=1 python tools/gemm_one.py $m 384 1152 wgrad 20 2>&1 | sort -u | tr '\n' ' '; echo
done
for m in 1040 4160 8320 33280; do
  PPLL_GEMM_VERBOSE=1 python tools/gemm_one.py $m 384 384 wgrad 20 2>&1 | sort -u | tr '\n' ' '; echo
  PPLL_GEMM_VERBOSE=1 python tools/gemm_one.py $m 384 1536 wgrad 20 2>&1 | sort -u | tr '\n' ' '; echo
done
