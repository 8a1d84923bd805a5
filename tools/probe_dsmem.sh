for bpc in 64 32 20 12; do
  echo "PPLL_DSMEM_BPC=$bpc"
  for s in "8320 384 1152" "8320 384 1536" "8320 1536 384" "8320 384 384"; do
    PPLL_DSMEM_BPC=$bpc PPLL_GEMM_VERBOSE=1 python tools/gemm_graph.py $s wgrad 2>&1 | sort -u | tr '\n' ' '; echo
  done
done
