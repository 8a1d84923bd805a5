for l2 in 1 0; do
for s in "8320 384 1152" "8320 384 1536" "8320 384 384"; do
  echo "L2RED=$l2 $s"
  PPLL_CLUSTER_L2RED=$l2 PPLL_GEMM_TIMELINE=1 PPLL_GEMM_VERBOSE=1 python tools/wgrad_timeline.py $s 2>&1 | grep -v "^\[gemm" 
  PPLL_CLUSTER_L2RED=$l2 PPLL_GEMM_VERBOSE=1 python tools/gemm_graph.py $s wgrad 2>&1 | sort -u
done
done
python -m pytest tests/test_gpu_parity.py -q -x -k "wgrad or tcgen05 or linear" 2>&1 | tail -2
