for m in 1040 4160 8320 33280; do python tools/gemm_graph.py $m 384 1152 wgrad fwd; done
python tools/gemm_graph.py 8320 384 1536 wgrad fwdgelu dgrad
python tools/gemm_graph.py 8320 1536 384 wgrad dgradmul fwd
python tools/gemm_graph.py 8320 384 384 wgrad fwd dgrad
python tools/gemm_graph.py 8320 384 1152 dgrad
python tools/gemm_graph.py 128 128 128 fwd wgrad
PPLL_PDL=0 python tools/gemm_graph.py 8320 384 1152 wgrad fwd
PPLL_PDL=0 python tools/gemm_graph.py 128 128 128 fwd wgrad
