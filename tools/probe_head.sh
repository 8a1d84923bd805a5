python tools/gemm_graph.py 128 384 10 fwd dgrad wgrad
python tools/gemm_graph.py 128 768 10 fwd dgrad wgrad
python tools/gemm_graph.py 8192 48 384 fwd wgrad
