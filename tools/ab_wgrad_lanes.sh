# TMA loads of a weight-gradient chunk issued by one lane per load vs by lane 0 alone;
# alt_lanes0.so = the same tree built with -DPPLL_WGRAD_LANES=0
timeout 900 python -m pytest tests/test_gpu_resnet.py -m gpu -x -q -k wgrad 2>&1 | tail -2
for L in libppll_b200.so alt_lanes0.so; do for v in 0 2; do echo "== $L PPLL_CONV_WGRAD_HALO=$v"; PPLL_LIB=$PWD/paper_2411_12780_b200/lib/$L PPLL_CONV_WGRAD_HALO=$v timeout 120 python tools/wgrad_graph.py 2>&1 | tail -3; done; done
