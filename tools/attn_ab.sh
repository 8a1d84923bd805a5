timeout 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -2
PPLL_ATTN_TIMELINE=1 python tools/attn_timeline.py 2>&1 | tail -5
python tools/attn_graph.py 2>&1 | tail -2
python tools/attn_graph.py 128 37 12 2>&1 | tail -2
