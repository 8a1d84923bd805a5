# attention backward: parity tests, per-launch times at the ViT-S / ViT-B geometries, grid sweep, ViT-S bench
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -3
for g in 0 148 256 384; do echo "== grid=$g"; PPLL_ATTN_BWD_GRID=$g timeout 120 python tools/attn_graph.py 2>&1 | tail -2; done
echo "== ViT-B/16 @96 (B=128 T=37 H=12)"; timeout 120 python tools/attn_graph.py 128 37 12 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('vit_s', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'], d['roofline']['frac'])"
