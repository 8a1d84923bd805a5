timeout 600 python -m pytest tests/test_gpu_norms.py tests/test_gpu_vit.py -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/norm_graph.py 2>&1 | grep "ln "
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('vit_s', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"; done
