timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_geometry_parity.py tests/test_gpu_e2e_families.py -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/conv_graph.py 2>&1 | tail -3
timeout 120 python tools/conv_graph.py 1 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --workload resnet32 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('resnet32', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']))"; done
