timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "PPLL_WGRAD_SHARED_CS=2" "PPLL_WGRAD_SHARED_CS=4" "PPLL_WGRAD_SHARED_CS=3" "PPLL_WGRAD_SHARED_CS=0"; do
  env $v timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v vit_s', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"
done
for v in "PPLL_WGRAD_SHARED_CS=2" "PPLL_WGRAD_SHARED_CS=0"; do
  env $v timeout 400 python bench.py --workload vit_b --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v vit_b', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"
  env $v timeout 400 python bench.py --workload mlp_m --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v mlp_m', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"
done
