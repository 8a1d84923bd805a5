timeout 900 python -m pytest tests/test_gpu_norms.py tests/test_gpu_resnet.py tests/test_gpu_geometry_parity.py tests/test_gpu_e2e_families.py -m gpu -x -q 2>&1 | tail -2
for v in "PPLL_BN_SPLIT=1" "PPLL_BN_SPLIT=0"; do for w in resnet32 resnet110; do
  env $v timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $w', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"
done; done
