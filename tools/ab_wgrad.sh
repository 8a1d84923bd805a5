# implicit-GEMM conv weight gradient: parity, per-launch time vs im2col + GEMM, ResNet benches
timeout 600 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_geometry_parity.py tests/test_gpu_e2e_families.py -m gpu -x -q 2>&1 | tail -3
for v in "PPLL_CONV_WGRAD_IMPLICIT=1" "PPLL_CONV_WGRAD_IMPLICIT=0"; do
  for j in 0 1 2 3; do env $v timeout 120 python tools/prof_gaps.py resnet $j 2>&1 | grep "graph replay"; done
  env $v timeout 400 python bench.py --workload resnet32 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v resnet32', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"
  env $v timeout 400 python bench.py --workload resnet110 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v resnet110', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"
done
timeout 120 python tools/prof_gaps.py resnet 0 2>&1 | grep -v Warn | head -16
