# NOTE: the fused-mask form was reverted after this A/B ("tried"); PPLL_BN_MASK_FUSED no longer exists
# ReLU mask fused into the split BN-backward kernels (PPLL_BN_MASK_FUSED) vs a separate mask pass
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_geometry_parity.py tests/test_gpu_e2e_families.py -m gpu -x -q 2>&1 | tail -2
PPLL_BN_FUSED=0 timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_geometry_parity.py tests/test_gpu_e2e_families.py -m gpu -x -q 2>&1 | tail -2
for w in resnet32 resnet110; do for v in 1 0 1 0; do
  PPLL_BN_MASK_FUSED=$v timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); bp=d['backprop_baselines']; print('mask_fused=$v $w', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'], round(bp['e2e_backprop_images_per_s']), round(bp['naive_pp_images_per_s']), d['final_losses'][0])"
done; done
