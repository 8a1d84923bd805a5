# halo producer for the implicit conv weight gradient (three shifted copies instead of
# nine tap windows): parity (both producers, both forms), per-launch times, ResNet benches
# with the default policy (1: wide form + CI = 32 cluster) vs never (0)
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_geometry_parity.py tests/test_gpu_e2e_families.py tests/test_gpu_norms.py -m gpu -x -q 2>&1 | tail -3
for v in 1 0 2; do echo "== PPLL_CONV_WGRAD_HALO=$v"; PPLL_CONV_WGRAD_HALO=$v timeout 120 python tools/wgrad_graph.py 2>&1 | tail -3; done
for w in resnet32 resnet110; do for v in 1 0; do
  PPLL_CONV_WGRAD_HALO=$v timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; bp=d['backprop_baselines']; print('halo=$v $w', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'], round(r['weight_gradient']['launch_us'],2), round(bp['e2e_backprop_images_per_s']))"
done; done
