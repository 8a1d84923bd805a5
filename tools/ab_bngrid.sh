# grid-form fused BN (cooperative, one CTA per SM) for the large ResNet tensors; used only when
# the stage owns its GPU (ppll_set_gpu_exclusive): sequential / E2E / one-stage-per-GPU runs
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/norm_graph.py 2>&1 | grep bn
for w in resnet32 resnet110; do for v in "PPLL_BN_GRID_MAX_MB=64" "PPLL_BN_GRID_MAX_MB=0"; do
  env $v timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); bp=d['backprop_baselines']; print('$w $v', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'], round(bp['e2e_backprop_images_per_s']), round(bp['naive_pp_images_per_s']))"
done; done
