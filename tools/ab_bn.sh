# fused single-cluster BN vs the three-/four-kernel path: parity tests, per-launch
# times (tools/norm_graph.py), phase timelines, ResNet-32 bench
timeout 600 python -m pytest tests/test_gpu_norms.py tests/test_gpu_resnet.py tests/test_gpu_e2e_families.py tests/test_gpu_geometry_parity.py -m gpu -x -q 2>&1 | tail -4
echo "== fused"; timeout 120 python tools/norm_graph.py 2>&1 | grep bn
echo "== legacy"; PPLL_BN_FUSED=0 timeout 120 python tools/norm_graph.py 2>&1 | grep bn
for pc in "32768 32" "131072 16" "8192 64"; do PPLL_BN_TIMELINE=1 timeout 60 python tools/bn_timeline.py $pc 2>&1 | tail -2; done
for v in "PPLL_BN_FUSED=1" "PPLL_BN_FUSED=0"; do env $v timeout 300 python bench.py --workload resnet32 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['sequential_schedule_images_per_s']), d['e2e']['value'], d['idle_fraction']['mean'])"; done
