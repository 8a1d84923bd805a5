# NOTE: the light GEMM form was reverted after this A/B ("tried"); PPLL_GEMM_LIGHT is a no-op on the current tree
# light GEMM form (8 epilogue warps, 2 stages, one TMEM accumulator, 2 CTAs/SM) for
# stage streams sharing the GPU: parity with the light form forced on, then the
# ViT-S / ResNet-32 / ViT-B pipeline benches with and without it
PPLL_GPU_EXCLUSIVE=0 PPLL_GEMM_LIGHT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vit.py tests/test_gpu_e2e_families.py tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -3
for sh in "8320 384 1152 fwd" "8320 384 1536 fwdgelu"; do for v in 1 0; do PPLL_GPU_EXCLUSIVE=0 PPLL_GEMM_LIGHT=$v timeout 60 python tools/gemm_one.py $sh 20 | head -1 | sed "s/^/light=$v /"; done; done
for w in vit_s resnet32 vit_b; do for v in 1 0; do
  PPLL_GEMM_LIGHT=$v timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('light=$v $w', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"
done; done
