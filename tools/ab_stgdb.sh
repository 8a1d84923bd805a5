# NOTE: the double-buffered form was reverted after this A/B ("tried"); PPLL_GEMM_STG_DB no longer exists
# double-buffered TMA-store staging in the GEMM epilogue (PPLL_GEMM_STG_DB, compile
# time): parity with the new layout, the ViT layer GEMM table and the benches,
# against alt_nodb.so (the same tree built with -DPPLL_GEMM_STG_DB=0)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vit.py tests/test_gpu_e2e_families.py tests/test_gpu_variants.py tests/test_gpu_resnet.py -m gpu -x -q 2>&1 | tail -3
for L in libppll_b200.so alt_nodb.so; do
  echo "== $L"
  PPLL_LIB=$PWD/paper_2411_12780_b200/lib/$L timeout 300 python tools/gemm_table.py 2>&1 | tail -16
  for w in vit_s resnet32 vit_b mlp_m; do
    PPLL_LIB=$PWD/paper_2411_12780_b200/lib/$L timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$L $w', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'], round(r.get('frac',0),4))"
  done
done
