timeout 900 python -m pytest tests/test_gpu_geometry_parity.py tests/test_gpu_vit.py tests/test_gpu_e2e_families.py tests/test_gpu_distributed.py -m gpu -x -q 2>&1 | tail -2
for v in "PPLL_GEMM_LN_FWD=1" "PPLL_GEMM_LN_FWD=0"; do echo "== $v"
  env $v PPLL_PDL=0 timeout 120 python tools/prof_gaps.py vit 1 2>&1 | grep -v Warn | head -3
  for i in 1 2; do env $v timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v vit_s', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"; done
done
