# dynamic (CLC) vs static tile scheduling of the persistent tcgen05 GEMM
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "PPLL_GEMM_CLC=1" "PPLL_GEMM_CLC=0"; do
  for j in 1 3; do env $v timeout 120 python tools/prof_gaps.py vit $j 2>&1 | grep "graph replay"; done
  env $v timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$v vit_s', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'], round(r['frac'],4), round(r['in_step_streams']['frac'],4), round(r['cold_alone']['frac'],4))"
done
for sh in "8192 8192 8192 fwd" "8320 384 1152 fwd" "8320 384 1536 fwdgelu"; do for v in 1 0; do PPLL_GEMM_CLC=$v python tools/gemm_one.py $sh 20 | head -1 | sed "s/^/clc=$v /"; done; done
