# SM budgets for the data-gradient GEMMs / cluster wgrads of the ViT backward (side stream on)
for v in "X=0" "PPLL_DGRAD_CAP=112" "PPLL_DGRAD_CAP=96" "PPLL_DGRAD_CAP=112 PPLL_WGRAD_CAP=36" "PPLL_DGRAD_CAP=96 PPLL_WGRAD_CAP=52" "PPLL_DGRAD_CAP=128 PPLL_WGRAD_CAP=20"; do
  echo "== $v"; env $v timeout 120 python tools/prof_gaps.py vit 1 2>&1 | grep "graph replay"
done
for v in "X=0" "PPLL_DGRAD_CAP=112" "PPLL_DGRAD_CAP=96 PPLL_WGRAD_CAP=52"; do env $v timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']))"; done
