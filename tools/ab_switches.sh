# one-off A/B of runtime switches on the single-GPU pipelines
run() { env $2 timeout 400 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'])"; }
run vit_s "X=0"
run vit_s "PPLL_PDL=1"
run vit_s "PPLL_ATTN_BWD_GRID=256"
run resnet32 "X=0"
run resnet32 "PPLL_BN_CS=8"
run resnet32 "PPLL_PDL=0"
run resnet32 "PPLL_BN_FWD_MAX_MB=5 PPLL_BN_BWD_MAX_MB=5"
