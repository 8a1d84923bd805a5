for v in "X=1" "X=2" "PPLL_CONV_WTMA=0"; do
  env $v timeout 300 python bench.py --workload resnet32 --steps 20 --warmup 5 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err; rc=$?
  echo "$v rc=$rc $(python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), round(r['frac'],4), [x['us'] for x in r['per_conv']])" 2>/dev/null)"
done
timeout 300 python bench.py --workload resnet110 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('resnet110', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']))"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
