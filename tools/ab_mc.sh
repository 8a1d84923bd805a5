for mc in 0 1; do
  PPLL_GEMM_MC=$mc python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('MC=$mc', round(d['value']), round(r['frac'],3), round(r['launch_us_in_sequence'],2), [g['us_in_sequence'] for g in r['per_gemm']])"
done
