# swapped implicit conv weight gradient (dWᵀ = dZᵀ·X, N = 9·CI per MMA) vs the tap-stacked
# form; alt_noswap.so = the same tree built with -DPPLL_WGRAD_SWAP=0
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_geometry_parity.py tests/test_gpu_e2e_families.py -m gpu -x -q 2>&1 | tail -3
for L in libppll_b200.so alt_noswap.so; do for v in 0 1 2; do echo "== $L PPLL_CONV_WGRAD_HALO=$v"; PPLL_LIB=$PWD/paper_2411_12780_b200/lib/$L PPLL_CONV_WGRAD_HALO=$v timeout 120 python tools/wgrad_graph.py 2>&1 | tail -3; done; done
for cfg in "libppll_b200.so 1" "libppll_b200.so 0" "alt_noswap.so 1"; do set -- $cfg; for w in resnet32 resnet110; do
  PPLL_LIB=$PWD/paper_2411_12780_b200/lib/$1 PPLL_CONV_WGRAD_HALO=$2 timeout 400 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; bp=d['backprop_baselines']; print('$1 halo=$2 $w', round(d['value']), round(d['sequential_schedule_images_per_s']), round(d['e2e']['value']), d['idle_fraction']['mean'], round(r['weight_gradient']['launch_us'],2), round(bp['e2e_backprop_images_per_s']))"
done; done
