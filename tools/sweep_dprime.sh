# paper-faithful aux depths (d' in {2,3,4}, n=3) and the other BASELINE configs
out=gpurun_out/sweep_dprime.jsonl
: > $out
for wl in vit_s resnet32; do
  for d in 1 2 4; do
    timeout 400 python bench.py --workload $wl --d-prime $d --steps 20 --warmup 5 --no-cpu-baseline 2>>gpurun_out/sweep_dprime.err | tail -1 >> $out
  done
done
for wl in resnet110 vit_b mlp_m; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline 2>>gpurun_out/sweep_dprime.err | tail -1 >> $out
done
wc -l $out
