# BASELINE configs[4] (C5): stage count x batch sweep for ResNet-32 and ViT-S on one
# B200 (all stages on one GPU, one stream per stage).  One JSON line per run.
out=gpurun_out/sweep_c5.jsonl
: > $out
for wl in vit_s resnet32; do
  for st in 1 2 4 8; do
    for b in 64 256 1024; do
      timeout 300 python bench.py --workload $wl --stages $st --batch $b --steps 20 --warmup 5 \
        --no-cpu-baseline 2>>gpurun_out/sweep_c5.err | tail -1 >> $out || echo "{\"failed\": \"$wl s=$st b=$b\"}" >> $out
    done
  done
  for b in 128 512; do
    timeout 300 python bench.py --workload $wl --stages 4 --batch $b --steps 20 --warmup 5 \
      --no-cpu-baseline 2>>gpurun_out/sweep_c5.err | tail -1 >> $out
  done
done
wc -l $out
