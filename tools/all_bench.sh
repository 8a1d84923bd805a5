# every bench workload on one B200 (N=1), one JSON line each, plus ResNet stage timelines
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in vit_s resnet32 resnet110 vit_b mlp_m; do timeout 400 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/all_$w.json 2> gpurun_out/all_$w.err; echo "$w rc=$?"; done
for j in 0 1 2 3; do timeout 120 python tools/prof_gaps.py resnet $j 2>&1 | grep -v Warn | head -16; done
