# round-end evidence: GPU tests, smoke, driver bench command + reference arm, every workload,
# ncu launch lists (ViT-S, ResNet-32), ncu --set full of the dominant kernels
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin_gputest.log 2>&1; echo rc=$? >> gpurun_out/fin_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo rc=$? >> gpurun_out/fin_smoke.log
timeout 400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 400 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
for w in resnet32 resnet110 vit_b mlp_m; do timeout 400 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/fin_all_$w.json 2> gpurun_out/fin_all_$w.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1200 --csv --log-file gpurun_out/fin_launches_vit_s.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/fin_launches_resnet32.csv python bench.py --workload resnet32 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_tc_bwd|gemm_tc_cluster|gemm_tc_kernel" -c 4 -o gpurun_out/fin_ncu_vit python tools/prof_gaps.py vit 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv3x3_tc|conv3x3_wgrad|bn_fwd_cluster|bn_bwd_cluster" -c 6 -o gpurun_out/fin_ncu_resnet python tools/prof_gaps.py resnet 2 > /dev/null 2>&1
ls gpurun_out | grep fin_
