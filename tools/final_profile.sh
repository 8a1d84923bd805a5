# round-end evidence: driver bench command + reference arm, ncu launch list of the bench, ncu --set full
# of the dominant kernels (GEMM dgrad/wgrad, attention backward, fused BN grid, conv wgrad)
timeout 400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 400 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1200 --csv --log-file gpurun_out/fin_launches_vit_s.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/fin_launches_resnet32.csv python bench.py --workload resnet32 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_tc_bwd|gemm_tc_cluster" -c 2 -o gpurun_out/fin_ncu_vit python tools/prof_gaps.py vit 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv3x3_wgrad|bn_fwd_cluster|bn_bwd_cluster" -c 4 -o gpurun_out/fin_ncu_resnet python tools/prof_gaps.py resnet 0 > /dev/null 2>&1
ls -la gpurun_out/ | tail -12
