# ncu --set full of the shared-GPU (one-cluster) weight gradient 16->16 @32x32, tap-window vs halo producer
for v in 0 1; do
  PPLL_CONV_WGRAD_HALO=$v timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv3x3_wgrad" -s 2 -c 1 -o gpurun_out/ncu_wgrad_h$v python tools/wgrad_one.py 16 32 0 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_wgrad_h$v.ncu-rep
  python tools/ncu_stalls.py gpurun_out/ncu_wgrad_h$v.ncu-rep 2>&1 | head -30
done
