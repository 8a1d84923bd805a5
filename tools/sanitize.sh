# compute-sanitizer passes over the hot path: memcheck / racecheck /
# synccheck on the smoke (MLP stage steps, fp32 + bf16), the attention kernels,
# one ViT and one ResNet bf16 stage step and the ring watchdog.
out=gpurun_out/sanitizer.txt
: > $out
run() {
  echo "== $*" >> $out
  timeout 900 compute-sanitizer "$@" 2>&1 | grep -E "ERROR SUMMARY|Error|error|passed|failed" | tail -5 >> $out
}
run --tool memcheck python -c "import __graft_entry__ as g; g.smoke()"
run --tool memcheck python -m pytest -q -x tests/test_gpu_attention.py -k "6-17-2 or 5-37-12"
run --tool memcheck python -m pytest -q -x tests/test_gpu_vit.py -k "test_vit_local_steps_match_oracle"
run --tool memcheck python -m pytest -q -x tests/test_gpu_resnet.py -k "bf16" 
run --tool synccheck python -c "import __graft_entry__ as g; g.smoke()"
run --tool racecheck python -m pytest -q -x tests/test_gpu_attention.py -k "6-17-2"
run --tool memcheck python -m pytest -q -x tests/test_gpu_ring_watchdog.py
cat $out
