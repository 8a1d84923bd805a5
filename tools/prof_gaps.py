"""Kernel timeline of one ViT-S (or ResNet-32) stage step replayed from a CUDA
graph on a single stream: per-kernel durations, the idle gaps between
consecutive kernels, and the step's wall time (torch.profiler / CUPTI).

usage: python tools/prof_gaps.py [vit|resnet] [stage] [batch]
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2411_12780_b200 as lp

fam = sys.argv[1] if len(sys.argv) > 1 else "vit"
j = int(sys.argv[2]) if len(sys.argv) > 2 else 1
torch.cuda.set_device(0)
hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=10 ** 6, seed=1, precision="bf16")
if fam == "vit":
    spec = lp.VitSpec()
    mods = lp.build_vit_modules(spec, lp.balanced_depths(spec.depth, 4), 1, 3, hyper)
else:
    mods = lp.build_resnet_modules(lp.ResNetSpec(), 4, 1, 3, hyper)
m = mods[j]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 128
x = torch.randn((B,) + tuple(m.in_shape), device="cuda").to(m.act_dtype)
y = torch.as_tensor(np.random.default_rng(0).integers(0, 10, B), device="cuda")
out = torch.empty((B,) + tuple(m.out_shape), device="cuda", dtype=m.act_dtype)
s = torch.cuda.Stream()
m.native(B)
with torch.cuda.stream(s):
    for _ in range(3):
        m.launch_step(B, x.data_ptr(), y.data_ptr(), out.data_ptr(), s.cuda_stream)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    m.launch_step(B, x.data_ptr(), y.data_ptr(), out.data_ptr(), s.cuda_stream)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    g.replay()
b.record()
torch.cuda.synchronize()
step_ms = a.elapsed_time(b) / 50
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev = sorted(ev, key=lambda e: e.time_range.start)
n = len(ev) // 3
ev = ev[n:2 * n]          # the middle replay
busy = sum(e.time_range.elapsed_us() for e in ev)
wall = ev[-1].time_range.end - ev[0].time_range.start
gaps = [ev[i + 1].time_range.start - ev[i].time_range.end for i in range(len(ev) - 1)]
per = defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e.name.split("(")[0][:70]
    per[k][0] += 1
    per[k][1] += e.time_range.elapsed_us()
print(f"{fam} stage {j}: graph replay {step_ms * 1e3:.1f} us/step (events), {len(ev)} kernels, "
      f"kernel busy {busy:.1f} us, first->last {wall:.1f} us, gaps sum {sum(gaps):.1f} us "
      f"(median {np.median(gaps):.2f} us)")
for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t / busy * 100:5.1f}%  {c:4d}  {t / c:7.2f} us  {k}")
if os.environ.get("TIMELINE"):   # every kernel of the middle replay: start / end offsets
    t0 = ev[0].time_range.start
    for e in ev:
        print(f"  {e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} "
              f"{e.time_range.elapsed_us():7.1f}  {e.name.split('(')[0][:60]}")
