"""Implicit-GEMM 3x3 convolution (ppll_conv3x3_bf16) at the ResNet-32 stage
shapes, batch 128: per launch inside a CUDA graph (20 back to back) and alone
after a clean L2 flush (bench.py's roofline_conv method), with algorithmic GB/s.
usage: python tools/conv_graph.py [dgrad]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2411_12780_b200 import _native as N
from gemm_graph import per_launch  # noqa: E402

dg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
lib = N.load()
B = 128
flush = torch.ones(128 << 20, device="cuda")
sink = torch.empty(1, device="cuda")
for C, H in ((16, 32), (32, 16), (64, 8)):
    x = torch.randn(B, H, H, C, device="cuda").bfloat16()
    w = (torch.randn(9 * C, C, device="cuda") * 0.05).bfloat16()
    y = torch.empty_like(x)
    fn = lambda s: lib.ppll_conv3x3_bf16(B, H, H, C, C, x.data_ptr(), w.data_ptr(), y.data_ptr(), dg, s)  # noqa
    g_us = per_launch(fn)
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = []
    for with_k in (True, False):
        best = 1e9
        for _ in range(3):
            a.record()
            for _ in range(10):
                torch.sum(flush, dim=(0,), out=sink[0])
                if with_k:
                    fn(st.cuda_stream)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        tot.append(best)
    cold = (tot[0] - tot[1]) / 10 * 1e3
    by = 2 * 2 * B * H * H * C + 2 * 9 * C * C
    print(f"conv{'T' if dg else ''} {C}->{C} @{H}x{H}: graph {g_us:6.2f} us ({by / g_us / 1e3:5.0f} GB/s), "
          f"cold alone {cold:6.2f} us ({by / cold / 1e3:5.0f} GB/s)")
