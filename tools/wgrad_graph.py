"""Implicit-GEMM 3x3 weight gradient (ppll_conv3x3_wgrad_bf16) at the ResNet
stage shapes, batch 128: per launch inside a CUDA graph (back to back), for the
exclusive-GPU form (wide split-K + reduction) and the shared-GPU form (one
cluster, DSMEM reduction).  PPLL_CONV_WGRAD_HALO=0|1 selects the tap-window /
halo producer.
usage: python tools/wgrad_graph.py [batch]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2411_12780_b200 import _native as N
from gemm_graph import per_launch  # noqa: E402

lib = N.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
for C, H in ((16, 32), (32, 16), (64, 8)):
    x = torch.randn(B, H, H, C, device="cuda").bfloat16()
    dz = torch.randn(B, H, H, C, device="cuda").bfloat16()
    nws = lib.ppll_conv3x3_wgrad_ws_floats(B, H, H, C, C)
    ws = torch.empty(nws, device="cuda")
    dw = torch.empty(9 * C, C, device="cuda")
    by = 2 * 2 * B * H * H * C + 4 * 9 * C * C
    row = []
    for excl in (1, 0):
        prev = lib.ppll_set_gpu_exclusive(excl)
        fn = lambda s: N.check(lib.ppll_conv3x3_wgrad_bf16(B, H, H, C, C, x.data_ptr(), dz.data_ptr(),  # noqa
                                                         dw.data_ptr(), ws.data_ptr(), nws, s), "wgrad")
        us = per_launch(fn)
        lib.ppll_set_gpu_exclusive(prev)
        row.append(f"{'wide' if excl else 'cluster'} {us:6.2f} us ({by / us / 1e3:5.0f} GB/s)")
    print(f"wgrad {C}->{C} @{H}x{H} B={B}: " + ", ".join(row))
