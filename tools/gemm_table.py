"""Per-GEMM timing table of one ViT layer's 12 tcgen05 launches (bench.py's
roofline_gemm, without the rest of the bench).

usage: python tools/gemm_table.py [vit_s|vit_b] ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
hbm, tf_burst, _, _ = bench.peaks()
for name in sys.argv[1:] or ["vit_s"]:
    r = bench.roofline_gemm(bench.WORKLOADS[name], tf_burst, hbm, dev)
    print(f"{name}: engine {r['achieved']:.1f} TF/s frac {r['frac']:.3f}  "
          f"mean launch {r['launch_us']:.2f} us")
    for g in r["per_gemm"]:
        print(f"  {g['us']:7.2f} us alone {g.get('us_in_sequence', 0):7.2f} us in seq "
              f"{g['tflops']:7.1f} TF/s  {g['gemm']}")
