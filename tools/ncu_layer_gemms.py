"""Launch the 12 GEMMs of one ViT-S layer once each (bench.vit_layer_gemms), for
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
       --csv --log-file profiles/r01_ncu_vit_layer_gemms.csv python tools/ncu_layer_gemms.py
(the traffic column of bench.py's GEMM roofline)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
gemms, keep = bench.vit_layer_gemms(bench.WORKLOADS["vit_s"], dev)
s = torch.cuda.current_stream()
for name, fl, by, fn in gemms:
    fn(s.cuda_stream)
torch.cuda.synchronize()
print("\n".join(g[0] for g in gemms))
