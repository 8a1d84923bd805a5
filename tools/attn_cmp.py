"""bench.py's attention roofline entry next to tools/attn_graph.py's timing, in one process
(checks that the two methods agree).  usage: python tools/attn_cmp.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
hbm, _, _, _ = bench.peaks()
for sets in (1, 4):
    r = bench.roofline_attention(bench.WORKLOADS["vit_s"], hbm, dev, sets=sets)
    print(f"bench method sets={sets}: bwd {r['launch_us']:.2f} us fwd {r['forward']['launch_us']:.2f} us; "
          f"warm bwd {r['warm_l2']['bwd_launch_us']:.2f} fwd {r['warm_l2']['fwd_launch_us']:.2f}")
os.system(f"{sys.executable} {os.path.join(os.path.dirname(os.path.abspath(__file__)), 'attn_graph.py')}")
