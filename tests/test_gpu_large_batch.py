"""Large-batch ViT stage steps (regression: the deferred LayerNorm partial
slabs were sized for the persistent LN-backward kernel's blocks only; past
~37k rows the fused GEMM + LN backward (gemm_ln.cu, one partial row per
128-row tile) wrote beyond its slab and the next reduction read garbage —
NonFiniteError at ViT-S batch 1024 with two or four stages).

ViT-S geometry (D = 384, T = 65: the fused kernel's range), batch 640
(41,600 rows = 325 tiles > the 296-block slab of the old sizing), two
stages, three PPLL batches: every loss finite, the error word clear, and the
update of every stage within 5e-2 (relative L2) of the same run through the
unfused GEMM + LN-kernel path (PPLL_GEMM_LN=0, own interpreter)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2411_12780_b200 as lp
torch.cuda.set_device(0)
steps, B = 3, 640
hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=steps, seed=3, precision="bf16")
spec = lp.VitSpec(image=32, channels=3, patch=4, dim=384, heads=6, mlp=1536, depth=2, classes=10)
mods = lp.build_vit_modules(spec, [1, 1], 1, 3, hyper)
th0 = [np.concatenate([p.data.astype(np.float64).ravel() for p in m.parameters()]) for m in mods]
rng = np.random.default_rng(11)
data = [(rng.standard_normal((B, 3, 32, 32)).astype(np.float32), rng.integers(0, 10, B))
        for _ in range(steps)]
met = lp.run_deterministic(lp.RunMode.PPLL, mods, iter(data), lp.RunConfig(buffer_capacity=2))
torch.cuda.synchronize()
d = [(np.concatenate([p.data.astype(np.float64).ravel() for p in m.parameters()]) - a).tolist()
     for m, a in zip(mods, th0)]
json.dump({"loss": [[float(v) for v in h] for h in met.loss_history], "dtheta": d},
          open(sys.argv[2], "w"))
"""


def test_vit_batch_640_fused_ln_backward(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    script = tmp_path / "run.py"
    script.write_text(SCRIPT)
    res = {}
    for fused in ("1", "0"):
        out = tmp_path / f"out{fused}.json"
        env = dict(os.environ, PPLL_GEMM_LN=fused)
        subprocess.run([sys.executable, str(script), ROOT, str(out)], env=env, check=True,
                       timeout=600)
        res[fused] = json.load(open(out))
    for h in res["1"]["loss"]:
        assert len(h) == 3 and all(np.isfinite(v) for v in h), h
    for a, b in zip(res["1"]["dtheta"], res["0"]["dtheta"]):
        a, b = np.array(a), np.array(b)
        assert np.isfinite(a).all()
        rel = np.linalg.norm(a - b) / np.linalg.norm(b)
        assert rel < 5e-2, rel
