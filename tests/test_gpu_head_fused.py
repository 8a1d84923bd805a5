"""The fused classifier head (kernels.cu ``head_xent_kernel``: logits = z·W + b,
softmax_xent and dz = dlog·Wᵀ in one launch, used by every ViT / ResNet local
step and by the final stage's E2E backward) against the three separate
launches it replaces (gemm_rowwarp → softmax_xent → gemm_dot,
PPLL_HEAD_FUSED=0).

The fused kernel keeps each replaced kernel's arithmetic and summation order,
so the check is BITWISE: loss histories and every parameter after PPLL and E2E
runs, fp32 and bf16, 10 classes (16 accumulators) and 20 classes (32
accumulators, the NP = 32 form), batch 4 (fewer warps than rows' worth of
threads) and 40 (rows strided over warps).  The switch is read once per
process, so each setting runs in its own interpreter."""
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
from paper_2411_12780_b200 import _native as N
torch.cuda.set_device(0)
out = {}
for family in ("vit", "resnet"):
    for precision in ("fp32", "bf16"):
        for classes, B in ((10, 4), (20, 40)):
            for mode in (lp.RunMode.PPLL, lp.RunMode.E2E):
                steps = 3
                hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=steps, seed=7,
                                       precision=precision)
                rng = np.random.default_rng(5)
                if family == "vit":
                    mods = lp.build_vit_modules(
                        lp.VitSpec(image=8, channels=3, patch=4, dim=128, heads=2, mlp=256,
                                   depth=3, classes=classes), [1, 1, 1], 1, 2, hyper)
                    shape = (B, 3, 8, 8)
                else:
                    mods = lp.build_resnet_modules(
                        lp.ResNetSpec(n=1, image=8, channels=3, widths=(16, 32, 64),
                                      classes=classes), 3, 1, 2, hyper)
                    shape = (B, 8, 8, 3)
                data = [(rng.standard_normal(shape).astype(np.float32),
                         rng.integers(0, classes, B)) for _ in range(steps)]
                n0 = N.launch_count()
                met = lp.run_deterministic(mode, mods, iter(data), lp.RunConfig(buffer_capacity=2))
                torch.cuda.synchronize()
                key = f"{family}-{precision}-{classes}-{mode.name}"
                out[key] = {
                    "loss": [[float(v) for v in h] for h in met.loss_history],
                    "params": [np.concatenate([p.data.astype(np.float64).ravel()
                                               for p in m.parameters()]).tobytes().hex()
                               for m in mods],
                    "launches": N.launch_count() - n0,
                }
json.dump(out, open(sys.argv[2], "w"))
"""


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = tmp_path_factory.mktemp("head")
    script = d / "run.py"
    script.write_text(SCRIPT)
    res = {}
    for fused in ("0", "1"):
        out = d / f"out{fused}.json"
        env = dict(os.environ, PPLL_HEAD_FUSED=fused)
        subprocess.run([sys.executable, str(script), ROOT, str(out)], env=env, check=True,
                       timeout=600)
        res[fused] = json.load(open(out))
    return res


def test_fused_head_is_bitwise_equal_to_the_separate_kernels(runs):
    a, b = runs["0"], runs["1"]
    assert a.keys() == b.keys() and len(a) == 16
    for k in a:
        assert a[k]["loss"] == b[k]["loss"], k
        assert a[k]["params"] == b[k]["params"], k
        assert all(np.isfinite(v) for h in b[k]["loss"] for v in h), k


def test_fused_head_removes_launches(runs):
    """Two launches fewer per head step enqueued (steps replayed from a
    captured CUDA graph count once, at capture)."""
    a, b = runs["0"], runs["1"]
    for k in a:
        saved = a[k]["launches"] - b[k]["launches"]
        assert saved >= 2 and saved % 2 == 0, (k, a[k]["launches"], b[k]["launches"])
