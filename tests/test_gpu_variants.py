"""Opt-in / environment-selected engine variants, each in a fresh process
(the switches are read once per process): the CTA-pair GEMM
(PPLL_GEMM_MC=1, tcgen05.mma.cta_group::2) against torch on the same bf16
operands, and a ViT stage trained with the weight gradients on the step's
own stream (PPLL_SIDE_WGRAD=0) bitwise equal to the side-stream default."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

GEMM_CHECK = r"""
import json, sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2411_12780_b200 import _native as N
lib = N.load()
s = torch.cuda.current_stream().cuda_stream
out = []
g = torch.Generator(device="cuda").manual_seed(3)
for M, K, Nn, op in [(1024, 512, 768, "dgrad"), (8320, 1536, 1024, "dgrad"),
                     (1000, 384, 512, "fwd"), (2048, 1024, 256, "fwd")]:
    if op == "fwd":
        X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
        W = (torch.randn(K, Nn, device="cuda", generator=g) * 0.05).bfloat16()
        b = torch.randn(Nn, device="cuda", generator=g)
        Y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
        N.check(lib.ppll_linear_fwd(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                    Y.data_ptr(), Nn, None, 0, 1, N.BF16, s), "fwd")
        ref = (X.float() @ W.float() + b).clamp_min(0)
    else:
        dY = torch.randn(M, Nn, device="cuda", generator=g).bfloat16()
        W = (torch.randn(K, Nn, device="cuda", generator=g) * 0.05).bfloat16()
        Y = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
        N.check(lib.ppll_linear_dgrad(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(), None, 0,
                                      Y.data_ptr(), K, N.BF16, s), "dgrad")
        ref = dY.float() @ W.float().t()
    torch.cuda.synchronize()
    out.append(((Y.float() - ref).abs().max() / ref.abs().max()).item())
print(json.dumps(out))
"""


def _run(code, env_extra, *args):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", code, ROOT, *args], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r


def test_cta_pair_gemm_matches_torch():
    r = _run(GEMM_CHECK, {"PPLL_GEMM_MC": "1", "PPLL_GEMM_VERBOSE": "1"})
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(e < 2e-2 for e in errs), errs
    assert "mc=1" in r.stderr          # the pair kernel actually ran


STAGE_RUN = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2411_12780_b200 as lp
torch.cuda.set_device(0)
spec = lp.VitSpec()
hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=3, precision="bf16")
mods = lp.build_vit_modules(spec, lp.balanced_depths(spec.depth, 4), 1, 3, hyper)
rng = np.random.default_rng(0)
data = [(rng.standard_normal((64, 3, 32, 32)).astype(np.float32), rng.integers(0, 10, 64))
        for _ in range(6)]
met = lp.run_epoch(lp.RunMode.PPLL, mods, data)
import hashlib
flat = [hashlib.sha256(m._flat["theta"].cpu().numpy().tobytes()).hexdigest() for m in mods]
print(json.dumps({"loss": met.loss_history, "theta": flat}))
"""


def test_side_stream_weight_gradients_bitwise():
    a = json.loads(_run(STAGE_RUN, {"PPLL_SIDE_WGRAD": "1"}).stdout.strip().splitlines()[-1])
    b = json.loads(_run(STAGE_RUN, {"PPLL_SIDE_WGRAD": "0"}).stdout.strip().splitlines()[-1])
    assert a == b
