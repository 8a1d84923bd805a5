"""CPU tests of the host-side logic: partition/aux-depth/bookkeeping against
the oracle, StageBuffer blocking semantics (test_runtime.py:36-135 restated),
error classes, and the C-ABI library's symbol table (no compute calls)."""
import ctypes
import os
import re
import threading
import time

import numpy as np
import pytest

import paper_2411_12780_b200 as lp
import ppll_oracle as orc
from conftest import ROOT
from paper_2411_12780_b200 import _native as N
from paper_2411_12780_b200.errors import (ConfigMismatch, PushAfterClose, StepOutOfRange,
                                          TooManyStages, ZeroDuration)


# --- the C-ABI boundary -----------------------------------------------------

def _header_symbols():
    text = open(os.path.join(ROOT, "include", "ppll.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ppll_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    declared = _header_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} not bound in _native.SIGNATURES"
    assert lib.ppll_abi_version() == 1


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_cosine_lr_c_abi_matches_reference_kats():
    lib = N.load()
    assert lib.ppll_cosine_lr(0, 0.2, 0.02, 100) == pytest.approx(0.2)
    assert lib.ppll_cosine_lr(50, 0.2, 0.02, 100) == pytest.approx(0.11)
    assert lib.ppll_cosine_lr(100, 0.2, 0.02, 100) == pytest.approx(0.02)
    assert np.isnan(lib.ppll_cosine_lr(101, 0.2, 0.02, 100))
    for k in range(0, 38):
        assert lib.ppll_cosine_lr(k, 0.1, 0.0, 37) == lp.cosine_lr(k, lp.LrSchedule(0.1, 0.0, 37))


# --- structure ----------------------------------------------------------------

def test_partition_matches_oracle_on_random_networks():
    rng = np.random.default_rng(19)
    for _ in range(60):
        n_layers = int(rng.integers(2, 8))
        dims = tuple(int(d) for d in rng.integers(1, 12, size=n_layers + 1))
        s = int(rng.integers(1, n_layers + 1))
        assert lp.partition(lp.NetworkSpec(dims), s).boundaries == orc.partition(dims, s)


def test_partition_reference_cases():
    assert lp.partition(lp.NetworkSpec((8, 8, 8, 8, 8)), 2).boundaries == ((0, 2), (2, 4))
    assert lp.partition(lp.NetworkSpec((2, 2, 2, 2)), 2).boundaries == ((0, 1), (1, 3))
    with pytest.raises(TooManyStages):
        lp.partition(lp.NetworkSpec((4, 4, 4)), 3)
    with pytest.raises(ConfigMismatch):
        lp.PartitionPlan(2, ((0, 1), (2, 3)))


def test_aux_depth_and_validation():
    for l in range(14):
        for d in range(5):
            for n in range(1, 4):
                assert lp.aux_depth(l, d, n) == orc.aux_depth(l, d, n)
    with pytest.raises(ValueError):
        lp.aux_depth(-1, 2, 3)
    with pytest.raises(ValueError):
        lp.Hyperparams(precision="fp8")


def test_schedule_and_cosine():
    sched = lp.LrSchedule(lr0=0.2, lr_min=0.02, total_steps=100)
    assert lp.cosine_lr(50, sched) == pytest.approx(0.11)
    with pytest.raises(StepOutOfRange):
        lp.cosine_lr(101, sched)
    with pytest.raises(ValueError):
        lp.LrSchedule(lr0=0.1, lr_min=0.2)


# --- StageBuffer (host twin of the device ring) ----------------------------------

def _slot(i, rows=2, cols=3):
    import torch
    return lp.BufferSlot(i, lp.Tensor(torch.zeros(rows, cols), device="cpu"),
                         np.zeros(rows, dtype=np.int64))


def test_buffer_fifo_high_water_close_and_sentinel():
    buf = lp.StageBuffer(capacity=3)
    for i in range(3):
        buf.push(_slot(i))
    assert buf.occupancy == 3 and buf.high_water == 3 and buf.total_pushed == 3
    assert [buf.pop().batch_id for _ in range(3)] == [0, 1, 2]
    buf.push(_slot(9))
    buf.close()
    assert buf.pop().batch_id == 9
    assert buf.pop() is lp.END_OF_STREAM
    with pytest.raises(PushAfterClose):
        buf.push(_slot(1))


def test_buffer_push_blocks_until_pop_and_close_releases_producer():
    buf = lp.StageBuffer(capacity=1)
    buf.push(_slot(0))
    pushed = threading.Event()

    def producer():
        buf.push(_slot(1))
        pushed.set()

    th = threading.Thread(target=producer, daemon=True)
    th.start()
    time.sleep(0.05)
    assert not pushed.is_set()
    assert buf.pop().batch_id == 0
    assert pushed.wait(2.0)
    th.join(2.0)
    raised = threading.Event()
    buf2 = lp.StageBuffer(1)
    buf2.push(_slot(0))

    def blocked():
        try:
            buf2.push(_slot(1))
        except PushAfterClose:
            raised.set()

    th = threading.Thread(target=blocked, daemon=True)
    th.start()
    time.sleep(0.05)
    buf2.close()
    assert raised.wait(2.0)


def test_buffer_slot_validation():
    import torch
    with pytest.raises(ValueError):
        lp.BufferSlot(0, lp.Tensor(torch.zeros(2, 3), track_grad=True, device="cpu"),
                      np.zeros(2, dtype=np.int64))
    with pytest.raises(ValueError):
        lp.BufferSlot(0, lp.Tensor(torch.zeros(2, 3), device="cpu"), np.zeros(4, dtype=np.int64))
    with pytest.raises(ValueError):
        lp.StageBuffer(0)


def test_metrics_helpers():
    m = lp.EpochMetrics(n_stages=2)
    assert m.batches_processed == [0, 0] and np.isnan(m.mean_loss(0))
    with pytest.raises(ZeroDuration):
        lp.throughput(m, 4)
    m.wall_time, m.busy_time = 2.0, [1.5, 2.0]
    assert m.idle_fraction == [0.25, 0.0]
    cfg = lp.RunConfig(sleep_padding=[0.1, 0.2])
    assert cfg.pad_for(5) == 0.2


def test_compute_refuses_cpu_tensors():
    """No CPU fallback: compute entry points fail loudly off-device."""
    import torch
    a = lp.Tensor(torch.zeros(2, 3), device="cpu")
    b = lp.Tensor(torch.zeros(3, 4), device="cpu")
    with pytest.raises(RuntimeError, match="CUDA"):
        lp.matmul(a, b)


def test_balanced_resnet_split_is_contiguous_and_minimax():
    from paper_2411_12780_b200.resnet import ResNetSpec, balanced_resnet_split, resnet_split
    for spec, s in ((ResNetSpec(), 4), (ResNetSpec(n=18), 8), (ResNetSpec(n=2), 3)):
        b = balanced_resnet_split(spec, s, 1, 3)
        flat = [x for blk in b for x in blk]
        assert flat == list(range(spec.n_blocks)) and len(b) == s
        assert all(len(blk) >= 1 for blk in b[1:])
    # the high-resolution early blocks are spread thinner than the even split
    assert len(balanced_resnet_split(ResNetSpec(), 4, 1, 3)[0]) < len(resnet_split(ResNetSpec(), 4)[0])


def test_balanced_vit_depths_minimax_earliest_cut_and_idle():
    """Cost-balanced ViT split: brute-force minimax over
    every contiguous split, earliest cut on ties, and the predicted
    one-stage-per-GPU idle fraction < 10 % for the bench configs at d'=1."""
    import itertools
    from paper_2411_12780_b200.vit import VitSpec, balanced_vit_depths, vit_stage_costs
    vit_s = VitSpec()
    vit_b = VitSpec(image=96, patch=16, dim=768, heads=12, mlp=3072, depth=12)
    for spec, s in ((vit_s, 4), (vit_b, 8), (vit_s, 2), (vit_b, 4)):
        for d in (1, 2, 4):
            got = balanced_vit_depths(spec, s, d, 3)
            assert sum(got) == spec.depth and min(got) >= 1
            best = min(max(vit_stage_costs(spec, [b - a for a, b in zip((0,) + c, c + (spec.depth,))],
                                           d, 3))
                       for c in itertools.combinations(range(1, spec.depth), s - 1))
            assert max(vit_stage_costs(spec, got, d, 3)) <= best * (1 + 1e-9)
    for spec, s, want in ((vit_s, 4, [1, 2, 2, 3]), (vit_b, 8, [1, 1, 1, 1, 2, 2, 2, 2])):
        got = balanced_vit_depths(spec, s, 1, 3)
        assert got == want
        c = vit_stage_costs(spec, got, 1, 3)
        assert sum(1 - x / max(c) for x in c) / s < 0.10
