"""GPU test of the one-process-per-GPU pipeline (DistributedPipeline): two
processes share cuda:0 (the only GPU a gpurun box has), so every cross-rank
boundary goes through the real CUDA-IPC ring (peer-mapped slots, system-scope
flags, credits) exactly as across NVLink.  The result must be bitwise equal
to the single-process device pipeline on the same data."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SPEC = dict(image=8, channels=3, patch=4, dim=128, heads=2, mlp=256, depth=4, classes=5)
N_BATCHES, B = 7, 6


def _data():
    rng = np.random.default_rng(5)
    return [(rng.standard_normal((B, 3, 8, 8)).astype(np.float32), rng.integers(0, 5, B))
            for _ in range(N_BATCHES)]


def _build(only=None, precision="bf16"):
    import paper_2411_12780_b200 as lp
    spec = lp.VitSpec(**SPEC)
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=3, precision=precision)
    return lp.build_vit_modules(spec, [1, 1, 1, 1], 1, 2, hyper, only=only)


def _rank(rank, world, port, precision, q, chunks=(N_BATCHES,)):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2411_12780_b200.distributed import (DistributedPipeline, gather_metrics,
                                                   stage_placement)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        placement = stage_placement(4, world)
        mine = [j for j in range(4) if placement[j] == rank]
        mods = _build(only=mine, precision=precision)
        pipe = DistributedPipeline(mods, placement, rank, None, capacity=2, max_batch=B)
        data = iter(_data())
        hist = [[] for _ in range(4)]
        errs = {}
        # several run() calls continue one batch sequence (flags
        # and credits carry over; 3 + 2 + 2 with M = 2 also shifts the slots)
        for n in chunks:
            res = pipe.run(data if rank == 0 else None, n, B)
            met = gather_metrics(res, 4, n, n * B, None)
            for j in range(4):
                hist[j] += met.loss_history[j]
            errs.update({k: errs.get(k, 0) | v for k, v in res["errors"].items()})
        met.loss_history = hist
        res = {"errors": errs}
        flat = {m.stage_index: np.concatenate([p.data.ravel() for p in m.parameters()])
                for m in mods}
        q.put((rank, met.loss_history, flat, res["errors"]))
        dist.barrier()
        pipe.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("precision,chunks", [("bf16", (N_BATCHES,)), ("fp32", (N_BATCHES,)),
                                              ("bf16", (3, 2, 2))])
def test_two_process_ipc_pipeline_bitwise_equals_single_process(precision, chunks):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2411_12780_b200 as lp
    torch.cuda.set_device(0)
    ref = _build(precision=precision)
    m = lp.run_epoch(lp.RunMode.PPLL, ref, iter(_data()), lp.RunConfig(buffer_capacity=2))
    ref_flat = {r.stage_index: np.concatenate([p.data.ravel() for p in r.parameters()])
                for r in ref}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 500 + (7 if precision == "fp32" else 0) + 13 * len(chunks)
    procs = [ctx.Process(target=_rank, args=(r, 2, port, precision, q, chunks)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r, losses, flat, errs = q.get(timeout=240)
        out[r] = (losses, flat, errs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    losses = out[0][0]
    assert losses == m.loss_history              # bitwise, all 4 stages
    for r in out:
        assert all(e == 0 for e in out[r][2].values())
        for j, f in out[r][1].items():
            assert np.array_equal(f, ref_flat[j]), (r, j)


def test_single_process_pipeline_across_two_devices_bitwise():
    """DevicePipeline with stages on cuda:0 and cuda:1 (peer access, the
    producer's epilogue storing into the peer's ring slot, cross-device
    events) equals the one-device pipeline bitwise.  Needs two GPUs; gpurun
    boxes have one, the driver's 8-GPU node runs it."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    import paper_2411_12780_b200 as lp
    spec = lp.VitSpec(**SPEC)

    def build(devs):
        hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=20, seed=3, precision="bf16")
        return lp.build_vit_modules(spec, [1, 1, 1, 1], 1, 2, hyper, devices=devs)
    one = build(["cuda:0"] * 4)
    two = build(["cuda:0", "cuda:0", "cuda:1", "cuda:1"])
    m1 = lp.run_epoch(lp.RunMode.PPLL, one, iter(_data()), lp.RunConfig(buffer_capacity=2))
    m2 = lp.run_epoch(lp.RunMode.PPLL, two, iter(_data()), lp.RunConfig(buffer_capacity=2))
    assert m1.loss_history == m2.loss_history
    for a, b in zip(one, two):
        assert np.array_equal(np.concatenate([p.data.ravel() for p in a.parameters()]),
                              np.concatenate([p.data.ravel() for p in b.parameters()]))
