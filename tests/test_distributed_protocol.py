"""CPU, multi-process (gloo, world_size 2) test of the cross-rank ring
protocol used by DistributedPipeline (paper_2411_12780_b200/distributed.py).

The device is emulated: ring slots, ready flags and credit counters live in a
multiprocessing shared-memory block, each rank interprets the exact op
schedule ``stage_ops`` produces (pop / credit / step / push / free / release),
and a "step" adds 1 to every feature.  The test checks FIFO delivery, that no
slot is overwritten before its consumer released it (backpressure), labels
travel with features, and that the schedule terminates (no deadlock)."""
import os
import time

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_12780_b200.distributed import plan_for_rank, stage_ops, stage_placement

F = 8          # features per sample
B = 4          # batch


def _worker(rank, world, port, n_stages, M, n_batches, shm_name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    from multiprocessing import shared_memory
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shm = shared_memory.SharedMemory(name=shm_name)
        s = n_stages
        # layout per stage j: x [M, B, F] f32, y [M, B] i64, ready [M] i64, credit [1] i64
        per = M * B * F * 4 + M * B * 8 + M * 8 + 8
        buf = shm.buf

        def view(j):
            off = j * per
            x = np.ndarray((M, B, F), np.float32, buf, off)
            y = np.ndarray((M, B), np.int64, buf, off + M * B * F * 4)
            ready = np.ndarray((M,), np.int64, buf, off + M * B * F * 4 + M * B * 8)
            credit = np.ndarray((1,), np.int64, buf, off + M * B * F * 4 + M * B * 8 + M * 8)
            return x, y, ready, credit

        placement = stage_placement(s, world)
        plan = plan_for_rank(rank, placement)
        seen = {p.stage: [] for p in plan}
        local_ready = {}                       # (j, slot) -> batch seq (events)
        local_free = {}
        deadline = time.time() + 30

        def spin(cond):
            while not cond():
                if time.time() > deadline:
                    raise TimeoutError("protocol deadlock")
                time.sleep(0.0005)

        for t in range(n_batches):
            slot = t % M
            if placement[0] == rank:               # source feeds stage 0
                if t >= M:
                    spin(lambda: local_free.get((0, slot), -1) >= t - M)
                x, y, _, _ = view(0)
                x[slot] = float(t)
                y[slot] = t
                local_ready[(0, slot)] = t + 1
            for p in plan:
                j = p.stage
                for op in stage_ops(p, t, M):
                    kind = op[0]
                    if kind == "pop_event":
                        spin(lambda: local_ready.get((j, slot), 0) >= t + 1)
                    elif kind == "pop_flag":
                        _, _, ready, _ = view(j)
                        spin(lambda: ready[slot] >= op[3])
                    elif kind == "credit_event":
                        spin(lambda: local_free.get((j + 1, slot), -1) >= t - M)
                    elif kind == "credit_flag":
                        _, _, _, credit = view(j)      # producer-side credit word
                        spin(lambda: credit[0] >= op[2])
                    elif kind == "step":
                        x, y, _, _ = view(j)
                        seen[j].append((int(y[slot][0]), float(x[slot][0, 0])))
                        assert np.all(y[slot] == t), "labels must travel with the batch"
                        if j < s - 1:
                            xo, yo, _, _ = view(j + 1)
                            xo[slot] = x[slot] + 1.0     # the push store (pre-update output)
                            yo[slot] = y[slot]
                    elif kind == "push_event":
                        local_ready[(j + 1, slot)] = t + 1
                    elif kind == "push_flag":
                        _, _, ready, _ = view(j + 1)
                        ready[slot] = op[3]
                    elif kind == "free_event":
                        local_free[(j, slot)] = t
                    elif kind == "release":
                        _, _, _, credit = view(j - 1)
                        credit[0] += 1
        q.put((rank, seen))
        shm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_stages,M", [(4, 1), (4, 2), (3, 2), (2, 3), (5, 1)])
def test_cross_rank_ring_protocol(n_stages, M):
    from multiprocessing import shared_memory
    world, n_batches = 2, 9
    per = M * B * F * 4 + M * B * 8 + M * 8 + 8
    shm = shared_memory.SharedMemory(create=True, size=per * n_stages)
    np.ndarray((per * n_stages,), np.uint8, shm.buf)[:] = 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + n_stages * 7 + M
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_stages, M, n_batches, shm.name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            r, seen = q.get(timeout=60)
            results[r] = seen
    finally:
        for p in procs:
            p.join(timeout=30)
        shm.close()
        shm.unlink()
    assert all(p.exitcode == 0 for p in procs)
    seen = {}
    for r in results.values():
        seen.update(r)
    assert sorted(seen) == list(range(n_stages))
    for j in range(n_stages):
        # FIFO, every batch exactly once, and the value proves no slot was
        # overwritten before the consumer popped it
        assert [b for b, _ in seen[j]] == list(range(n_batches))
        assert [v for _, v in seen[j]] == [float(b + j) for b in range(n_batches)]


def test_placement_and_plans():
    assert stage_placement(4, 4) == [0, 1, 2, 3]
    assert stage_placement(4, 2) == [0, 0, 1, 1]
    assert stage_placement(8, 4) == [0, 0, 1, 1, 2, 2, 3, 3]
    assert stage_placement(4, 1) == [0, 0, 0, 0]
    plan = plan_for_rank(1, [0, 0, 1, 1])
    assert [(p.stage, p.input, p.output) for p in plan] == [(2, "remote", "local"),
                                                           (3, "local", "none")]
    ops = stage_ops(plan[0], 5, 2)
    assert ops[0] == ("pop_flag", 2, 1, 6) and ops[-1] == ("release", 1)
