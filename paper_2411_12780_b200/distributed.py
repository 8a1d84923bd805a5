"""One process per GPU: the PPLL pipeline sharded by stage across ranks.

Stage j runs on rank ``placement[j]`` (contiguous blocks of stages, SURVEY
§8e).  The only traffic is the forward activation + labels at each stage
boundary (runtime.py:353) — there are no backward messages, no all-reduce.

A boundary whose producer and consumer live on different ranks is a
device-resident ring on the CONSUMER's GPU:

* ``x``/``y`` slots (``capacity`` of them) and a ``ready[slot]`` flag word per
  slot live in consumer memory; the producer maps them with CUDA IPC and its
  last block epilogue stores the activation straight into the peer slot
  (P2P over NVLink), copies the labels, then ``ppll_ring_publish`` does a
  system-scope release store of ``ready[slot] = batch_id + 1``;
* a ``credit`` counter lives in PRODUCER memory; the consumer increments it
  (system-scope atomic) after finishing a batch, and the producer waits
  ``credit >= t - capacity + 1`` before overwriting slot ``t % capacity`` —
  the bounded-buffer backpressure of StageBuffer.push (runtime.py:88-100);
* both waits are device-side acquire spins on LOCAL memory; the host only
  enqueues, never blocks per batch.

Same-rank boundaries use the event rings of ``DevicePipeline``.  The control
plane (IPC handles, batch counts, metrics) goes through a torch.distributed
process group (gloo is enough); nothing on the data path uses a collective.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import WorkerPanic
from .runtime import EpochMetrics, _capture

_HANDLE = 64


def stage_placement(n_stages: int, world: int) -> list:
    """Contiguous stage -> rank map: stage j on rank floor(j·world/s)."""
    if n_stages < 1 or world < 1:
        raise ValueError("need at least one stage and one rank")
    return [j * world // n_stages for j in range(n_stages)]


@dataclass(frozen=True)
class StagePlan:
    stage: int
    input: str       # "source" | "local" | "remote"
    output: str      # "none" | "local" | "remote"


def plan_for_rank(rank: int, placement: Sequence[int]) -> list:
    """The local stages of ``rank`` with the kind of each input / output edge."""
    s = len(placement)
    out = []
    for j in range(s):
        if placement[j] != rank:
            continue
        inp = "source" if j == 0 else ("local" if placement[j - 1] == rank else "remote")
        outp = "none" if j == s - 1 else ("local" if placement[j + 1] == rank else "remote")
        out.append(StagePlan(j, inp, outp))
    return out


def stage_ops(p: StagePlan, t: int, capacity: int) -> list:
    """The ordered device operations one rank enqueues for local stage
    ``p.stage`` and batch ``t`` (the interpreter in DistributedPipeline.run
    and the CPU protocol test share this schedule):

      ("pop_event", j, slot) | ("pop_flag", j, slot, seq)      wait for the input
      ("credit_event", j+1, slot) | ("credit_flag", j, need)   backpressure
      ("step", j, slot)                                        local step (+push store)
      ("push_event", j+1, slot) | ("push_flag", j+1, slot, seq)
      ("free_event", j, slot)                                  input slot reusable
      ("release", j-1)                                         credit to a remote producer
    """
    j, slot, seq = p.stage, t % capacity, t + 1
    ops = [("pop_flag", j, slot, seq) if p.input == "remote" else ("pop_event", j, slot)]
    if t >= capacity:
        if p.output == "local":
            ops.append(("credit_event", j + 1, slot))
        elif p.output == "remote":
            ops.append(("credit_flag", j, credit_needed(t, capacity)))
    ops.append(("step", j, slot))
    if p.output == "local":
        ops.append(("push_event", j + 1, slot))
    elif p.output == "remote":
        ops.append(("push_flag", j + 1, slot, seq))
    ops.append(("free_event", j, slot))
    if p.input == "remote":
        ops.append(("release", j - 1))
    return ops


def credit_needed(t: int, capacity: int) -> int:
    """Producer of batch t may overwrite slot t % capacity once the consumer
    has released batches 0..t-capacity, i.e. credit >= t - capacity + 1."""
    return t - capacity + 1


class _DevBuf:
    """cudaMalloc'd (IPC-exportable) buffer owned by the runtime."""

    def __init__(self, nbytes: int):
        lib = N.load()
        self.nbytes = nbytes
        self.ptr = lib.ppll_dev_alloc(nbytes)
        if not self.ptr:
            raise N.NativeError("ppll_dev_alloc failed: " + lib.ppll_last_error().decode())

    def handle(self) -> bytes:
        h = (C.c_char * _HANDLE)()
        N.check(N.load().ppll_ipc_get_handle(self.ptr, h), "ipc get handle")
        return bytes(h)

    def free(self):
        if self.ptr:
            N.load().ppll_dev_free(self.ptr)
            self.ptr = None


def _open(handle: bytes) -> int:
    out = C.c_void_p()
    buf = (C.c_char * _HANDLE).from_buffer_copy(handle)
    N.check(N.load().ppll_ipc_open_handle(buf, C.byref(out)), "ipc open handle")
    return int(out.value)


class DistributedPipeline:
    """The PPLL dataflow for the stages this rank owns (see module docstring).

    ``modules`` are this rank's LocalModule/VitLocalModule objects (built
    with ``only=``), ``placement`` the full stage -> rank map, ``group`` a
    torch.distributed group used only for the control plane."""

    def __init__(self, modules, placement, rank, group, capacity=2, max_batch=128,
                 use_graphs=True):
        import torch.distributed as dist
        self.dist = dist
        self.mods = {m.stage_index: m for m in modules}
        self.placement = list(placement)
        self.rank = rank
        self.group = group
        self.M = capacity
        self.Bmax = max_batch
        self.use_graphs = use_graphs
        self.plan = plan_for_rank(rank, placement)
        assert sorted(self.mods) == [p.stage for p in self.plan], "modules do not match placement"
        dev = next(iter(self.mods.values())).device
        self.device = dev
        self.lib = N.load()
        self.streams = {p.stage: torch.cuda.Stream(device=dev) for p in self.plan}
        self.src_stream = torch.cuda.Stream(device=dev)
        self._own = []
        # per local stage input ring (local or remote-fed) and flags
        self.x_in, self.y_in = {}, {}              # stage -> base ptr (local memory)
        self.ready_local, self.credit_local = {}, {}
        self.x_peer, self.y_peer, self.ready_peer, self.credit_peer = {}, {}, {}, {}
        self.ev_ready, self.ev_free = {}, {}
        self.graphs = {}
        self.graph_kernels = {}
        self.replayed_kernels = 0      # kernels launched through graph replays
        # batches this pipeline has already moved: the ready flags and credit
        # counters are never reset, so every run() continues the global batch
        # sequence (seq = t + 1, credit >= t - M + 1 for the GLOBAL index t);
        # restarting at 0 would let a consumer pass on the previous run's flags
        self.batches_done = 0
        self._pdl = 1
        self._setup()

    # -- setup ---------------------------------------------------------------
    def _feat(self, j):
        return self.mods[j].in_features

    def _esz(self, j):
        return 2 if self.mods[j].precision == "bf16" else 4

    def _setup(self):
        handles = {}
        for p in self.plan:
            j = p.stage
            m = self.mods[j]
            m.native(self.Bmax)
            xbytes = self.M * self.Bmax * self._feat(j) * self._esz(j)
            xb, yb = _DevBuf(xbytes), _DevBuf(self.M * self.Bmax * 8)
            self._own += [xb, yb]
            self.x_in[j], self.y_in[j] = xb.ptr, yb.ptr
            self.ev_ready[j] = [torch.cuda.Event() for _ in range(self.M)]
            self.ev_free[j] = [torch.cuda.Event() for _ in range(self.M)]
            if p.input == "remote":
                rd = _DevBuf(256)
                self._own.append(rd)
                self.ready_local[j] = rd.ptr
                handles[("in", j)] = (xb.handle(), yb.handle(), rd.handle())
            if p.output == "remote":
                cr = _DevBuf(256)
                self._own.append(cr)
                self.credit_local[j] = cr.ptr
                handles[("credit", j)] = cr.handle()
        gathered = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(gathered, handles, group=self.group)
        allh = {}
        for d in gathered:
            allh.update(d)
        for p in self.plan:
            j = p.stage
            if p.output == "remote":
                xh, yh, rh = allh[("in", j + 1)]
                self.x_peer[j + 1] = _open(xh)
                self.y_peer[j + 1] = _open(yh)
                self.ready_peer[j + 1] = _open(rh)
            if p.input == "remote":
                self.credit_peer[j - 1] = _open(allh[("credit", j - 1)])
        self.dist.barrier(group=self.group)

    def close(self):
        for b in self._own:
            b.free()
        self._own = []

    # -- one stage step --------------------------------------------------------
    def _slot(self, base, slot, feat, esz):
        return base + slot * self.Bmax * feat * esz

    def _launch(self, p, slot, B, stream):
        j = p.stage
        m = self.mods[j]
        h = stream.cuda_stream
        esz = self._esz(j)
        x_in = self._slot(self.x_in[j], slot, m.in_features, esz)
        y_in = self.y_in[j] + slot * self.Bmax * 8
        x_out = None
        if p.output == "local":
            x_out = self._slot(self.x_in[j + 1], slot, m.out_features, esz)
            N.check(self.lib.ppll_copy_async(self.y_in[j + 1] + slot * self.Bmax * 8, y_in, B * 8, h),
                    "labels")
        elif p.output == "remote":
            x_out = self._slot(self.x_peer[j + 1], slot, m.out_features, esz)
            N.check(self.lib.ppll_copy_async(self.y_peer[j + 1] + slot * self.Bmax * 8, y_in, B * 8, h),
                    "labels (peer)")
        m.launch_step(B, x_in, y_in, x_out, h)

    def _step(self, p, slot, B):
        stream = self.streams[p.stage]
        if not self.use_graphs or B != self.Bmax:
            with torch.cuda.stream(stream):
                self._launch(p, slot, B, stream)
            return
        # a graph keeps the PDL edges / kernel forms it was captured with
        key = (p.stage, slot, self._pdl, getattr(self, "_excl", 1))
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device=self.device)
            cap.wait_stream(stream)
            n0 = N.launch_count()
            _capture(g, cap, lambda: self._launch(p, slot, B, cap))
            self.graph_kernels[key] = N.launch_count() - n0
            stream.wait_stream(cap)
            self.graphs[key] = g
        with torch.cuda.stream(stream):
            g.replay()
        self.replayed_kernels += self.graph_kernels[key]

    def _drain(self):
        for st in self.streams.values():
            st.synchronize()
        self.src_stream.synchronize()

    # -- the epoch -------------------------------------------------------------
    def run(self, batches: Iterable | None, n_batches: int, batch_size: int) -> dict:
        """Enqueue ``n_batches`` batches through this rank's stages.  The rank
        owning stage 0 consumes ``batches`` (device or host (x, y) pairs).
        Returns this rank's timings and loss histories (after a sync).  PDL
        policy as in ``DevicePipeline.run`` (off for several ViT stage
        streams on this GPU unless PPLL_PDL is set)."""
        off = (len(self.mods) > 1 and
               not all(getattr(m, "shared_gpu_pdl", True) for m in self.mods.values()))
        want = int(os.environ["PPLL_PDL"] != "0") if "PPLL_PDL" in os.environ else int(not off)
        prev = self.lib.ppll_set_pdl(want)
        self._pdl = want
        # several stages on this rank's GPU: no full-GPU cooperative kernels
        excl = int(len(self.mods) == 1)
        prev_excl = self.lib.ppll_set_gpu_exclusive(excl)
        self._excl = excl
        try:
            return self._run(batches, n_batches, batch_size)
        finally:
            self.lib.ppll_set_pdl(prev)
            self.lib.ppll_set_gpu_exclusive(prev_excl)

    def _run(self, batches: Iterable | None, n_batches: int, batch_size: int) -> dict:
        M, B = self.M, batch_size
        lib = self.lib
        step0 = {j: m.optimizer.step_count for j, m in self.mods.items()}
        it = iter(batches) if batches is not None else None
        t_start = {j: [] for j in self.mods}
        t_end = {j: [] for j in self.mods}
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record(self.src_stream)
        for st in self.streams.values():
            st.wait_stream(self.src_stream)
        m0 = self.mods.get(0)
        base = self.batches_done
        for t_local in range(n_batches):
            t = base + t_local                 # global batch index (flags / credits)
            slot = t % M
            for j, m in self.mods.items():     # host-side twin of the device step guard
                if m.optimizer.step_count + 1 > m.schedule.total_steps + 1:
                    self._drain()
                    raise WorkerPanic(j, f"StepOutOfRange: step {m.optimizer.step_count} > "
                                         f"{m.schedule.total_steps}")
            if m0 is not None:
                x, y = next(it)
                xt = torch.as_tensor(x).reshape(B, -1)
                yt = torch.as_tensor(np.asarray(y) if not torch.is_tensor(y) else y)
                src = self.src_stream
                with torch.cuda.stream(src):
                    if t >= M:
                        src.wait_event(self.ev_free[0][slot])
                    xd = xt.to(self.device, non_blocking=True)
                    if m0.precision == "bf16":
                        N.check(lib.ppll_cast(B * m0.in_features, xd.float().data_ptr(), N.F32,
                                              self.x_in[0] + slot * self.Bmax * m0.in_features * 2,
                                              N.BF16, src.cuda_stream), "cast")
                    else:
                        N.check(lib.ppll_copy_async(self.x_in[0] + slot * self.Bmax * m0.in_features * 4,
                                                    xd.float().contiguous().data_ptr(),
                                                    B * m0.in_features * 4, src.cuda_stream), "x")
                    yd = yt.to(self.device, torch.int64, non_blocking=True).contiguous()
                    N.check(lib.ppll_copy_async(self.y_in[0] + slot * self.Bmax * 8, yd.data_ptr(),
                                                B * 8, src.cuda_stream), "y")
                    self.ev_ready[0][slot].record(src)
            for p in self.plan:
                j = p.stage
                st = self.streams[j]
                h = st.cuda_stream
                for op in stage_ops(p, t, M):
                    kind = op[0]
                    if kind == "pop_event":
                        st.wait_event(self.ev_ready[j][slot])
                    elif kind == "pop_flag":
                        N.check(lib.ppll_ring_wait(self.ready_local[j] + 4 * slot, op[3], h), "pop")
                    elif kind == "credit_event":
                        st.wait_event(self.ev_free[j + 1][slot])
                    elif kind == "credit_flag":
                        N.check(lib.ppll_ring_wait_credit(self.credit_local[j], op[2], h), "credit")
                    elif kind == "step":
                        e = torch.cuda.Event(enable_timing=True)
                        e.record(st)
                        t_start[j].append(e)
                        self._step(p, slot, B)
                    elif kind == "push_event":
                        self.ev_ready[j + 1][slot].record(st)
                    elif kind == "push_flag":
                        N.check(lib.ppll_ring_publish(self.ready_peer[j + 1] + 4 * slot, op[3], h),
                                "push")
                    elif kind == "free_event":
                        self.ev_free[j][slot].record(st)
                    elif kind == "release":
                        N.check(lib.ppll_ring_release(self.credit_peer[j - 1], h), "release")
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                t_end[j].append(e)
                self.mods[j].optimizer.step_count += 1
            self.batches_done = t + 1
        self._drain()
        stall = (C.c_int * 4)()
        if lib.ppll_ring_stall(stall, 1):
            # the device watchdog gave up on a ring wait (a peer stopped
            # producing or consuming): the same surface as a dead worker
            # thread in the reference (runtime.py:400-402)
            what = "ready flag (pop)" if stall[3] == 0 else "credit (backpressure)"
            raise WorkerPanic(min(self.mods), f"ring wait timed out on the {what}: wanted "
                                               f"{stall[1]}, saw {stall[2]}")
        out = {"wall": 0.0, "busy": {}, "loss": {}, "errors": {}}
        for j, m in self.mods.items():
            out["errors"][j] = m.error_word()
        if any(out["errors"].values()):
            # resync the host step counters with the device ones, then surface
            # the first failing local stage (runtime.py:400-402)
            for j, m in self.mods.items():
                m.optimizer.step_count = step0[j] + max(0, m.device_step() - step0[j])
            for j, m in sorted(self.mods.items()):
                m.raise_for_error(stage=j)
        for j, m in self.mods.items():
            out["loss"][j] = m.loss_history(step0[j], n_batches)
            if n_batches:
                out["busy"][j] = sum(a.elapsed_time(b) for a, b in zip(t_start[j], t_end[j])) / 1e3
                out["wall"] = max(out["wall"], ev0.elapsed_time(t_end[j][-1]) / 1e3)
        return out


def gather_metrics(local: dict, n_stages: int, n_batches: int, images: int, group) -> EpochMetrics:
    """Combine the per-rank results into one EpochMetrics (wall = max over ranks)."""
    import torch.distributed as dist
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, local, group=group)
    met = EpochMetrics(n_stages=n_stages)
    met.n_batches = n_batches
    met.images = images
    met.batches_processed = [n_batches] * n_stages
    met.wall_time = max(p["wall"] for p in parts)
    for p in parts:
        for j, b in p["busy"].items():
            met.busy_time[j] = b
        for j, l in p["loss"].items():
            met.loss_history[j] = l
    return met
