"""Pipeline execution of gradient-isolated stages (mirrors locopipe runtime.py).

The reference runs one Python thread per stage joined by bounded
``StageBuffer`` FIFOs.  Here the PPLL dataflow is expressed on the device:

* each stage has its own CUDA stream (on its module's device);
* each stage boundary is a device-resident ring of ``buffer_capacity`` slots
  (activation + labels) on the CONSUMER's device — the producer's last block
  epilogue stores straight into the slot (over NVLink when the consumer is a
  peer GPU), labels travel with the features;
* "pop" is a stream wait on the slot's ready event, "push backpressure" is a
  stream wait on the consumer's free event for the slot (credit) — the host
  only enqueues, it never waits per batch (except to recycle its pinned
  staging buffer, the analog of the source blocking on a full buffer);
* every stage step is a CUDA graph (one per ring slot) of the native local
  step, so the host issue cost per batch is a handful of launches.

Because every ring is FIFO with one producer and one consumer, each stage
consumes batches in order and its trajectory is independent of timing, so
the device pipeline is bitwise equal to ``run_deterministic`` (the reference's
round-robin replay, reproduced here with its exact integer bookkeeping).
Staleness, buffer high water and busy/idle time are reconstructed from CUDA
event timestamps recorded around every stage step.
"""
from __future__ import annotations

import os

import threading
import time
from collections import Counter, deque
from dataclasses import dataclass, field
from enum import Enum
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _native as N
from .blocks import LocalModule
from .errors import ConfigMismatch, InvalidMode, PushAfterClose, WorkerPanic, ZeroDuration
from .tensor import Tensor


class RunMode(Enum):
    E2E = "E2E"
    NAIVE_PP = "NaivePP"
    PPLL = "PPLL"


class _EndOfStream:
    def __repr__(self) -> str:
        return "EndOfStream"


#: Sentinel returned by pop() once a buffer is closed and drained (runtime.py:43-49).
END_OF_STREAM = _EndOfStream()


@dataclass
class BufferSlot:
    """One batch travelling between stages: id, detached features, labels
    (runtime.py:52-65).  Features may be device tensors of any rank >= 2."""

    batch_id: int
    features: Tensor
    labels: object

    def __post_init__(self):
        if self.features.track_grad:
            raise ValueError("buffer slots must carry detached tensors")
        shp = self.features.shape
        if len(shp) != 2 or shp[0] != len(self.labels):
            raise ValueError(f"features {shp} do not match {len(self.labels)} labels")


class StageBuffer:
    """Host-side twin of the device ring (runtime.py:68-120 semantics).

    Laid out like the device ring: ``capacity`` slots addressed by sequence
    number (slot = seq % capacity), a write sequence and a read sequence.  A
    producer waits for a free slot (the credit wait, never overwrite —
    SPEC.md:319), a consumer for a filled one; after ``close`` the consumer
    drains what is left and then gets END_OF_STREAM, and a producer still
    waiting is released with PushAfterClose.  Counters as in the reference:
    ``high_water`` (max occupancy after a push), ``total_pushed``,
    ``producer_progress`` (set by the producer side)."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        self.capacity = capacity
        self._ring = [None] * capacity
        self._wseq = 0                       # next sequence number to write
        self._rseq = 0                       # next sequence number to read
        self._lock = threading.Lock()
        self._filled = threading.Condition(self._lock)   # consumer waits here
        self._freed = threading.Condition(self._lock)    # producer waits here
        self._closed = False
        self.high_water = 0
        self.producer_progress = -1

    @property
    def total_pushed(self) -> int:
        return self._wseq

    def _count(self) -> int:
        return self._wseq - self._rseq

    def push(self, slot: BufferSlot) -> None:
        with self._lock:
            if self._closed:
                raise PushAfterClose("push on closed buffer")
            self._freed.wait_for(lambda: self._closed or self._count() < self.capacity)
            if self._closed:
                raise PushAfterClose("buffer closed while waiting to push")
            self._ring[self._wseq % self.capacity] = slot
            self._wseq += 1
            self.high_water = max(self.high_water, self._count())
            self._filled.notify()

    def pop(self):
        with self._lock:
            self._filled.wait_for(lambda: self._closed or self._count() > 0)
            if self._count() == 0:
                return END_OF_STREAM
            k = self._rseq % self.capacity
            slot, self._ring[k] = self._ring[k], None
            self._rseq += 1
            self._freed.notify()
            return slot

    def close(self) -> None:
        with self._lock:
            self._closed = True
            self._filled.notify_all()
            self._freed.notify_all()

    @property
    def occupancy(self) -> int:
        with self._lock:
            return self._count()


@dataclass
class RunConfig:
    """Knobs for one epoch run (runtime.py:123-141).

    ``sleep_padding`` / ``comm_padding`` exist for API compatibility with the
    reference's thread emulation; the device pipeline has real compute and
    real transfers, so they must be 0.  ``use_graphs`` replays each stage step
    from a CUDA graph; ``timing`` records per-step CUDA events (busy/idle,
    staleness and high-water reconstruction).
    """

    buffer_capacity: int = 2
    sleep_padding: float | Sequence[float] = 0.0
    comm_padding: float = 0.0
    use_graphs: bool = True
    timing: bool = True

    def pad_for(self, stage: int) -> float:
        if isinstance(self.sleep_padding, (int, float)):
            return float(self.sleep_padding)
        pads = self.sleep_padding
        return float(pads[stage]) if stage < len(pads) else float(pads[-1])


@dataclass
class EpochMetrics:
    """What one epoch did (runtime.py:144-183; the field names and helpers are
    the reference's API contract, restated deliberately).  Threaded (device)
    runs report seconds measured with CUDA events; deterministic runs report
    scheduler rounds (virtual time), like the reference."""

    n_stages: int
    n_batches: int = 0
    wall_time: float = 0.0
    batches_processed: list = field(default_factory=list)
    busy_time: list = field(default_factory=list)
    loss_history: list = field(default_factory=list)
    staleness: Counter = field(default_factory=Counter)
    buffer_high_water: list = field(default_factory=list)
    images: int = 0

    def __post_init__(self):
        if not self.batches_processed:
            self.batches_processed = [0] * self.n_stages
        if not self.busy_time:
            self.busy_time = [0.0] * self.n_stages
        if not self.loss_history:
            self.loss_history = [[] for _ in range(self.n_stages)]

    def mean_loss(self, stage: int) -> float:
        hist = self.loss_history[stage]
        return float(sum(hist) / len(hist)) if hist else float("nan")

    @property
    def final_stage_mean_loss(self) -> float:
        return self.mean_loss(self.n_stages - 1)

    @property
    def mean_staleness(self) -> float:
        total = sum(self.staleness.values())
        if total == 0:
            return 0.0
        return sum(k * v for k, v in self.staleness.items()) / total

    @property
    def idle_fraction(self) -> list:
        """Per-stage 1 - busy/wall."""
        if self.wall_time <= 0:
            return [float("nan")] * self.n_stages
        return [max(0.0, 1.0 - b / self.wall_time) for b in self.busy_time]


def throughput(metrics: EpochMetrics, n_batches: int) -> float:
    """Batches per second (or per virtual step), runtime.py:186-190."""
    if metrics.wall_time <= 0.0:
        raise ZeroDuration("epoch wall time is not positive")
    return n_batches / metrics.wall_time


def _validate_modules(modules: Sequence[LocalModule]) -> None:
    """runtime.py:193-202."""
    if not modules:
        raise ConfigMismatch("no modules to run")
    for j, m in enumerate(modules):
        if m.stage_index != j:
            raise ConfigMismatch(f"module {j} carries stage_index {m.stage_index}")
        if j > 0 and m.in_features != modules[j - 1].out_features:
            raise ConfigMismatch(
                f"stage {j} input width {m.input_width} != stage {j - 1} "
                f"output width {modules[j - 1].output_width}")
        if j > 0 and m.precision != modules[j - 1].precision:
            raise ConfigMismatch("all stages must share one precision")


def run_epoch(mode: RunMode, modules: Sequence[LocalModule], dataset_iter: Iterable,
              config: RunConfig | None = None) -> EpochMetrics:
    """Feed every batch of ``dataset_iter`` through the pipeline once
    (runtime.py:211-223).  PPLL runs as the device pipeline."""
    config = config or RunConfig()
    _validate_modules(modules)
    if mode == RunMode.PPLL:
        return _pipeline_for(modules, config).run(dataset_iter)
    if mode in (RunMode.E2E, RunMode.NAIVE_PP):
        return _run_backprop(modules, dataset_iter, config, pipelined=mode == RunMode.NAIVE_PP,
                             virtual_time=False)
    raise ConfigMismatch(f"unknown mode {mode!r}")


def run_deterministic(mode: RunMode, modules: Sequence[LocalModule], dataset_iter: Iterable,
                      config: RunConfig | None = None) -> EpochMetrics:
    """Single-stream replay with the reference's virtual timing
    (runtime.py:226-243, 475-533)."""
    config = config or RunConfig()
    _validate_modules(modules)
    if mode == RunMode.PPLL:
        return _run_ppll_roundrobin(modules, dataset_iter, config)
    if mode in (RunMode.E2E, RunMode.NAIVE_PP):
        # naive PP collapses to strict per-batch serialisation (runtime.py:423-426):
        # both replay as the single-stream backprop chain with virtual time
        return _run_backprop(modules, dataset_iter, config, pipelined=False, virtual_time=True)
    raise ConfigMismatch(f"unknown mode {mode!r}")


# --------------------------------------------------------------------------
# the paper's baselines: E2E and naive PP on the device
# --------------------------------------------------------------------------

def _run_backprop(modules, dataset_iter, config, pipelined: bool, virtual_time: bool):
    """End-to-end backprop through all blocks (E2E, runtime.py:248-284) or the
    same computation as a naive pipeline (NAIVE_PP, runtime.py:294-408 with
    ppll=False): stage j forwards batch t, the final stage takes the task loss
    on its block output, and dLoss/d(boundary) flows back stage to stage;
    each stage then steps its BLOCK parameters (aux heads unused).  Both
    modes compute identical numbers (test_runtime.py:154-179).

    Device schedule: one stream per stage when ``pipelined`` (the boundary
    activations and gradients are single buffers on the consumer's device,
    ordered by CUDA events: forward j-1 -> forward j, backward j+1 ->
    backward j), else a single stream.  Naive PP serialises every batch across
    the whole pipeline, so stage j's forward of t+1 waits for its backward of t
    by stream order — that bubble is the baseline's cost."""
    mods = list(modules)
    s = len(mods)
    for m in mods:
        if not getattr(m, "supports_e2e", False):
            raise InvalidMode(f"{type(m).__name__} has no block-only forward/backward; "
                              f"it runs PPLL only")
    metrics = EpochMetrics(n_stages=s)
    step0 = [m.optimizer.step_count for m in mods]
    dev0 = mods[0].device
    streams = ([torch.cuda.Stream(device=m.device) for m in mods] if pipelined
               else [torch.cuda.Stream(device=dev0)] * s)
    # stage streams sharing a GPU: no full-GPU cooperative kernels
    shared_dev = pipelined and len({str(m.device) for m in mods}) < s
    lib = N.load()
    prev_excl = lib.ppll_set_gpu_exclusive(int(not shared_dev))
    try:
        return _run_backprop_body(mods, dataset_iter, config, pipelined, virtual_time, metrics,
                                  step0, dev0, streams)
    finally:
        lib.ppll_set_gpu_exclusive(prev_excl)


def _run_backprop_body(mods, dataset_iter, config, pipelined, virtual_time, metrics, step0, dev0,
                       streams):
    s = len(mods)
    src = torch.cuda.Stream(device=dev0)
    _enable_peers(mods)
    timing = config.timing and not virtual_time
    bufs = None
    maxb = 0
    ev_fwd = [torch.cuda.Event() for _ in range(s)]
    ev_bwd = [torch.cuda.Event() for _ in range(s)]
    ev_in = torch.cuda.Event()
    used = False
    t_evs = [[] for _ in range(s)]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev0.record(src)
    n = 0
    images = 0
    for x, y in dataset_iter:
        xt = torch.as_tensor(np.asarray(x, dtype=np.float32) if not torch.is_tensor(x) else x)
        B = int(xt.shape[0])
        if B < 1:
            raise WorkerPanic(-1, "empty batch")
        if xt[0].numel() != mods[0].in_features:
            raise WorkerPanic(0, f"DimensionMismatch: stage 0 expects width {mods[0].in_shape}, "
                                 f"got {tuple(xt.shape)}")
        yt = torch.as_tensor(np.asarray(y)) if not torch.is_tensor(y) else y
        if yt.dtype.is_floating_point or tuple(yt.shape) != (B,):
            raise WorkerPanic(0, "labels must be integers matching the batch")
        for m in mods:
            if m.optimizer.step_count + 1 > m.schedule.total_steps + 1:
                raise WorkerPanic(m.stage_index, f"StepOutOfRange: step "
                                  f"{m.optimizer.step_count} > {m.schedule.total_steps}")
        if bufs is None or B > maxb:
            for st in streams + [src]:
                st.synchronize()
            maxb = max(B, maxb)
            for m in mods:
                m.native(maxb)
            bufs = {
                "x": torch.empty((maxb, mods[0].in_features), dtype=mods[0].act_dtype, device=dev0),
                "y": torch.empty((maxb,), dtype=torch.int64, device=mods[-1].device),
                # h[j]: output of stage j on stage j+1's device; g[j]: its gradient on stage j's
                "h": [torch.empty((maxb, mods[j].out_features), dtype=mods[j].act_dtype,
                                  device=mods[j + 1].device) for j in range(s - 1)],
                "g": [torch.empty((maxb, mods[j].out_features), dtype=mods[j].act_dtype,
                                  device=mods[j].device) for j in range(s - 1)],
            }
        with torch.cuda.stream(src):
            if used:
                src.wait_event(ev_bwd[0])                  # stage 0 done with the input
            xd = xt.reshape(B, -1).to(device=dev0, dtype=torch.float32, non_blocking=True)
            if mods[0].act_dtype == torch.float32:
                bufs["x"][:B].copy_(xd)
            else:
                N.check(N.load().ppll_cast(B * mods[0].in_features, xd.data_ptr(), N.F32,
                                           bufs["x"].data_ptr(), N.BF16, src.cuda_stream), "cast")
            if used:
                src.wait_event(ev_bwd[s - 1])
            bufs["y"][:B].copy_(yt.to(torch.int64), non_blocking=True)
            ev_in.record(src)
        used = True
        xin = [bufs["x"]] + bufs["h"]
        # forward, stage order (records precede the waits that name them)
        for j, m in enumerate(mods):
            st = streams[j]
            st.wait_event(ev_in if j == 0 else ev_fwd[j - 1])
            if timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                t_evs[j].append(e)
            out = bufs["h"][j].data_ptr() if j < s - 1 else None
            m.launch_block_forward(B, xin[j].data_ptr(), out, st.cuda_stream)
            ev_fwd[j].record(st)
            if timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                t_evs[j].append(e)
        # backward, reverse stage order
        for j in reversed(range(s)):
            m, st = mods[j], streams[j]
            if j == s - 1:
                st.wait_event(ev_in)                       # labels
                gout, yptr = None, bufs["y"].data_ptr()
            else:
                st.wait_event(ev_bwd[j + 1])
                gout, yptr = bufs["g"][j].data_ptr(), None
            gin = bufs["g"][j - 1].data_ptr() if j > 0 else None
            if timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                t_evs[j].append(e)
            m.launch_block_backward(B, xin[j].data_ptr(), gout, yptr, gin, st.cuda_stream)
            ev_bwd[j].record(st)
            if timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                t_evs[j].append(e)
            m.optimizer.step_count += 1
        n += 1
        images += B
    for st in set(streams) | {src}:
        st.synchronize()
    for j, m in enumerate(mods):
        try:
            m.raise_for_error(stage=j)
        except WorkerPanic:
            for k, mm in enumerate(mods):
                mm.optimizer.step_count = step0[k] + max(0, mm.device_step() - step0[k])
            raise
    metrics.n_batches = n
    metrics.images = images
    metrics.batches_processed = [n] * s
    metrics.loss_history = [[] for _ in range(s - 1)] + [mods[-1].loss_history(step0[-1], n)]
    metrics.buffer_high_water = [min(1, n)] * s
    if virtual_time:
        metrics.wall_time = float(n)
        metrics.busy_time = [float(n)] * s
    elif timing and n:
        ms = lambda e: ev0.elapsed_time(e) / 1e3  # noqa: E731
        ts = [[ms(e) for e in t_evs[j]] for j in range(s)]
        # per batch: fwd start/end, bwd start (after the gradient arrived) /
        # end; busy excludes the wait for the returning gradient
        # (runtime.py:369-372)
        metrics.busy_time = [sum(b - a for a, b in zip(ts[j][0::2], ts[j][1::2])) for j in range(s)]
        metrics.wall_time = max(t[-1] for t in ts)
    return metrics


def _pipeline_for(modules, config):
    """The DevicePipeline of this module list and ring configuration, reused
    across epochs (its rings, staging buffers and per-(stage, slot) CUDA graphs
    are built once; a training loop calls run_epoch once per epoch)."""
    key = (tuple(id(m) for m in modules), config.buffer_capacity, config.use_graphs,
           config.timing)
    cache = modules[0].__dict__.setdefault("_pipelines", {})
    pipe = cache.get(key)
    if pipe is None:
        pipe = cache[key] = DevicePipeline(modules, config)
    return pipe


def _capture(graph, stream, fn):
    """Capture fn() into graph on stream.  The graphs hold only library kernel
    launches and copies into preallocated buffers, so the allocator pool
    bookkeeping (and the cache flush) of torch.cuda.graph is skipped."""
    with torch.cuda.stream(stream):
        graph.capture_begin(capture_error_mode="thread_local")
        try:
            fn()
        finally:
            graph.capture_end()


# --------------------------------------------------------------------------
# device rings
# --------------------------------------------------------------------------

class _Rings:
    """Per-boundary device rings: ring j is stage j's input (ring 0 is filled
    by the source).  Slot k holds [max_batch, in_w_j] features and labels."""

    def __init__(self, modules, capacity, max_batch):
        self.M = capacity
        self.x, self.y = [], []
        for m in modules:
            self.x.append(torch.empty((capacity, max_batch, m.in_features), dtype=m.act_dtype,
                                      device=m.device))
            self.y.append(torch.zeros((capacity, max_batch), dtype=torch.int64, device=m.device))
        m0 = modules[0]
        # host-input staging, decoupled from the ring capacity M: P pinned
        # slots + P device fp32 slots, so host->device copies run up to P
        # batches ahead of the ring's credits (the ring itself still holds
        # exactly M slots: backpressure semantics unchanged)
        self.P = max(8, 2 * capacity)
        self.cast = m0.act_dtype != torch.float32
        self.x_pin = torch.empty((self.P, max_batch, m0.in_features), dtype=torch.float32,
                                 pin_memory=True)
        self.y_pin = torch.empty((self.P, max_batch), dtype=torch.int64, pin_memory=True)
        self.x_stage = torch.empty((self.P, max_batch, m0.in_features), dtype=torch.float32,
                                   device=m0.device)
        self.y_stage = torch.empty((self.P, max_batch), dtype=torch.int64, device=m0.device)


def _enable_peers(modules):
    devs = sorted({m.device.index for m in modules})
    if len(devs) < 2:
        return
    lib = N.load()
    for a in devs:
        with torch.cuda.device(a):
            for b in devs:
                if a != b and torch.cuda.can_device_access_peer(a, b):
                    N.check(lib.ppll_enable_peer(b), "enable peer access")


class DevicePipeline:
    """The PPLL pipeline on CUDA streams (see module docstring)."""

    def __init__(self, modules, config: RunConfig, max_batch: int | None = None):
        if config.pad_for(0) or config.comm_padding:
            raise ConfigMismatch("sleep/comm padding is a thread-emulation knob; "
                                 "the device pipeline must run unpadded")
        self.modules = list(modules)
        self.config = config
        self.M = config.buffer_capacity
        self.max_batch = max_batch
        self.rings = None
        self.graphs = {}
        self.streams = [torch.cuda.Stream(device=m.device) for m in self.modules]
        self.src_stream = torch.cuda.Stream(device=self.modules[0].device)
        self.h2d_stream = torch.cuda.Stream(device=self.modules[0].device)
        s, M = len(self.modules), self.M
        self.ev_ready = [[torch.cuda.Event() for _ in range(M)] for _ in range(s)]
        self.ev_free = [[torch.cuda.Event() for _ in range(M)] for _ in range(s)]
        self.ev_h2d, self.ev_cast = [], []     # per staging slot (sized in _ensure)
        self.used_free = [[False] * M for _ in range(s)]
        self._pdl = 1
        _enable_peers(self.modules)

    # -- setup ----------------------------------------------------------
    def _ensure(self, batch: int):
        if self.rings is not None and batch <= self.max_batch:
            return
        self.max_batch = max(batch, self.max_batch or 0)
        for m in self.modules:
            m.native(self.max_batch)
        self.rings = _Rings(self.modules, self.M, self.max_batch)
        self.graphs = {}
        self.ev_h2d = [torch.cuda.Event() for _ in range(self.rings.P)]
        self.held = [None] * self.rings.P
        self.ev_cast = [torch.cuda.Event() for _ in range(self.rings.P)]
        self.used_stage = [False] * self.rings.P

    def _launch(self, j: int, slot: int, B: int, stream):
        """Enqueue stage j's local step on ring slot ``slot`` (B rows)."""
        m, r = self.modules[j], self.rings
        last = j == len(self.modules) - 1
        x_in = r.x[j][slot]
        y = r.y[j][slot]
        x_out = None if last else r.x[j + 1][slot]
        if not last:
            r.y[j + 1][slot][:B].copy_(y[:B], non_blocking=True)
        m.launch_step(B, x_in.data_ptr(), y.data_ptr(), N.ptr(x_out), stream.cuda_stream)

    def _step(self, j: int, slot: int, B: int):
        stream = self.streams[j]
        if not self.config.use_graphs or B != self.max_batch:
            with torch.cuda.stream(stream):
                self._launch(j, slot, B, stream)
            return
        # a graph keeps the PDL edges / kernel forms it was captured with
        key = (j, slot, self._pdl, getattr(self, "_excl", 1))
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device=self.modules[j].device)
            cap.wait_stream(stream)
            with torch.cuda.device(self.modules[j].device):
                _capture(g, cap, lambda: self._launch(j, slot, B, cap))
            stream.wait_stream(cap)
            self.graphs[key] = g
        with torch.cuda.stream(stream):
            g.replay()

    # -- the epoch -------------------------------------------------------
    def run(self, dataset_iter: Iterable) -> EpochMetrics:
        """One epoch.  Programmatic dependent launch (PDL) pays when a GPU runs
        one stage stream (the next kernel's prologue overlaps the current
        tail).  With several stage streams on a GPU it depends on the family
        (``shared_gpu_pdl``): early-launched kernels hold SM slots while they
        wait, which costs the ViT step (4 streams on one B200: PDL off
        +1.4 %) but not the short-kernel ResNet / MLP steps (PDL off -11 %
        for ResNet-32).  PPLL_PDL in the environment overrides."""
        per_dev = {}
        for st, m in zip(self.streams, self.modules):
            per_dev.setdefault(str(m.device), set()).add(st.cuda_stream)
        shared = (max(len(v) for v in per_dev.values()) > 1 and
                  not all(getattr(m, "shared_gpu_pdl", True) for m in self.modules))
        lib = N.load()
        want = int(os.environ["PPLL_PDL"] != "0") if "PPLL_PDL" in os.environ else int(not shared)
        prev = lib.ppll_set_pdl(want)
        self._pdl = want
        # several stage streams on one GPU: no full-GPU cooperative kernels
        excl = int(max(len(v) for v in per_dev.values()) == 1)
        prev_excl = lib.ppll_set_gpu_exclusive(excl)
        self._excl = excl
        try:
            return self._run(dataset_iter)
        finally:
            lib.ppll_set_pdl(prev)
            lib.ppll_set_gpu_exclusive(prev_excl)

    def _run(self, dataset_iter: Iterable) -> EpochMetrics:
        mods, M, s = self.modules, self.M, len(self.modules)
        metrics = EpochMetrics(n_stages=s)
        step0 = [m.optimizer.step_count for m in mods]
        timing = self.config.timing
        # timing events come from a pool reused across epochs (an event is
        # only re-recorded after the previous epoch read its elapsed time)
        pool = self.__dict__.setdefault("_tev_pool", [])
        tev_i = [0]

        def tev():
            if tev_i[0] == len(pool):
                pool.append(torch.cuda.Event(enable_timing=True))
            tev_i[0] += 1
            return pool[tev_i[0] - 1]
        t_start, t_end, t_src = [[] for _ in range(s)], [[] for _ in range(s)], []
        ev0 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(self.src_stream):
            ev0.record(self.src_stream)
        n = 0
        images = 0
        for batch_id, (x, y) in enumerate(dataset_iter):
            resident = torch.is_tensor(x) and x.device.type == "cuda"
            x = np.asarray(x, dtype=np.float32) if not torch.is_tensor(x) else x
            B = int(x.shape[0])
            if B < 1:
                raise WorkerPanic(-1, "empty batch")
            for m in mods:
                if m.optimizer.step_count + 1 > m.schedule.total_steps + 1:
                    raise WorkerPanic(m.stage_index, f"StepOutOfRange: step "
                                      f"{m.optimizer.step_count} > {m.schedule.total_steps}")
            self._ensure(B)
            r = self.rings
            slot = batch_id % M
            # ---- source: host -> ring 0 (runtime.py:312-323) ----
            xt = torch.as_tensor(x)
            if xt.dim() >= 2 and xt[0].numel() == mods[0].in_features:
                xt = xt.reshape(B, mods[0].in_features)
            else:
                raise WorkerPanic(0, f"DimensionMismatch: stage 0 expects width "
                                     f"{mods[0].in_shape}, got {tuple(xt.shape)}")
            yt = torch.as_tensor(np.asarray(y)) if not torch.is_tensor(y) else y
            if yt.dtype.is_floating_point or tuple(yt.shape) != (B,):
                raise WorkerPanic(0, "labels must be integers matching the batch")
            src = self.src_stream
            if not resident:
                ps = batch_id % r.P
                if self.used_stage[ps]:
                    self.ev_h2d[ps].synchronize()        # recycle pinned staging
                    self.held[ps] = None
                # caller-pinned fp32 / int64 tensors are copied straight to the
                # device (held until the copy completes); anything else goes
                # through this pipeline's pinned staging slot first
                x_pinned = (xt.is_pinned() and xt.dtype == torch.float32 and
                            xt.is_contiguous())
                y_pinned = (torch.is_tensor(yt) and yt.is_pinned() and
                            yt.dtype == torch.int64)
                if not x_pinned:
                    r.x_pin[ps, :B].copy_(xt)
                if not y_pinned:
                    r.y_pin[ps, :B].copy_(yt)
                h2d = self.h2d_stream
                with torch.cuda.stream(h2d):
                    if self.used_stage[ps]:
                        h2d.wait_event(self.ev_cast[ps])  # device staging slot consumed
                    r.x_stage[ps, :B].copy_(xt if x_pinned else r.x_pin[ps, :B],
                                            non_blocking=True)
                    r.y_stage[ps, :B].copy_(yt if y_pinned else r.y_pin[ps, :B],
                                            non_blocking=True)
                    self.ev_h2d[ps].record(h2d)
                self.held[ps] = (xt, yt) if (x_pinned or y_pinned) else None
                self.used_stage[ps] = True
                x_src, y_src = r.x_stage[ps, :B], r.y_stage[ps, :B]
            else:                                        # inputs already in HBM
                ps = None
                x_src, y_src = xt, yt
                src.wait_stream(torch.cuda.current_stream(xt.device))   # producer of x
                for t_ in (xt, yt):
                    if torch.is_tensor(t_) and t_.is_cuda:
                        t_.record_stream(src)            # no recycling while src reads
            with torch.cuda.stream(src):
                if ps is not None:
                    src.wait_event(self.ev_h2d[ps])
                if self.used_free[0][slot]:
                    src.wait_event(self.ev_free[0][slot])
                if timing:
                    e = tev()
                    e.record(src)
                    t_src.append(e)
                if not r.cast or x_src.dtype == r.x[0].dtype:
                    r.x[0][slot, :B].copy_(x_src, non_blocking=True)
                else:
                    if x_src.dtype != torch.float32:
                        x_src = x_src.float()
                    N.check(N.load().ppll_cast(B * mods[0].in_features, x_src.data_ptr(),
                                               N.F32, r.x[0][slot].data_ptr(), N.BF16,
                                               src.cuda_stream), "cast")
                r.y[0][slot, :B].copy_(y_src, non_blocking=True)
                if ps is not None:
                    self.ev_cast[ps].record(src)
                self.ev_ready[0][slot].record(src)
            # ---- stages (runtime.py:325-388 worker loop, on device) ----
            for j in range(s):
                st = self.streams[j]
                st.wait_event(self.ev_ready[j][slot])                  # pop
                if j < s - 1 and self.used_free[j + 1][slot]:
                    st.wait_event(self.ev_free[j + 1][slot])           # credit (backpressure)
                if timing:
                    e = tev()
                    e.record(st)
                    t_start[j].append(e)
                self._step(j, slot, B)
                self.ev_free[j][slot].record(st)
                self.used_free[j][slot] = True
                if j < s - 1:
                    self.ev_ready[j + 1][slot].record(st)              # push
                if timing:
                    e = tev()
                    e.record(st)
                    t_end[j].append(e)
                mods[j].optimizer.step_count += 1
            n += 1
            images += B
        for st in self.streams:
            st.synchronize()
        self.src_stream.synchronize()
        self.h2d_stream.synchronize()
        # ---- errors: first failing stage surfaces as WorkerPanic ----
        for j, m in enumerate(mods):
            try:
                m.raise_for_error(stage=j)
            except WorkerPanic:
                for k, mm in enumerate(mods):
                    mm.optimizer.step_count = step0[k] + max(0, mm.device_step() - step0[k])
                raise
        # ---- metrics ----
        metrics.n_batches = n
        metrics.images = images
        metrics.batches_processed = [n] * s
        metrics.loss_history = [m.loss_history(step0[j], n) for j, m in enumerate(mods)]
        metrics.buffer_high_water = [0] * s
        if timing and n:
            # every timestamp in one native call (cudaEventElapsedTime loop)
            evs = t_src + [e for j in range(s) for e in t_start[j]] + \
                [e for j in range(s) for e in t_end[j]]
            handles = np.array([e.cuda_event for e in evs], dtype=np.uint64)
            out = np.empty(len(evs), dtype=np.float32)
            N.check(N.load().ppll_events_elapsed(len(evs), handles.ctypes.data, ev0.cuda_event,
                                                 out.ctypes.data), "events_elapsed")
            flat = out.astype(np.float64).tolist()
            src_t = flat[:n]
            st_t = [flat[n + j * n:n + (j + 1) * n] for j in range(s)]
            en_t = [flat[n + s * n + j * n:n + s * n + (j + 1) * n] for j in range(s)]
            metrics.wall_time = max(en_t[-1][-1], max(v[-1] for v in en_t)) / 1e3
            metrics.busy_time = [sum(b - a for a, b in zip(st_t[j], en_t[j])) / 1e3
                                 for j in range(s)]
            for j in range(s):
                prod_start = src_t if j == 0 else st_t[j - 1]
                push_t = src_t if j == 0 else en_t[j - 1]
                for t in range(n):
                    # producer_progress at pop time (runtime.py:336-337)
                    prog = int(np.searchsorted(prod_start, st_t[j][t], side="right")) - 1
                    metrics.staleness[max(0, min(prog, t + M) - t)] += 1
                # occupancy right after each push (runtime.py:96-99)
                hw = 0
                for t in range(n):
                    popped = int(np.searchsorted(st_t[j], push_t[t], side="right"))
                    hw = max(hw, min(M, max(1, t + 1 - popped)))
                metrics.buffer_high_water[j] = hw
        else:
            metrics.staleness[0] += n * s
            metrics.buffer_high_water = [min(M, n)] * s
            metrics.wall_time = 0.0
        return metrics


# --------------------------------------------------------------------------
# deterministic round-robin replay (runtime.py:475-533)
# --------------------------------------------------------------------------

def _run_ppll_roundrobin(modules, dataset_iter, config) -> EpochMetrics:
    s = len(modules)
    M = config.buffer_capacity
    metrics = EpochMetrics(n_stages=s)
    pipe = DevicePipeline(modules, RunConfig(buffer_capacity=M, use_graphs=False, timing=False))
    stream = torch.cuda.current_stream(modules[0].device)
    step0 = [m.optimizer.step_count for m in modules]
    it = iter(dataset_iter)
    stream_done = False
    bufs = [deque() for _ in range(s)]
    closed = [False] * s
    progress = [-1] * s
    done = [False] * s
    next_id = 0
    rounds = 0
    high_water = [0] * s
    sizes = {}
    lib = N.load()
    while not all(done):
        rounds += 1
        while not stream_done and len(bufs[0]) < M:
            try:
                x, y = next(it)
            except StopIteration:
                stream_done = True
                closed[0] = True
                break
            xt = torch.as_tensor(np.asarray(x, dtype=np.float32) if not torch.is_tensor(x) else x)
            B = int(xt.shape[0])
            xt = xt.reshape(B, -1)
            pipe._ensure(B)
            r = pipe.rings
            slot = next_id % M
            sizes[next_id] = B
            with torch.cuda.stream(stream):
                xd = xt.to(device=modules[0].device, dtype=torch.float32)
                if not r.cast:
                    r.x[0][slot, :B].copy_(xd)
                else:
                    N.check(lib.ppll_cast(B * modules[0].in_features, xd.data_ptr(), N.F32,
                                          r.x[0][slot].data_ptr(), N.BF16, stream.cuda_stream),
                            "cast")
                yt = y if torch.is_tensor(y) else torch.as_tensor(np.asarray(y))
                r.y[0][slot, :B].copy_(yt.to(torch.int64))
            progress[0] = next_id
            bufs[0].append(next_id)
            high_water[0] = max(high_water[0], len(bufs[0]))
            next_id += 1
        for j in range(s):
            if done[j]:
                continue
            if not bufs[j]:
                if closed[j]:
                    done[j] = True
                    if j < s - 1:
                        closed[j + 1] = True
                continue
            last = j == s - 1
            if not last and len(bufs[j + 1]) >= M:
                continue
            bid = bufs[j].popleft()
            metrics.staleness[max(0, progress[j] - bid)] += 1
            if not last:
                progress[j + 1] = bid
            with torch.cuda.stream(stream):
                pipe._launch(j, bid % M, sizes[bid], stream)
            modules[j].optimizer.step_count += 1
            if not last:
                bufs[j + 1].append(bid)
                high_water[j + 1] = max(high_water[j + 1], len(bufs[j + 1]))
            metrics.batches_processed[j] += 1
    stream.synchronize()
    for j, m in enumerate(modules):
        m.raise_for_error(stage=j)
    metrics.n_batches = metrics.batches_processed[0]
    metrics.images = sum(sizes.values())
    metrics.loss_history = [m.loss_history(step0[j], metrics.batches_processed[j])
                            for j, m in enumerate(modules)]
    metrics.wall_time = float(rounds)
    metrics.busy_time = [float(c) for c in metrics.batches_processed]
    metrics.buffer_high_water = high_water
    return metrics
