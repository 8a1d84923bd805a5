"""Batch-time model and schedule simulator (the reference's costs.py vocabulary:
StageProfile / CommModel / t_e2e / t_pp / t_ppll / ratio_ideal / ppll_beats_pp /
simulate_schedule / render_gantt_csv, costs.py:30-303), plus the calibration
the reference cannot do: ``calibrate`` measures every stage's local step on the
device (CUDA events around graph replays) and turns it into StageProfiles, so
``simulate_schedule`` predicts the steady batch time and per-stage idle
fraction of a pipeline with one stage per GPU.

Disciplines (costs.py:1-18):
  * e2e      — one device, per batch: all forwards, all backwards, all updates;
  * naive_pp — the same chain plus the per-batch transfer total Q after the
               forwards, each stage updating right after its own backward;
  * ppll     — stages run concurrently; stage j starts batch t when stage j-1
               has pushed t and stage j finished t-1; its push (after its block
               forward, plus Q on stage 0) waits for a free downstream slot
               (batch t - capacity popped by stage j+1).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

from .errors import EmptyEvents, EmptyProfiles, InvalidMode, ZeroDuration

MODES = ("e2e", "naive_pp", "ppll")


@dataclass(frozen=True)
class StageProfile:
    """Per-batch costs of one stage: block forward/backward/update (f, b, u)
    and the same for its aux head (f_a, b_a, u_a).  Non-negative."""

    f: float
    b: float
    u: float
    f_a: float = 0.0
    b_a: float = 0.0
    u_a: float = 0.0

    def __post_init__(self):
        for k in ("f", "b", "u", "f_a", "b_a", "u_a"):
            if getattr(self, k) < 0:
                raise ValueError(f"stage cost {k} must be >= 0")

    @property
    def cycle(self) -> float:
        """One full local step of the stage (block + aux), no transfer."""
        return self.f + self.f_a + (self.b + self.b_a) + (self.u + self.u_a)


@dataclass(frozen=True)
class CommModel:
    """Per-batch transfer total Q, charged once per batch."""

    q_total: float = 0.0

    def __post_init__(self):
        if self.q_total < 0:
            raise ValueError("q_total must be >= 0")


@dataclass(frozen=True)
class CostEstimate:
    mode: str
    batch_time: float
    components: dict = field(default_factory=dict)


def _need(profiles):
    if not profiles:
        raise EmptyProfiles("need at least one stage profile")


def t_e2e(profiles: Sequence[StageProfile]) -> CostEstimate:
    """Serial single-device batch time ΣF + ΣB + ΣU (no aux, no transfer)."""
    _need(profiles)
    F = sum(p.f for p in profiles)
    B = sum(p.b for p in profiles)
    U = sum(p.u for p in profiles)
    return CostEstimate("e2e", F + B + U, {"F": F, "B": B, "U": U})


def t_pp(profiles: Sequence[StageProfile], comm: CommModel) -> CostEstimate:
    """Naive pipeline: the serial chain plus Q."""
    base = t_e2e(profiles)
    return CostEstimate("naive_pp", base.batch_time + comm.q_total,
                        dict(base.components, Q=comm.q_total))


def t_ppll(profiles: Sequence[StageProfile], comm: CommModel) -> CostEstimate:
    """Steady PPLL batch time when stage 1 governs: its block forward, Q, its
    aux forward, block+aux backward and update (summed in the simulator's
    event order)."""
    _need(profiles)
    p = profiles[0]
    total = p.f + comm.q_total + p.f_a + (p.b + p.b_a) + (p.u + p.u_a)
    return CostEstimate("ppll", total, {"F_a1": p.f + p.f_a, "B_a1": p.b + p.b_a,
                                        "U_a1": p.u + p.u_a, "Q": comm.q_total})


def ratio_ideal(k: float, s: int) -> float:
    """(k + 1) / s: PPLL over PP for uniform stages and aux cost k."""
    if s < 1:
        raise ValueError(f"need s >= 1, got {s}")
    if k < 0:
        raise ValueError(f"need k >= 0, got {k}")
    return (k + 1.0) / s


def ppll_beats_pp(profiles: Sequence[StageProfile], comm: CommModel):
    """Verdict plus the three margins whose joint positivity suffices."""
    _need(profiles)
    p1 = profiles[0]
    margins = {
        "backward_margin": sum(p.b for p in profiles) - (p1.b + p1.b_a),
        "update_margin": sum(p.u for p in profiles) - (p1.u + p1.u_a),
        "forward_margin": sum(p.f for p in profiles[1:]) - p1.f_a,
    }
    return t_ppll(profiles, comm).batch_time < t_pp(profiles, comm).batch_time, margins


@dataclass(frozen=True)
class ScheduleEvent:
    stage: int
    kind: str      # forward | aux_forward | backward | update | comm
    batch_id: int
    start: float
    end: float


@dataclass(frozen=True)
class ScheduleResult:
    events: tuple
    makespan: float
    steady_batch_time: float
    batch_finish: tuple

    def idle_fraction(self, n_stages: int, skip: int | None = None) -> list:
        """Per-stage 1 − busy/span in steady state: for stage j the span runs
        from the end of its batch ``skip - 1`` to the end of its last batch
        and busy is its (non-transfer) event time for the batches in between
        (default skip: the 2·s-batch fill transient)."""
        n = len(self.batch_finish)
        skip = 2 * n_stages if skip is None else skip
        if n <= skip + 1:
            skip = 1 if n > 1 else 0
        out = []
        for j in range(n_stages):
            ev = [e for e in self.events if e.stage == j]
            if not ev:
                out.append(1.0)
                continue
            end = {}
            for e in ev:
                end[e.batch_id] = max(end.get(e.batch_id, 0.0), e.end)
            t0 = end.get(skip - 1, 0.0) if skip > 0 else min(e.start for e in ev)
            t1 = end[n - 1]
            busy = sum(e.end - e.start for e in ev if e.batch_id >= skip and e.kind != "comm")
            out.append(max(0.0, 1.0 - busy / max(t1 - t0, 1e-30)))
        return out


def simulate_schedule(profiles: Sequence[StageProfile], comm: CommModel, mode: str,
                      n_batches: int, buffer_capacity: int = 2) -> ScheduleResult:
    """Event timeline of ``n_batches``; ``steady_batch_time`` is the finish
    gap of the last two batches (run >= 2·s batches)."""
    _need(profiles)
    if mode not in MODES:
        raise InvalidMode(f"mode must be one of {MODES}, got {mode!r}")
    if n_batches < 1:
        raise ValueError("n_batches must be >= 1")
    if buffer_capacity < 1:
        raise ValueError("buffer_capacity must be >= 1")
    if mode == "ppll":
        events, fin = _ppll_timeline(profiles, comm, n_batches, buffer_capacity)
    else:
        events, fin = _serial_timeline(profiles, comm, mode, n_batches)
    makespan = max((e.end for e in events), default=0.0)
    steady = fin[-1] - fin[-2] if n_batches >= 2 else fin[-1]
    return ScheduleResult(tuple(events), makespan, steady, tuple(fin))


def _serial_timeline(profiles, comm, mode, n):
    s = len(profiles)
    ev, fin = [], []
    now = [0.0]

    def run(stage, kind, t, dur):
        ev.append(ScheduleEvent(stage, kind, t, now[0], now[0] + dur))
        now[0] += dur

    for t in range(n):
        for j, p in enumerate(profiles):
            run(j, "forward", t, p.f)
        if mode == "naive_pp":
            run(s - 1, "comm", t, comm.q_total)
            for j in range(s - 1, -1, -1):
                run(j, "backward", t, profiles[j].b)
                run(j, "update", t, profiles[j].u)
        else:
            for j in range(s - 1, -1, -1):
                run(j, "backward", t, profiles[j].b)
            for j, p in enumerate(profiles):
                run(j, "update", t, p.u)
        fin.append(now[0])
    return ev, fin


def _ppll_timeline(profiles, comm, n, cap):
    s = len(profiles)
    ev = []
    pushed = [[0.0] * n for _ in range(s)]
    started = [[0.0] * n for _ in range(s)]
    finished = [[0.0] * n for _ in range(s)]
    for t in range(n):
        for j, p in enumerate(profiles):
            now = max(pushed[j - 1][t] if j else 0.0, finished[j][t - 1] if t else 0.0)
            started[j][t] = now
            seq = [("forward", p.f)] + ([("comm", comm.q_total)] if j == 0 else [])
            for kind, dur in seq:
                ev.append(ScheduleEvent(j, kind, t, now, now + dur))
                now += dur
            if j < s - 1:
                if t >= cap:                      # credit: slot t-cap drained
                    now = max(now, started[j + 1][t - cap])
                pushed[j][t] = now
            for kind, dur in (("aux_forward", p.f_a), ("backward", p.b + p.b_a),
                              ("update", p.u + p.u_a)):
                ev.append(ScheduleEvent(j, kind, t, now, now + dur))
                now += dur
            finished[j][t] = now
    return ev, [max(finished[j][t] for j in range(s)) for t in range(n)]


def steady_throughput(result: ScheduleResult) -> float:
    if result.steady_batch_time <= 0.0:
        raise ZeroDuration("steady batch time is not positive")
    return 1.0 / result.steady_batch_time


def render_gantt_csv(events: Sequence[ScheduleEvent]) -> str:
    """One row per event, ordered by (start, stage)."""
    if not events:
        raise EmptyEvents("no events to render")
    out = ["stage,kind,batch_id,start,end"]
    for e in sorted(events, key=lambda e: (e.start, e.stage)):
        out.append(f"{e.stage},{e.kind},{e.batch_id},{e.start!r},{e.end!r}")
    return "\n".join(out) + "\n"


# --------------------------------------------------------------------------
# calibration on the device
# --------------------------------------------------------------------------

def _fwd_fraction(m) -> float:
    """Share of a stage's forward time spent before the push (its block):
    MLP by parameter (= FLOP) count, ViT by layer count, ResNet by units."""
    if hasattr(m, "n_block_layers") and hasattr(m, "n_aux_layers"):
        nb, na = m.n_block_layers, m.n_aux_layers
        return nb / max(1, nb + na)
    if hasattr(m, "block_ids") and hasattr(m, "n_aux_convs"):
        nb = 2 * len(m.block_ids) + (1 if getattr(m, "has_stem", False) else 0)
        return nb / max(1, nb + m.n_aux_convs)
    if hasattr(m, "layers") and hasattr(m, "aux"):
        blk = sum(l.W.data.size for l in m.layers)
        aux = sum(l.W.data.size for l in m.aux.layers) if m.aux is not None else 0
        return blk / max(1, blk + aux)
    return 0.8


def calibrate(modules, batch: int, reps: int = 20) -> list:
    """Measured StageProfiles (seconds) for a batch of ``batch`` rows: each
    stage's full local step and its forward are replayed from CUDA graphs on
    one stream and timed with CUDA events; the forward splits into block
    (before the push) and aux by ``_fwd_fraction``, the remainder of the step
    (backward + update) is charged to ``b`` (the simulator only uses the push
    point and the cycle)."""
    import numpy as np
    import torch
    out = []
    for m in modules:
        dev = m.device
        with torch.cuda.device(dev):
            m.native(batch)
            x = torch.randn((batch,) + tuple(m.in_shape), device=dev).to(m.act_dtype)
            y = torch.as_tensor(np.arange(batch) % m.num_classes, device=dev)
            h = torch.empty((batch,) + tuple(m.out_shape), device=dev, dtype=m.act_dtype)
            lg = torch.empty((batch, m.num_classes), device=dev, dtype=m.act_dtype)
            st = torch.cuda.Stream(device=dev)
            step0 = m.device_step()
            times = {}
            for kind in ("forward", "step"):
                fn = ((lambda s: m.launch_forward(batch, x.data_ptr(), h.data_ptr(),
                                                  lg.data_ptr(), s)) if kind == "forward"
                      else (lambda s: m.launch_step(batch, x.data_ptr(), y.data_ptr(),
                                                    h.data_ptr(), s)))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    fn(st.cuda_stream)
                g.replay()
                torch.cuda.synchronize(dev)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st):
                    a.record(st)
                    for _ in range(reps):
                        g.replay()
                    b.record(st)
                b.synchronize()
                times[kind] = a.elapsed_time(b) / reps / 1e3
            # the calibration steps trained the module: restore its step count
            # bookkeeping (parameters moved; callers calibrate on scratch modules)
            m.optimizer.step_count += m.device_step() - step0
            fr = _fwd_fraction(m)
            f = times["forward"] * fr
            f_a = times["forward"] - f
            out.append(StageProfile(f=f, b=max(0.0, times["step"] - times["forward"]), u=0.0,
                                    f_a=f_a))
    return out
