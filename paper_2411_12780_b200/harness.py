"""Evaluation and metrics records (harness.py:40-52,
121-131, 238-252 of the reference).

``evaluate`` is the accuracy of the composed network — every stage's block
forward, the final stage's output as the task logits — computed on the
device: the dataset is made HBM-resident once (``DeviceDataset``), each chunk
is gathered on the device, runs the stages' native forward and is scored by
``ppll_count_correct`` (numpy-style first-maximum argmax, integer count).
``write_metrics_csv`` writes the reference's CSV schema.  ``device_memory``
reports the bytes a stage actually holds on its GPU (parameters, momenta,
gradients, bf16 shadow, executor workspace), next to the reference's float
count proxy ``memory_footprint``.

``run_experiment`` is the reference's caller of the hot path
(harness.py:78-235): every requested mode trains from bit-identical freshly
built modules on the same seeded batch order (shuffle seed ``seed + epoch``),
one ``MetricsRecord`` per epoch, then a ``ComparisonReport`` with the
measured aux/block cost ratio ``k``.  Here the training set is made
HBM-resident once and every epoch's batches are gathered on the device.
``ExperimentConfig`` keeps the reference's keys, defaults and validation
(config.py:18-72, 155-183); its text grammar / CLI are out of scope.
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import torch

from . import _native as N
from .blocks import Hyperparams, NetworkSpec, build_modules, memory_footprint, partition
from .data import Dataset, DeviceDataset, gen_blobs, gen_spirals, load_idx
from .errors import ConfigMismatch, InvalidValue, IoError
from .runtime import RunConfig, RunMode, run_deterministic, run_epoch, throughput

CSV_HEADER = ("mode,epoch,batches_per_sec,mean_loss,train_acc,test_acc,"
              "params_max_stage,activations_max_stage,mean_staleness")


@dataclass(frozen=True)
class MetricsRecord:
    """One epoch of one mode, as it appears in the metrics CSV."""

    mode: str
    epoch: int
    batches_per_sec: float
    mean_loss: float
    train_acc: float
    test_acc: float
    params_max_stage: int
    activations_max_stage: int
    mean_staleness: float


@dataclass(frozen=True)
class ModeSummary:
    """Final-epoch numbers of one mode (harness.py:58-66)."""

    mode: str
    batches_per_sec: float
    test_acc: float
    params_max_stage: int
    activations_max_stage: int


@dataclass(frozen=True)
class ComparisonReport:
    """Per-mode summaries plus the analytic PPLL/PP ratio (k+1)/s
    (harness.py:69-75)."""

    stages: int
    measured_k: float
    analytic_ratio: float
    summaries: tuple
    ppll_over_pp_throughput: float | None


@dataclass(frozen=True)
class ExperimentConfig:
    """A training run (config.py:18-67): dataset, network, pipeline and
    optimizer settings, with the reference's defaults.  ``precision`` is this
    build's addition (device arithmetic, ``Hyperparams.precision``)."""

    dataset: str = ""
    n_per_class: int = 100
    classes: int = 2
    dim: int = 2
    spread: float = 0.5
    noise: float = 0.08
    idx_train_images: str | None = None
    idx_train_labels: str | None = None
    idx_test_images: str | None = None
    idx_test_labels: str | None = None
    layer_dims: tuple = ()
    stages: int = 1
    buffer_capacity: int = 2
    aux_depth_max: int = 2
    aux_depth_interval: int = 3
    aux_hidden_width: int | None = None
    batch_size: int = 32
    epochs: int = 1
    lr0: float = 0.01
    lr_min: float = 0.0
    momentum: float = 0.9
    weight_decay: float = 1e-4
    seed: int = 42
    modes: tuple = (RunMode.E2E, RunMode.NAIVE_PP, RunMode.PPLL)
    sleep_padding: tuple = (0.0,)
    comm_padding: float = 0.0
    precision: str = "fp32"

    def __post_init__(self):
        validate_config(self)


def validate_config(cfg: ExperimentConfig) -> None:
    """The reference's semantic checks, as ``InvalidValue`` (config.py:155-183)."""
    if cfg.dataset not in ("blobs", "spirals", "idx"):
        raise InvalidValue(f"dataset must be blobs, spirals, or idx, got {cfg.dataset!r}")
    dims = tuple(cfg.layer_dims)
    if len(dims) < 2 or min(dims) < 1:
        raise InvalidValue(f"layer_dims needs >= 2 positive entries, got {dims}")
    if cfg.dataset == "idx" and not (cfg.idx_train_images and cfg.idx_train_labels):
        raise InvalidValue("dataset idx needs idx_train_images and idx_train_labels")
    for name in ("n_per_class", "classes", "dim", "stages", "buffer_capacity",
                 "aux_depth_interval", "batch_size", "epochs"):
        if getattr(cfg, name) < 1:
            raise InvalidValue(f"{name} must be >= 1, got {getattr(cfg, name)}")
    for name in ("spread", "noise", "aux_depth_max", "lr0", "lr_min", "weight_decay",
                 "comm_padding"):
        if getattr(cfg, name) < 0:
            raise InvalidValue(f"{name} must be >= 0, got {getattr(cfg, name)}")
    if not 0.0 <= cfg.momentum < 1.0:
        raise InvalidValue(f"momentum must lie in [0, 1), got {cfg.momentum}")
    if cfg.lr_min > cfg.lr0:
        raise InvalidValue(f"lr_min {cfg.lr_min} exceeds lr0 {cfg.lr0}")
    if cfg.aux_hidden_width is not None and cfg.aux_hidden_width < 1:
        raise InvalidValue("aux_hidden_width must be >= 1 when given")
    if any(p < 0 for p in cfg.sleep_padding):
        raise InvalidValue("sleep_padding entries must be >= 0")
    if cfg.stages > len(dims) - 1:
        raise InvalidValue(f"stages = {cfg.stages} exceeds the {len(dims) - 1} layers "
                           f"of layer_dims {dims}")
    if not cfg.modes or len(set(cfg.modes)) != len(cfg.modes):
        raise InvalidValue("modes must list each mode at most once and not be empty")
    if cfg.precision not in ("fp32", "bf16"):
        raise InvalidValue(f"precision must be fp32 or bf16, got {cfg.precision!r}")


def make_datasets(cfg: ExperimentConfig) -> tuple:
    """(train, test) for the config (harness.py:78-106): synthetic data uses
    ``seed`` for training and ``seed + 1`` for test; IDX without a test pair
    evaluates on the training set."""
    if cfg.dataset == "blobs":
        train = gen_blobs(cfg.n_per_class, cfg.classes, cfg.dim, cfg.spread, cfg.seed)
        test = gen_blobs(cfg.n_per_class, cfg.classes, cfg.dim, cfg.spread, cfg.seed + 1)
    elif cfg.dataset == "spirals":
        train = gen_spirals(cfg.n_per_class, cfg.noise, cfg.seed)
        test = gen_spirals(cfg.n_per_class, cfg.noise, cfg.seed + 1)
    elif cfg.dataset == "idx":
        train = load_idx(cfg.idx_train_images, cfg.idx_train_labels)
        test = (load_idx(cfg.idx_test_images, cfg.idx_test_labels)
                if cfg.idx_test_images and cfg.idx_test_labels else train)
    else:
        raise InvalidValue(f"unknown dataset kind {cfg.dataset!r}")
    if train.dim != cfg.layer_dims[0]:
        raise ConfigMismatch(f"dataset dim {train.dim} != layer_dims[0] {cfg.layer_dims[0]}")
    if train.num_classes != cfg.layer_dims[-1]:
        raise ConfigMismatch(f"dataset has {train.num_classes} classes but layer_dims ends "
                             f"in {cfg.layer_dims[-1]}")
    return train, test


def build_pipeline(cfg: ExperimentConfig, steps_per_epoch: int) -> list:
    """Fresh modules for one mode (harness.py:109-118): same seed, same init."""
    spec = NetworkSpec(tuple(cfg.layer_dims))
    hyper = Hyperparams(lr0=cfg.lr0, lr_min=cfg.lr_min,
                        total_steps=cfg.epochs * steps_per_epoch, momentum=cfg.momentum,
                        weight_decay=cfg.weight_decay, seed=cfg.seed,
                        aux_hidden_width=cfg.aux_hidden_width, precision=cfg.precision)
    return build_modules(spec, partition(spec, cfg.stages), cfg.aux_depth_max,
                         cfg.aux_depth_interval, hyper)


def estimate_k(cfg: ExperimentConfig, train, trials: int = 3) -> float:
    """Aux/block forward cost ratio of stage 0 (harness.py:134-155), timed on
    the device with CUDA events: block forward alone vs block + aux forward
    on one training batch, on throwaway modules."""
    steps = max(1, -(-train.n // cfg.batch_size))
    first = build_pipeline(cfg, steps)[0]
    b = min(train.n, cfg.batch_size)
    dd = _device_dataset(train, first.device)
    with torch.cuda.device(first.device):
        x = torch.empty((b, dd.dim), dtype=first.act_dtype, device=first.device)
        y = torch.empty((b,), dtype=torch.int64, device=first.device)
        dd.gather(torch.arange(b, device=first.device), x, y)
        h = torch.empty((b, first.out_features), dtype=first.act_dtype, device=first.device)
        first.native(b)
        stream = torch.cuda.current_stream(first.device)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        f = f_a = 0.0
        for _ in range(trials + 1):      # the first pass is a warm-up
            ev[0].record(stream)
            first.launch_block_forward(b, x.data_ptr(), h.data_ptr(), stream.cuda_stream)
            ev[1].record(stream)
            first.launch_forward(b, x.data_ptr(), h.data_ptr(), None, stream.cuda_stream)
            ev[2].record(stream)
            ev[2].synchronize()
            t_f, t_fa = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
            if _ > 0:
                f, f_a = f + t_f, f_a + max(0.0, t_fa - t_f)
        first.close()
    return f_a / f if f > 0 else 0.0


def _epoch_record(cfg, mode, epoch, metrics, modules, train, test) -> MetricsRecord:
    """One CSV row (harness.py:158-172); accuracies are computed on the device."""
    fps = [memory_footprint(m, cfg.batch_size) for m in modules]
    return MetricsRecord(
        mode=mode.value, epoch=epoch,
        batches_per_sec=throughput(metrics, metrics.n_batches),
        mean_loss=metrics.final_stage_mean_loss,
        train_acc=evaluate(modules, train), test_acc=evaluate(modules, test),
        params_max_stage=max(fp.params for fp in fps),
        activations_max_stage=max(fp.activations for fp in fps),
        mean_staleness=metrics.mean_staleness)


def run_experiment(cfg: ExperimentConfig, deterministic: bool = False, out_dir=None):
    """Train every mode of ``cfg.modes`` for ``cfg.epochs`` epochs and build the
    comparison report (harness.py:175-206).  On failure, records collected so
    far are written to ``out_dir/metrics.csv`` before the error propagates."""
    train, test = make_datasets(cfg)
    steps_per_epoch = max(1, -(-train.n // cfg.batch_size))
    run_cfg = RunConfig(buffer_capacity=cfg.buffer_capacity, sleep_padding=cfg.sleep_padding,
                        comm_padding=cfg.comm_padding)
    runner = run_deterministic if deterministic else run_epoch
    records: list = []
    try:
        for mode in cfg.modes:
            modules = build_pipeline(cfg, steps_per_epoch)
            resident = _device_dataset(train, modules[0].device)
            dtype = modules[0].act_dtype
            for epoch in range(cfg.epochs):
                it = resident.batches(cfg.batch_size, shuffle=True, seed=cfg.seed + epoch,
                                      dtype=dtype)
                metrics = runner(mode, modules, it, run_cfg)
                records.append(_epoch_record(cfg, mode, epoch, metrics, modules, train, test))
            for m in modules:
                m.close()
    except Exception:
        if out_dir is not None and records:
            write_metrics_csv(records, Path(out_dir) / "metrics.csv")
        raise
    k = estimate_k(cfg, train)
    return records, _build_report(cfg, records, k)


def _build_report(cfg, records, k) -> ComparisonReport:
    """Final epoch per mode; PPLL/NaivePP throughput ratio when both ran
    (harness.py:209-235)."""
    final = {}
    for r in records:
        final[r.mode] = r if r.mode not in final or r.epoch >= final[r.mode].epoch else final[r.mode]
    summaries = tuple(ModeSummary(final[m.value].mode, final[m.value].batches_per_sec,
                                  final[m.value].test_acc, final[m.value].params_max_stage,
                                  final[m.value].activations_max_stage)
                      for m in cfg.modes if m.value in final)
    ratio = None
    pp, ppll = final.get(RunMode.NAIVE_PP.value), final.get(RunMode.PPLL.value)
    if pp is not None and ppll is not None and pp.batches_per_sec > 0:
        ratio = ppll.batches_per_sec / pp.batches_per_sec
    return ComparisonReport(stages=cfg.stages, measured_k=k,
                            analytic_ratio=(k + 1.0) / cfg.stages, summaries=summaries,
                            ppll_over_pp_throughput=ratio)


def report_table(report: ComparisonReport) -> str:
    """Aligned text table, one row per mode, plus the analytic (k+1)/s line;
    numbers formatted as in the metrics CSV (harness.py:255-273)."""
    rows = [("mode", "batches_per_sec", "test_acc", "params_max_stage",
             "activations_max_stage")]
    rows += [(s.mode, f"{s.batches_per_sec:.6f}", f"{s.test_acc:.6f}",
              str(s.params_max_stage), str(s.activations_max_stage)) for s in report.summaries]
    widths = [max(len(r[i]) for r in rows) for i in range(len(rows[0]))]
    out = ["  ".join(c.ljust(w) for c, w in zip(r, widths)).rstrip() for r in rows]
    out.append(f"analytic (k+1)/s = {report.analytic_ratio:.6f}")
    return "\n".join(out) + "\n"


_resident: dict = {}


def _device_dataset(dataset, device) -> DeviceDataset:
    if isinstance(dataset, DeviceDataset):
        return dataset
    key = (id(dataset), str(device))
    hit = _resident.get(key)
    if hit is None or hit.dataset is not dataset:
        hit = DeviceDataset(dataset, device)
        _resident[key] = hit
    return hit


def evaluate(modules: Sequence, dataset, chunk: int = 512) -> float:
    """Accuracy of the composed network (the final stage's task head) over
    ``dataset`` (a ``Dataset`` or ``DeviceDataset``), on the device."""
    mods = list(modules)
    if not mods:
        raise InvalidValue("evaluate needs at least one stage")
    dev0 = mods[0].device
    dd = _device_dataset(dataset, dev0)
    if dd.dim != mods[0].in_features:
        raise InvalidValue(f"dataset dim {dd.dim} != stage 0 input {mods[0].in_features}")
    # stay within the executors' current batch capacity when they exist
    cap = min([m._native_batch for m in mods if getattr(m, "_native_batch", 0)] or [chunk])
    chunk = max(1, min(chunk, cap))
    lib = N.load()
    stream = torch.cuda.current_stream(dev0)
    count = torch.zeros(1, dtype=torch.int64, device=mods[-1].device)
    h_bufs = [torch.empty((chunk, m.out_features), dtype=m.act_dtype,
                          device=mods[j + 1].device if j + 1 < len(mods) else m.device)
              for j, m in enumerate(mods)]
    last = mods[-1]
    logits = torch.empty((chunk, last.num_classes), dtype=last.act_dtype, device=last.device)
    x0 = torch.empty((chunk, dd.dim), dtype=mods[0].act_dtype, device=dev0)
    y0 = torch.empty((chunk,), dtype=torch.int64, device=dev0)
    ylast = y0 if mods[-1].device == dev0 else torch.empty_like(y0, device=mods[-1].device)
    with torch.cuda.device(dev0):
        for start in range(0, dd.n, chunk):
            b = min(chunk, dd.n - start)
            idx = torch.arange(start, start + b, dtype=torch.int64, device=dev0)
            dd.gather(idx, x0[:b], y0[:b], stream)
            h = x0
            for j, m in enumerate(mods):
                m.native(chunk)
                # the final stage has no aux head: its "logits" are the task head
                lg = logits.data_ptr() if m is last else None
                m.launch_forward(b, h.data_ptr(), h_bufs[j].data_ptr(), lg, stream.cuda_stream)
                h = h_bufs[j]
            if ylast is not y0:
                ylast[:b].copy_(y0[:b], non_blocking=True)
            C = last.num_classes
            N.check(lib.ppll_count_correct(b, C, logits.data_ptr(), C,
                                           N.BF16 if last.act_dtype == torch.bfloat16 else N.F32,
                                           ylast.data_ptr(), count.data_ptr(), stream.cuda_stream),
                    "count_correct")
    return int(count.item()) / dd.n


def device_memory(module) -> dict:
    """Bytes this stage holds on its GPU: flat parameter/momentum/gradient
    buffers (+ bf16 shadow, LR table, loss history) and the native executor's
    workspace (activations kept for the backward, gradient and split-K
    buffers), measured when the executor was created."""
    flat = getattr(module, "_flat", None) or {}
    tensors = sum(t.numel() * t.element_size() for t in flat.values() if torch.is_tensor(t))
    ws = int(getattr(module, "_native_bytes", 0))
    return {"params_state_bytes": int(tensors), "workspace_bytes": ws,
            "total_bytes": int(tensors) + ws}


def write_metrics_csv(records: Sequence[MetricsRecord], path) -> None:
    """The reference's metrics CSV: fixed header, rows ordered by (mode,
    epoch), floats with 6 decimals (harness.py:238-252)."""
    if not records:
        raise InvalidValue("no records to write")
    lines = [CSV_HEADER]
    for r in sorted(records, key=lambda r: (r.mode, r.epoch)):
        lines.append(",".join([
            r.mode, str(r.epoch), f"{r.batches_per_sec:.6f}", f"{r.mean_loss:.6f}",
            f"{r.train_acc:.6f}", f"{r.test_acc:.6f}", str(r.params_max_stage),
            str(r.activations_max_stage), f"{r.mean_staleness:.6f}"]))
    try:
        Path(path).write_text("\n".join(lines) + "\n")
    except OSError as exc:
        raise IoError(f"could not write {path}: {exc}") from exc


__all__ = ["CSV_HEADER", "MetricsRecord", "ModeSummary", "ComparisonReport", "ExperimentConfig",
           "validate_config", "make_datasets", "build_pipeline", "estimate_k", "run_experiment",
           "report_table", "evaluate", "device_memory", "write_metrics_csv", "Dataset",
           "DeviceDataset"]
