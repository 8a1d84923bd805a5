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

The experiment driver, config parser and comparison report of the reference
are orchestration/UI outside the hot path and are not rebuilt.
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import torch

from . import _native as N
from .data import Dataset, DeviceDataset
from .errors import InvalidValue, IoError

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


__all__ = ["CSV_HEADER", "MetricsRecord", "evaluate", "device_memory", "write_metrics_csv",
           "Dataset", "DeviceDataset"]
