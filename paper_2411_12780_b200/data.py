"""Data path: the reference's dataset container and seeded batch order
(``data.py:24-48, 148-179``), plus an HBM-resident twin that assembles every
batch on the device.

``Dataset`` / ``BatchIterator`` / ``batches`` keep the reference's contract:
float features ``[N x D]`` with integer labels in ``[0, C)``, a single pass in
a fixed order — ``default_rng(seed).permutation(N)`` when shuffling, the
identity otherwise — and a short final batch.  ``DeviceDataset`` uploads the
features (fp32) and labels once; ``DeviceDataset.batches`` yields the SAME
index order as device tensors gathered by ``ppll_gather_rows`` (one warp per
row, 16-B vectors, optional fused bf16 cast), so an epoch moves no host data
per batch.  ``run_epoch`` consumes either form (host arrays are staged
through pinned memory; device tensors go straight to the first ring).

The synthetic generators and the IDX reader of the reference are data
tooling outside the hot path and are not rebuilt here.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import InvalidArg


@dataclass(frozen=True)
class Dataset:
    """Feature matrix [N x D] with integer labels in [0, C) (data.py:24-48)."""

    features: np.ndarray
    labels: np.ndarray
    num_classes: int

    def __post_init__(self):
        f, y = np.asarray(self.features), np.asarray(self.labels)
        if f.ndim != 2 or f.shape[0] < 1:
            raise InvalidArg(f"features must be a non-empty [N x D] matrix, got {f.shape}")
        if y.shape != (f.shape[0],):
            raise InvalidArg("labels must be one integer per row of features")
        if not np.isfinite(f).all():
            raise InvalidArg("features contain non-finite values")
        if self.num_classes < 1 or y.min() < 0 or y.max() >= self.num_classes:
            raise InvalidArg(f"labels must lie in [0, {self.num_classes})")

    @property
    def n(self) -> int:
        return self.features.shape[0]

    @property
    def dim(self) -> int:
        return self.features.shape[1]


def _order(n: int, shuffle: bool, seed: int) -> np.ndarray:
    """The epoch's row order (data.py:155-158)."""
    return np.random.default_rng(seed).permutation(n) if shuffle else np.arange(n)


class BatchIterator:
    """Single pass over a dataset in a fixed (optionally shuffled) order;
    ``ceil(N / batch_size)`` batches, the last may be short (data.py:148-173)."""

    def __init__(self, dataset: Dataset, batch_size: int, shuffle: bool, seed: int):
        if batch_size < 1:
            raise InvalidArg(f"batch_size must be >= 1, got {batch_size}")
        self.dataset = dataset
        self.batch_size = batch_size
        self.order = _order(dataset.n, shuffle, seed)
        self.cursor = 0

    def __len__(self) -> int:
        return -(-self.dataset.n // self.batch_size)

    def __iter__(self) -> "BatchIterator":
        return self

    def __next__(self):
        if self.cursor >= self.dataset.n:
            raise StopIteration
        idx = self.order[self.cursor:self.cursor + self.batch_size]
        self.cursor += self.batch_size
        return self.dataset.features[idx], self.dataset.labels[idx]


def batches(dataset: Dataset, batch_size: int, shuffle: bool = False,
            seed: int = 0) -> BatchIterator:
    """Fresh batch iterator; equal seeds yield equal orders (data.py:176-179)."""
    return BatchIterator(dataset, batch_size, shuffle, seed)


class DeviceDataset:
    """A ``Dataset`` resident in HBM (fp32 features, int64 labels).

    ``batches(batch_size, shuffle, seed, dtype)`` yields ``(x, y)`` device
    tensors in exactly ``BatchIterator``'s order; ``x`` is fp32 or, with
    ``dtype=torch.bfloat16``, already cast for a bf16 first stage.  Each batch
    is one gather launch into fresh caching-allocator blocks on the current
    stream; consumers on other streams mark them with ``record_stream`` (as
    ``run_epoch`` does) so a block is not recycled while still being read."""

    def __init__(self, dataset: Dataset, device=None):
        self.dataset = dataset
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.features = torch.as_tensor(np.ascontiguousarray(dataset.features, dtype=np.float32),
                                        device=self.device)
        self.labels = torch.as_tensor(np.asarray(dataset.labels, dtype=np.int64),
                                      device=self.device)

    @property
    def n(self) -> int:
        return self.dataset.n

    @property
    def dim(self) -> int:
        return self.dataset.dim

    def gather(self, idx: torch.Tensor, out_x: torch.Tensor, out_y: torch.Tensor,
               stream=None) -> None:
        """out_x[r] = features[idx[r]], out_y[r] = labels[idx[r]] (device)."""
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        code = N.BF16 if out_x.dtype == torch.bfloat16 else N.F32
        N.check(N.load().ppll_gather_rows(int(idx.numel()), self.dim, self.features.data_ptr(),
                                          idx.data_ptr(), out_x.data_ptr(), code,
                                          self.labels.data_ptr(), out_y.data_ptr(), s), "gather")

    def batches(self, batch_size: int, shuffle: bool = False, seed: int = 0,
                dtype=torch.float32):
        if batch_size < 1:
            raise InvalidArg(f"batch_size must be >= 1, got {batch_size}")
        order = torch.as_tensor(_order(self.n, shuffle, seed), dtype=torch.int64,
                                device=self.device)
        for start in range(0, self.n, batch_size):
            idx = order[start:start + batch_size]
            b = int(idx.numel())
            x = torch.empty((b, self.dim), dtype=dtype, device=self.device)
            y = torch.empty((b,), dtype=torch.int64, device=self.device)
            self.gather(idx, x, y)
            yield x, y
