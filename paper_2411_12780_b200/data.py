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

The reference's dataset sources are here too: the
seeded synthetic generators ``gen_blobs`` / ``gen_spirals`` (same PCG64 draw
order, so the same seed gives the same rows) and the big-endian IDX reader
``load_idx``.  An IDX dataset keeps the file's pixel bytes next to the
float view; ``DeviceDataset`` then holds those bytes in HBM (1 B/feature)
and ``ppll_gather_rows_u8`` applies the /255 scaling per batch on the device.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .errors import BadMagic, CountMismatch, InvalidArg, TruncatedFile


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


@dataclass(frozen=True)
class IdxDataset(Dataset):
    """A ``Dataset`` read from IDX files that also keeps the raw pixel bytes
    ``[N x D]`` uint8 (``features == pixels / 255``)."""

    pixels: np.ndarray = field(default=None, repr=False, compare=False)


# blob class means: the class index unravelled on a side^dim integer lattice,
# scaled by 4 (data.py:14-16, 64-75)
BLOB_LATTICE_SPACING = 4.0
# spiral arm: theta in [0.5, 0.5 + 1.5 * 2pi), radius = theta / theta_end
# (data.py:18-21, 78-87)
SPIRAL_BASE_ANGLE = 0.5
SPIRAL_TURNS = 1.5


def gen_blobs(n_per_class: int, classes: int, dim: int, spread: float,
              seed: int) -> Dataset:
    """One isotropic Gaussian cluster per class (data.py:52-75).

    Rows are grouped by class; class ``c`` is centred at the lattice point
    ``unravel_index(c, (side,)*dim) * 4`` with the smallest ``side`` such that
    ``side**dim >= classes``.  One ``default_rng(seed)``, drawn class by class
    ``normal(0, spread, (n_per_class, dim))``, so equal seeds give bit-equal
    data.  ``spread == 0`` puts every row on its mean.
    """
    if min(n_per_class, classes, dim) < 1:
        raise InvalidArg("n_per_class, classes, and dim must all be >= 1")
    if spread < 0:
        raise InvalidArg(f"spread must be >= 0, got {spread}")
    side = 1
    while side ** dim < classes:
        side += 1
    rng = np.random.default_rng(seed)
    n = classes * n_per_class
    features = np.empty((n, dim), dtype=np.float64)
    for c in range(classes):
        centre = np.asarray(np.unravel_index(c, (side,) * dim), dtype=np.float64)
        rows = slice(c * n_per_class, (c + 1) * n_per_class)
        features[rows] = centre * BLOB_LATTICE_SPACING + \
            rng.normal(0.0, spread, size=(n_per_class, dim))
    labels = np.repeat(np.arange(classes, dtype=np.int64), n_per_class)
    return Dataset(features, labels, classes)


def spiral_reference(n_per_class: int) -> tuple[np.ndarray, np.ndarray]:
    """The two noise-free spiral arms, ``[n x 2]`` each (data.py:78-87); the
    second arm is the first rotated by pi."""
    t = np.arange(n_per_class, dtype=np.float64) / n_per_class
    end = SPIRAL_BASE_ANGLE + 2.0 * np.pi * SPIRAL_TURNS
    theta = SPIRAL_BASE_ANGLE + 2.0 * np.pi * SPIRAL_TURNS * t
    r = theta / end
    arm = np.stack([r * np.cos(theta), r * np.sin(theta)], axis=1)
    return arm, -arm


def gen_spirals(n_per_class: int, noise: float, seed: int) -> Dataset:
    """Two interleaved spiral arms, class 0 then class 1, plus isotropic
    Gaussian noise ``normal(0, noise, (2n, 2))`` from ``default_rng(seed)``
    (data.py:90-104)."""
    if n_per_class < 1:
        raise InvalidArg("n_per_class must be >= 1")
    if noise < 0:
        raise InvalidArg(f"noise must be >= 0, got {noise}")
    arm0, arm1 = spiral_reference(n_per_class)
    clean = np.concatenate([arm0, arm1], axis=0)
    labels = np.repeat(np.array([0, 1], dtype=np.int64), n_per_class)
    noisy = clean + np.random.default_rng(seed).normal(0.0, noise, size=clean.shape)
    return Dataset(noisy, labels, 2)


_IDX_IMAGES = 0x00000803     # unsigned-byte data, 3 dimensions
_IDX_LABELS = 0x00000801     # unsigned-byte data, 1 dimension


def _idx_dims(raw: bytes, n_dims: int, magic: int, path) -> tuple[int, ...]:
    """Big-endian magic + ``n_dims`` uint32 sizes (data.py:107-115)."""
    need = 4 * (n_dims + 1)
    if len(raw) < need:
        raise TruncatedFile(f"{path}: header needs {need} bytes, file has {len(raw)}")
    head = struct.unpack(">" + "I" * (n_dims + 1), raw[:need])
    if head[0] != magic:
        raise BadMagic(f"{path}: magic {head[0]:#010x}, expected {magic:#010x}")
    return head[1:]


def load_idx(images_path, labels_path) -> IdxDataset:
    """An IDX image/label pair as a flat dataset (data.py:118-144).

    Images ``[count, rows, cols]`` bytes become feature rows scaled by 1/255;
    labels are bytes; ``num_classes = max label + 1``.  Bytes after the
    declared payload are ignored; a short payload raises ``TruncatedFile``, a
    wrong magic ``BadMagic``, differing counts ``CountMismatch``.
    """
    img = Path(images_path).read_bytes()
    count, rows, cols = _idx_dims(img, 3, _IDX_IMAGES, images_path)
    n_pix = count * rows * cols
    if len(img) - 16 < n_pix:
        raise TruncatedFile(f"{images_path}: payload has {len(img) - 16} bytes, "
                            f"header declares {n_pix}")
    lbl = Path(labels_path).read_bytes()
    (n_lbl,) = _idx_dims(lbl, 1, _IDX_LABELS, labels_path)
    if len(lbl) - 8 < n_lbl:
        raise TruncatedFile(f"{labels_path}: payload has {len(lbl) - 8} bytes, "
                            f"header declares {n_lbl}")
    if n_lbl != count:
        raise CountMismatch(f"{count} images but {n_lbl} labels")
    pixels = np.frombuffer(img, dtype=np.uint8, count=n_pix, offset=16).reshape(count, rows * cols).copy()
    labels = np.frombuffer(lbl, dtype=np.uint8, count=n_lbl, offset=8).astype(np.int64)
    features = pixels.astype(np.float64) / 255.0
    return IdxDataset(features, labels, int(labels.max()) + 1 if n_lbl else 0, pixels=pixels)


# ---------------------------------------------------------------------------
# the image datasets of the paper's configurations (BASELINE configs: CIFAR-10
# 32x32, SVHN 32x32, STL-10 96x96) in their distribution formats.  The
# reference ships only the IDX reader above; these follow the same contract
# (uint8 pixels kept for the 1-B/feature HBM copy, features = pixels / 255 in
# fp32 — the device's ppll_gather_rows_u8 rounding) and the same error
# classes.  ``layout`` picks the feature order a family's stage 0 takes:
# "nchw" (ViT patch embedding, VitLocalModule.in_shape) or "nhwc" (ResNet,
# ResNetLocalModule.in_shape).
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ImageDataset(IdxDataset):
    """An image dataset: ``pixels`` [N x C·H·W] uint8 in ``layout`` order."""

    shape: tuple = (0, 0, 0)          # (C, H, W)
    layout: str = "nchw"


def _image_dataset(chw: np.ndarray, labels: np.ndarray, classes: int, layout: str) -> ImageDataset:
    """chw: uint8 [N, C, H, W] -> ImageDataset in the requested layout."""
    if layout not in ("nchw", "nhwc"):
        raise InvalidArg(f"layout must be 'nchw' or 'nhwc', got {layout!r}")
    n, c, h, w = chw.shape
    arr = chw if layout == "nchw" else chw.transpose(0, 2, 3, 1)
    pixels = np.ascontiguousarray(arr).reshape(n, c * h * w)
    features = (pixels.astype(np.float64) / 255.0).astype(np.float32)
    return ImageDataset(features, labels.astype(np.int64), classes, pixels=pixels,
                        shape=(c, h, w), layout=layout)


def load_cifar10(paths, layout: str = "nchw", cifar100: bool = False) -> ImageDataset:
    """CIFAR-10 (or -100) binary batches (``data_batch_*.bin`` /
    ``test_batch.bin``): records of a label byte (CIFAR-100: coarse + fine,
    the fine label is used) followed by 3072 bytes — the red, green and blue
    32x32 planes, row-major.  ``paths``: one file or a list (concatenated)."""
    if isinstance(paths, (str, Path)):
        paths = [paths]
    lb = 2 if cifar100 else 1
    rec = lb + 3072
    imgs, labels = [], []
    for p in paths:
        raw = Path(p).read_bytes()
        if len(raw) == 0 or len(raw) % rec:
            raise TruncatedFile(f"{p}: {len(raw)} bytes is not a whole number of "
                                f"{rec}-byte records")
        a = np.frombuffer(raw, dtype=np.uint8).reshape(-1, rec)
        labels.append(a[:, lb - 1])
        imgs.append(a[:, lb:].reshape(-1, 3, 32, 32))
    y = np.concatenate(labels)
    classes = 100 if cifar100 else 10
    if y.max() >= classes:
        raise InvalidArg(f"label {int(y.max())} outside [0, {classes})")
    return _image_dataset(np.concatenate(imgs), y, classes, layout)


def load_svhn(path, layout: str = "nchw") -> ImageDataset:
    """SVHN cropped digits (``train_32x32.mat`` / ``test_32x32.mat``, MATLAB
    v5): ``X`` uint8 [32, 32, 3, N], ``y`` [N, 1] with the digit 0 stored as
    label 10 (mapped back to 0)."""
    from scipy.io import loadmat
    try:
        m = loadmat(str(path))
    except (ValueError, TypeError, OSError) as e:
        raise TruncatedFile(f"{path}: not a readable MATLAB v5 file ({e})") from e
    if "X" not in m or "y" not in m:
        raise InvalidArg(f"{path}: expected variables X and y")
    x, y = np.asarray(m["X"]), np.asarray(m["y"]).reshape(-1).astype(np.int64)
    if x.ndim != 4 or x.shape[2] != 3 or x.shape[3] != y.size:
        raise CountMismatch(f"{path}: X {x.shape} does not match {y.size} labels")
    y = np.where(y == 10, 0, y)
    if y.min() < 0 or y.max() > 9:
        raise InvalidArg(f"{path}: labels outside [1, 10]")
    return _image_dataset(np.ascontiguousarray(x.transpose(3, 2, 0, 1)), y, 10, layout)


def load_stl10(x_path, y_path, layout: str = "nchw") -> ImageDataset:
    """STL-10 binary (``train_X.bin`` / ``train_y.bin``): images uint8
    [N, 3, 96, 96] with each channel plane stored column-major, labels 1..10
    (mapped to 0..9)."""
    raw = Path(x_path).read_bytes()
    per = 3 * 96 * 96
    if len(raw) == 0 or len(raw) % per:
        raise TruncatedFile(f"{x_path}: {len(raw)} bytes is not a whole number of images")
    x = np.frombuffer(raw, dtype=np.uint8).reshape(-1, 3, 96, 96).transpose(0, 1, 3, 2)
    y = np.frombuffer(Path(y_path).read_bytes(), dtype=np.uint8).astype(np.int64)
    if y.size != x.shape[0]:
        raise CountMismatch(f"{x.shape[0]} images but {y.size} labels")
    if y.size and (y.min() < 1 or y.max() > 10):
        raise InvalidArg(f"{y_path}: labels outside [1, 10]")
    return _image_dataset(np.ascontiguousarray(x), y - 1, 10, layout)


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
    """A ``Dataset`` resident in HBM (fp32 features, int64 labels; an
    ``IdxDataset`` is held as its uint8 pixels and scaled per batch).

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
        pixels = getattr(dataset, "pixels", None)
        src = pixels if pixels is not None else np.ascontiguousarray(dataset.features,
                                                                     dtype=np.float32)
        self.features = torch.as_tensor(np.ascontiguousarray(src), device=self.device)
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
        fn = N.load().ppll_gather_rows_u8 if self.features.dtype == torch.uint8 \
            else N.load().ppll_gather_rows
        N.check(fn(int(idx.numel()), self.dim, self.features.data_ptr(), idx.data_ptr(),
                   out_x.data_ptr(), code, self.labels.data_ptr(), out_y.data_ptr(), s), "gather")

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
