"""Device-resident tensors with the reference ``Tensor`` surface (tensor.py:46-83).

The reference keeps float64 numpy arrays and a thread-local tape.  Here a
``Tensor`` wraps a CUDA ``torch`` tensor (fp32 in parity mode, bf16 in
performance mode); there is no tape — each stage's backward is an explicit,
fused kernel sequence in the native executor (``csrc/stage.cu``).  ``.data``
returns a host float64 copy so code written against the reference
(``np.array_equal(p.data, …)``) keeps working; ``.dev`` is the device tensor.

A ``Tensor`` may sit on the CPU only as a container (host bookkeeping such as
``BufferSlot``); every compute entry point requires CUDA and fails loudly
otherwise — there is no CPU fallback.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import DimensionMismatch, LabelOutOfRange, NonFiniteError, NotScalar

_TORCH_DT = {"fp32": torch.float32, "bf16": torch.bfloat16}
_CODE = {torch.float32: N.F32, torch.bfloat16: N.BF16}


def default_device() -> torch.device:
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def require_cuda(t: torch.Tensor, what: str) -> None:
    if t.device.type != "cuda":
        raise RuntimeError(f"{what}: PPLL compute runs only on CUDA devices "
                           f"(got a {t.device} tensor; there is no CPU path)")


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _CODE[t.dtype]
    except KeyError:
        raise DimensionMismatch(f"unsupported dtype {t.dtype}") from None


class Tensor:
    """A device array plus an optional gradient (reference tensor.py:46-83)."""

    __slots__ = ("dev", "grad", "track_grad")

    def __init__(self, data, track_grad: bool = False, dtype=None, device=None):
        if isinstance(data, Tensor):
            data = data.dev
        if torch.is_tensor(data):
            t = data
        else:
            arr = np.asarray(data, dtype=np.float64)
            if not np.isfinite(arr).all():          # tensor.py:41-43,58
                raise NonFiniteError("tensor construction produced non-finite values")
            t = torch.from_numpy(arr)
        if dtype is None:
            dtype = t.dtype if t.dtype in (torch.float32, torch.bfloat16) else torch.float32
        elif isinstance(dtype, str):
            dtype = _TORCH_DT[dtype]
        dev = torch.device(device) if device is not None else (
            t.device if t.device.type == "cuda" else default_device())
        self.dev = t.to(device=dev, dtype=dtype).contiguous()
        self.grad = None
        self.track_grad = bool(track_grad)

    # -- reference surface -------------------------------------------------
    @property
    def shape(self) -> tuple:
        return tuple(self.dev.shape)

    @property
    def size(self) -> int:
        return self.dev.numel()

    @property
    def data(self) -> np.ndarray:
        """Host float64 copy (synchronises the device)."""
        return self.dev.detach().to("cpu", torch.float64).numpy()

    @data.setter
    def data(self, value) -> None:
        src = torch.as_tensor(np.asarray(value, dtype=np.float64))
        if tuple(src.shape) != self.shape:
            raise DimensionMismatch(f"assigning {tuple(src.shape)} into {self.shape}")
        self.dev.copy_(src.to(self.dev.device, self.dev.dtype))

    def detach(self) -> "Tensor":
        """Same storage, no gradient tracking (tensor.py:72-74)."""
        out = Tensor.__new__(Tensor)
        out.dev = self.dev
        out.grad = None
        out.track_grad = False
        return out

    def item(self) -> float:
        if self.size != 1:
            raise NotScalar(f"item() on tensor of shape {self.shape}")
        return float(self.dev.reshape(()).item())

    def numpy(self) -> np.ndarray:
        return self.data

    def __repr__(self) -> str:
        flag = ", track_grad=True" if self.track_grad else ""
        return f"Tensor(shape={self.shape}, dtype={self.dev.dtype}{flag})"


def as_labels(labels, batch: int, num_classes: int, device, check_range: bool = True):
    """Validate labels like softmax_xent (tensor.py:210-219) and place them on
    the device as int64.  With ``check_range=False`` the [0, C) range check is
    left to the device kernel's sticky error word (so callers can keep the
    reference's raise-after-push ordering)."""
    if torch.is_tensor(labels):
        if labels.dtype.is_floating_point:
            raise LabelOutOfRange("labels must be integers")
        y = labels
        if tuple(y.shape) != (batch,):
            raise DimensionMismatch(f"labels shape {tuple(y.shape)} does not match batch {batch}")
        return y.to(device=device, dtype=torch.int64)
    y = np.asarray(labels)
    if y.shape != (batch,):
        raise DimensionMismatch(f"labels shape {y.shape} does not match batch {batch}")
    if not np.issubdtype(y.dtype, np.integer):
        raise LabelOutOfRange("labels must be integers")
    if check_range and batch and (y.min() < 0 or y.max() >= num_classes):
        raise LabelOutOfRange(f"labels must lie in [0, {num_classes})")
    return torch.from_numpy(y.astype(np.int64)).to(device, non_blocking=False)


def matmul(a: Tensor, b: Tensor) -> Tensor:
    """Forward 2-D product a @ b on the device (tensor.py:137-150; no tape)."""
    if a.dev.dim() != 2 or b.dev.dim() != 2:
        raise DimensionMismatch(f"matmul needs 2-D operands, got {a.shape} and {b.shape}")
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"matmul inner dims differ: {a.shape} x {b.shape}")
    require_cuda(a.dev, "matmul")
    if a.dev.dtype != b.dev.dtype:
        raise DimensionMismatch("matmul operands must share a dtype")
    M, K = a.shape
    Nn = b.shape[1]
    out = torch.empty((M, Nn), dtype=a.dev.dtype, device=a.dev.device)
    lib = N.load()
    st = torch.cuda.current_stream(a.dev.device).cuda_stream
    N.check(lib.ppll_linear_fwd(M, K, Nn, a.dev.data_ptr(), K, b.dev.data_ptr(), None,
                                out.data_ptr(), Nn, None, 0, 0, dtype_code(a.dev), st),
            "matmul")
    return Tensor(out)


def softmax_xent(logits: Tensor, labels) -> Tensor:
    """Mean softmax cross-entropy of [B x C] logits (tensor.py:201-234),
    computed by the fused device kernel; returns a scalar fp32 Tensor."""
    if logits.dev.dim() != 2:
        raise DimensionMismatch(f"softmax_xent needs [B x C] logits, got {logits.shape}")
    B, Cc = logits.shape
    if B < 1 or Cc < 1:
        raise DimensionMismatch("softmax_xent needs a non-empty batch")
    require_cuda(logits.dev, "softmax_xent")
    dev = logits.dev.device
    y = as_labels(labels, B, Cc, dev)
    dz = torch.empty_like(logits.dev)
    loss = torch.zeros(1, dtype=torch.float32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = N.load()
    st = torch.cuda.current_stream(dev).cuda_stream
    N.check(lib.ppll_softmax_xent(B, Cc, logits.dev.data_ptr(), Cc, y.data_ptr(), dz.data_ptr(),
                                  Cc, loss.data_ptr(), None, err.data_ptr(),
                                  dtype_code(logits.dev), st), "softmax_xent")
    if int(err.item()) & N.ERRBIT_LOSS:
        raise NonFiniteError("softmax_xent produced non-finite values")
    out = Tensor(loss.reshape(()))
    out.grad = None
    return out
