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
import threading

from .errors import DimensionMismatch, EmptyTape, LabelOutOfRange, NonFiniteError, NotScalar

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

    __slots__ = ("dev", "grad", "track_grad", "_tape")

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
        self._tape = None

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
        out._tape = None
        return out

    def item(self) -> float:
        if self.size != 1:
            raise NotScalar(f"item() on tensor of shape {self.shape}")
        return float(self.dev.reshape(()).item())

    def numpy(self) -> np.ndarray:
        return self.data

    def copy(self) -> np.ndarray:
        """Host copy (the reference's gradients are arrays: ``x.grad.copy()``)."""
        return self.data.copy()

    def __array__(self, dtype=None, copy=None):
        """numpy interop (np.allclose(p.grad, …) as in the reference's tests)."""
        a = self.data
        return a if dtype is None else a.astype(dtype)

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


# --------------------------------------------------------------------------
# the device tape (tensor.py:24-38, 86-132, 239-278)
# --------------------------------------------------------------------------
#
# The PPLL hot path never uses a tape: a stage step is one fused native call
# with an explicit backward.  This Wengert list exists so that a training loop
# written against locopipe's GradTape / backward keeps running, on the device:
# every recorded adjoint is a C-ABI kernel (ppll_linear_dgrad / _wgrad,
# ppll_ew, ppll_colsum), and gradients stay device tensors (``.grad`` is a
# Tensor; ``.grad.data`` is the host float64 copy).

_TLS = threading.local()


def _stack() -> list:
    try:
        return _TLS.stack
    except AttributeError:
        _TLS.stack = []
        return _TLS.stack


def active_tape():
    """The innermost open tape on this thread, or None (tensor.py:33-38)."""
    st = _stack()
    return st[-1] if st else None


class _Node:
    __slots__ = ("out", "pulls")

    def __init__(self, out, pulls):
        self.out = out
        self.pulls = pulls


class GradTape:
    """Ordered record of primitive ops, consumed by one backward pass
    (tensor.py:96-115).  Thread-local like the reference's."""

    def __init__(self):
        self.nodes: list = []
        self.consumed = False
        self.adjoints_run = 0

    def __enter__(self) -> "GradTape":
        _stack().append(self)
        return self

    def __exit__(self, exc_type, exc, tb) -> None:
        _stack().pop()

    def _record(self, out: "Tensor", pulls) -> None:
        out.track_grad = True
        out._tape = self
        self.nodes.append(_Node(out, pulls))


def _record_op(out: "Tensor", pairs) -> "Tensor":
    tape = active_tape()
    if tape is not None:
        pulls = [(t, fn) for t, fn in pairs if t.track_grad]
        if pulls:
            tape._record(out, pulls)
    return out


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _ew(op, a: torch.Tensor, b, alpha=1.0, rows=None, cols=None, check=None) -> torch.Tensor:
    """One ppll_ew launch (tensor.py's elementwise primitives / adjoints)."""
    require_cuda(a, "tape op")
    out = torch.empty_like(a)
    if cols is None:
        cols = a.shape[-1] if a.dim() else 1
        rows = a.numel() // max(cols, 1)
    err = torch.zeros(1, dtype=torch.int32, device=a.device) if check else None
    N.check(N.load().ppll_ew(op, rows, cols, a.data_ptr(), None if b is None else b.data_ptr(),
                             float(alpha), out.data_ptr(), dtype_code(a),
                             None if err is None else err.data_ptr(), _stream(a)), "ppll_ew")
    if err is not None and int(err.item()):
        raise NonFiniteError(f"{check} produced non-finite values")
    return out


def _accumulate(t: "Tensor", g: torch.Tensor) -> None:
    """First write copies, later writes add (tensor.py:128-132)."""
    if t.grad is None:
        t.grad = Tensor(g.clone())
    else:
        t.grad.dev = _ew(3, g, t.grad.dev.to(g.dtype))


def _gemm_dtype(a: Tensor, b: Tensor) -> None:
    if a.dev.dtype != b.dev.dtype:
        raise DimensionMismatch("matmul operands must share a dtype")


def matmul(a: Tensor, b: Tensor) -> Tensor:
    """2-D product a @ b on the device (tensor.py:137-150); under an open tape
    its adjoints dA = g·Bᵀ (ppll_linear_dgrad) and dB = Aᵀ·g
    (ppll_linear_wgrad) are recorded."""
    if a.dev.dim() != 2 or b.dev.dim() != 2:
        raise DimensionMismatch(f"matmul needs 2-D operands, got {a.shape} and {b.shape}")
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"matmul inner dims differ: {a.shape} x {b.shape}")
    require_cuda(a.dev, "matmul")
    _gemm_dtype(a, b)
    M, K = a.shape
    Nn = b.shape[1]
    out = torch.empty((M, Nn), dtype=a.dev.dtype, device=a.dev.device)
    lib = N.load()
    st = _stream(a.dev)
    N.check(lib.ppll_linear_fwd(M, K, Nn, a.dev.data_ptr(), K, b.dev.data_ptr(), None,
                                out.data_ptr(), Nn, None, 0, 0, dtype_code(a.dev), st),
            "matmul")
    _finite(out, "matmul")

    def pull_a(g, b=b, M=M, K=K, Nn=Nn):
        dA = torch.empty((M, K), dtype=g.dtype, device=g.device)
        N.check(N.load().ppll_linear_dgrad(M, K, Nn, g.data_ptr(), Nn, b.dev.data_ptr(), None, 0,
                                           dA.data_ptr(), K, dtype_code(g), _stream(g)),
                "matmul adjoint dA")
        return dA

    def pull_b(g, a=a, M=M, K=K, Nn=Nn):
        dB = torch.empty((K, Nn), dtype=torch.float32, device=g.device)
        N.check(N.load().ppll_linear_wgrad(M, K, Nn, a.dev.data_ptr(), K, g.data_ptr(), Nn,
                                           dB.data_ptr(), None, dtype_code(g), _stream(g)),
                "matmul adjoint dB")
        return dB.to(b.dev.dtype)

    return _record_op(Tensor(out), [(a, pull_a), (b, pull_b)])


def _finite(t: torch.Tensor, op: str) -> None:
    """_ensure_finite (tensor.py:41-43) on a device result."""
    err = torch.zeros(1, dtype=torch.int32, device=t.device)
    N.check(N.load().ppll_ew(3, t.numel(), 1, t.data_ptr(), None, 1.0, t.data_ptr(),
                             dtype_code(t), err.data_ptr(), _stream(t)), "finite check")
    if int(err.item()):
        raise NonFiniteError(f"{op} produced non-finite values")


def relu(x: Tensor) -> Tensor:
    """max(x, 0); adjoint g·[x > 0], subgradient 0 at 0 (tensor.py:153-157)."""
    out = _ew(0, x.dev, None, check="relu")
    return _record_op(Tensor(out), [(x, lambda g, x=x: _ew(1, g, x.dev.to(g.dtype)))])


def add(a: Tensor, b: Tensor) -> Tensor:
    """Elementwise a + b (tensor.py:160-167)."""
    if a.shape != b.shape:
        raise DimensionMismatch(f"add shapes differ: {a.shape} vs {b.shape}")
    out = _ew(3, a.dev, b.dev.to(a.dev.dtype), check="add")
    return _record_op(Tensor(out), [(a, lambda g: g), (b, lambda g: g)])


def bias_add(m: Tensor, v: Tensor) -> Tensor:
    """Row-broadcast m + v; adjoints g and g.sum(axis=0) (tensor.py:170-180)."""
    if m.dev.dim() != 2 or v.dev.dim() != 1 or v.shape[0] != m.shape[1]:
        raise DimensionMismatch(f"bias_add shapes: {m.shape} + {v.shape}")
    out = _ew(2, m.dev, v.dev.to(m.dev.dtype), check="bias_add")

    def pull_v(g, v=v):
        db = torch.empty((g.shape[1],), dtype=torch.float32, device=g.device)
        N.check(N.load().ppll_colsum(g.shape[0], g.shape[1], g.data_ptr(), db.data_ptr(),
                                     dtype_code(g), _stream(g)), "bias_add adjoint")
        return db.to(v.dev.dtype)

    return _record_op(Tensor(out), [(m, lambda g: g), (v, pull_v)])


def scale(x: Tensor, c: float) -> Tensor:
    """x · c for a finite scalar c (tensor.py:183-191)."""
    c = float(c)
    if not np.isfinite(c):
        raise NonFiniteError("scale factor is non-finite")
    out = _ew(3, x.dev, None, alpha=c, check="scale")
    return _record_op(Tensor(out), [(x, lambda g, c=c: _ew(3, g, None, alpha=c))])


def sum_all(x: Tensor) -> Tensor:
    """Sum of every element as a scalar (tensor.py:194-198)."""
    require_cuda(x.dev, "sum_all")
    out = torch.empty((), dtype=torch.float32, device=x.dev.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.dev.device)
    N.check(N.load().ppll_sum_all(x.dev.numel(), x.dev.data_ptr(), out.data_ptr(),
                                  dtype_code(x.dev), err.data_ptr(), _stream(x.dev)), "sum_all")
    if int(err.item()):
        raise NonFiniteError("sum_all produced non-finite values")
    shape = x.dev.shape
    dt = x.dev.dtype

    def pull(g, shape=shape, dt=dt):
        src = g.reshape(1).to(dt)
        o = torch.empty(shape, dtype=dt, device=g.device)
        n = o.numel()
        N.check(N.load().ppll_ew(4, n, 1, src.data_ptr(), None, 1.0, o.data_ptr(),
                                 dtype_code(o), None, _stream(o)), "sum_all adjoint")
        return o

    return _record_op(Tensor(out), [(x, pull)])


def backward(loss: Tensor) -> None:
    """Replay the tape that produced ``loss`` with seed 1 (tensor.py:239-250)."""
    if loss.size != 1:
        raise NotScalar(f"backward needs a scalar loss, got shape {loss.shape}")
    _replay(loss, torch.ones_like(loss.dev))


def backward_from(output: Tensor, out_grad) -> None:
    """Replay seeding ``output`` with an external gradient (tensor.py:253-265)."""
    g = out_grad.dev if isinstance(out_grad, Tensor) else torch.as_tensor(
        np.asarray(out_grad, dtype=np.float64) if not torch.is_tensor(out_grad) else out_grad)
    if tuple(g.shape) != output.shape:
        raise DimensionMismatch(
            f"seed gradient shape {tuple(g.shape)} does not match output {output.shape}")
    g = g.to(device=output.dev.device, dtype=output.dev.dtype)
    _finite(g, "backward_from seed")
    _replay(output, g)


def _replay(seed_t: Tensor, seed_g: torch.Tensor) -> None:
    """tensor.py:268-278: reverse node order, adjoints accumulate."""
    tape = seed_t._tape
    if tape is None or tape.consumed or not tape.nodes:
        raise EmptyTape("no recorded operations to replay")
    _accumulate(seed_t, seed_g)
    for node in reversed(tape.nodes):
        out_grad = node.out.grad
        if out_grad is None:
            continue
        for t, fn in node.pulls:
            _accumulate(t, fn(out_grad.dev))
        tape.adjoints_run += 1
    tape.consumed = True
    tape.nodes.clear()


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
    # adjoint (softmax - onehot) · g / B: the kernel already wrote dz for g = 1
    return _record_op(out, [(logits, lambda g, dz=dz: _ew(3, dz, None, alpha=float(g.item())))])
