"""Network blocks, stage partitioning and per-stage auxiliary heads
(mirrors locopipe blocks.py:1-317), with device-resident parameters.

Each ``LocalModule`` owns ONE flat fp32 parameter buffer (θ), one momentum
buffer (v), one gradient buffer (g) and — in ``bf16`` precision — one bf16
shadow of θ used as the tensor-core operand.  Layer tensors ``W`` (stored
[in, out] like blocks.py:193) and ``b`` are views into θ at 256-byte aligned
offsets.  A local step (blocks.py:266-289) is one call into the native
executor (``ppll_stage_step``): fused forward → push → aux → softmax-CE →
backward → cosine-LR Nesterov, no host sync inside.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import (ConfigMismatch, DimensionMismatch, LabelOutOfRange, NonFiniteError,
                     StepOutOfRange, TooManyStages, WorkerPanic)
from .optim import LrSchedule, OptimizerState, lr_table
from .tensor import Tensor, as_labels, default_device, require_cuda

_ALIGN = 64  # elements (256 B of fp32): TMA / float4 alignment of every param view


@dataclass(frozen=True)
class NetworkSpec:
    """Layer widths of a fully-connected classifier (blocks.py:24-55)."""

    layer_dims: tuple
    activation: str = "relu"

    def __post_init__(self):
        object.__setattr__(self, "layer_dims", tuple(int(d) for d in self.layer_dims))
        if len(self.layer_dims) < 2:
            raise ValueError("need at least two layer dims (input and output)")
        if any(d < 1 for d in self.layer_dims):
            raise ValueError(f"layer dims must be positive, got {self.layer_dims}")
        if self.activation != "relu":
            raise ValueError(f"unsupported activation {self.activation!r}")

    @property
    def n_layers(self) -> int:
        return len(self.layer_dims) - 1

    @property
    def num_classes(self) -> int:
        return self.layer_dims[-1]

    def layer_params(self, i: int) -> int:
        return self.layer_dims[i] * self.layer_dims[i + 1] + self.layer_dims[i + 1]


@dataclass(frozen=True)
class PartitionPlan:
    """Contiguous, disjoint, covering assignment of layers to stages (blocks.py:58-72)."""

    n_stages: int
    boundaries: tuple

    def __post_init__(self):
        if self.n_stages != len(self.boundaries):
            raise ConfigMismatch("stage count does not match boundary list")
        prev_end = 0
        for start, end in self.boundaries:
            if start != prev_end or end <= start:
                raise ConfigMismatch(f"boundaries not contiguous/non-empty: {self.boundaries}")
            prev_end = end


def partition(spec: NetworkSpec, s: int) -> PartitionPlan:
    """Minimax contiguous split of layer parameter counts with the
    earliest-cut tie-break (blocks.py:75-96)."""
    n = spec.n_layers
    if s < 1:
        raise ValueError(f"need at least one stage, got {s}")
    if s > n:
        raise TooManyStages(f"{s} stages requested but only {n} layers")
    costs = [spec.layer_params(i) for i in range(n)]
    prefix = [0]
    for c in costs:
        prefix.append(prefix[-1] + c)
    best_cuts, best_load = None, math.inf
    for cuts in itertools.combinations(range(1, n), s - 1):
        edges = (0,) + cuts + (n,)
        load = max(prefix[b] - prefix[a] for a, b in zip(edges, edges[1:]))
        if load < best_load:
            best_load, best_cuts = load, cuts
    edges = (0,) + best_cuts + (n,)
    return PartitionPlan(s, tuple(zip(edges, edges[1:])))


def aux_depth(l: int, d_prime: int, n: int) -> int:
    """d' - floor(l / n), at least 0 (blocks.py:99-106)."""
    if l < 0 or d_prime < 0 or n < 1:
        raise ValueError(f"bad aux_depth arguments ({l}, {d_prime}, {n})")
    return max(0, d_prime - l // n)


@dataclass
class LinearLayer:
    """One dense layer (blocks.py:109-119); W, b are views into the stage's θ."""

    W: Tensor
    b: Tensor
    relu_after: bool

    @property
    def out_width(self) -> int:
        return self.W.shape[1]


@dataclass
class AuxHead:
    """``depth`` hidden ReLU layers then a linear readout (blocks.py:122-131)."""

    depth: int
    hidden_width: int
    layers: list

    def parameters(self) -> list:
        return [t for layer in self.layers for t in (layer.W, layer.b)]


@dataclass(frozen=True)
class Hyperparams:
    """Training settings shared by every stage (blocks.py:134-144), plus the
    device-side ``precision`` ("fp32" parity mode or "bf16" tensor-core mode)."""

    lr0: float = 0.01
    lr_min: float = 0.0
    total_steps: int = 1
    momentum: float = 0.9
    weight_decay: float = 1e-4
    seed: int = 42
    aux_hidden_width: int | None = None
    precision: str = "fp32"
    # the local optimizer: "nesterov" (the reference's, optim.py:71-89) or
    # "adamw" (north_star's "local SGD/Adam update"; torch.optim.AdamW rule,
    # ``weight_decay`` decoupled, ``momentum`` unused)
    optimizer: str = "nesterov"
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-8

    def __post_init__(self):
        if self.precision not in ("fp32", "bf16"):
            raise ValueError(f"precision must be 'fp32' or 'bf16', got {self.precision!r}")
        if self.optimizer not in ("nesterov", "adamw"):
            raise ValueError(f"optimizer must be 'nesterov' or 'adamw', got {self.optimizer!r}")


def attach_local_optimizer(flat: dict, hyper: "Hyperparams") -> None:
    """Register the stage's update rule with the library (keyed by its flat θ
    buffer; ppll_set_local_optimizer).  AdamW needs a second-moment buffer
    (``flat["mom2"]``; the first moment is ``flat["mom"]``).  The registration
    is dropped when θ is freed, before its memory can be reused."""
    if hyper.optimizer != "adamw":
        return
    import weakref
    theta = flat["theta"]
    flat["mom2"] = torch.zeros_like(theta)
    lib = N.load()
    b1, b2 = (float(b) for b in hyper.betas)
    N.check(lib.ppll_set_local_optimizer(theta.data_ptr(), 1, flat["mom2"].data_ptr(), b1, b2,
                                         float(hyper.eps)), "set_local_optimizer")
    weakref.finalize(theta, lib.ppll_set_local_optimizer, theta.data_ptr(), 0, None, 0.0, 0.0, 0.0)


class LocalModule:
    """One gradient-isolated pipeline stage: block layers + optional aux head
    (blocks.py:147-187), resident on one CUDA device."""

    # keep programmatic dependent launch when several stage streams share a
    # GPU (measured: the many short MLP / ResNet kernels gain from it; the
    # ViT step's long GEMMs lose 1.4 % — VitLocalModule turns it off)
    shared_gpu_pdl = True

    def __init__(self, stage_index, layers, aux, optimizer, schedule, assigned_aux_depth,
                 *, flat=None, device=None, precision="fp32"):
        if not layers:
            raise ConfigMismatch("a stage needs at least one layer")
        self.stage_index = stage_index
        self.layers = layers
        self.aux = aux
        self.optimizer = optimizer
        self.schedule = schedule
        self.assigned_aux_depth = assigned_aux_depth
        self.device = device
        self.precision = precision
        self._flat = flat            # dict of device buffers (see build_modules)
        self._native = None
        self._native_batch = 0

    @property
    def input_width(self) -> int:
        return self.layers[0].W.shape[0]

    @property
    def output_width(self) -> int:
        return self.layers[-1].out_width

    @property
    def num_classes(self) -> int:
        return (self.aux.layers[-1] if self.aux is not None else self.layers[-1]).out_width

    def block_parameters(self) -> list:
        return [t for layer in self.layers for t in (layer.W, layer.b)]

    def parameters(self) -> list:
        params = self.block_parameters()
        if self.aux is not None:
            params += self.aux.parameters()
        return params

    def all_layers(self) -> list:
        return list(self.layers) + (list(self.aux.layers) if self.aux is not None else [])

    @property
    def act_dtype(self) -> torch.dtype:
        return torch.bfloat16 if self.precision == "bf16" else torch.float32

    # -- native executor ----------------------------------------------------
    def native(self, batch: int):
        """The ``ppll_stage`` handle sized for at least ``batch`` rows."""
        if self._flat is None:
            raise ConfigMismatch("module was not built by build_modules (no device buffers)")
        if self._native is not None and batch <= self._native_batch:
            return self._native
        self.close()
        f = self._flat
        layers = self.all_layers()
        L = len(layers)
        arr = lambda vals, ct: (ct * len(vals))(*vals)  # noqa: E731
        import ctypes as C
        in_w = arr([l.W.shape[0] for l in layers], C.c_int)
        out_w = arr([l.W.shape[1] for l in layers], C.c_int)
        relu = arr([int(l.relu_after) for l in layers], C.c_int)
        offs = arr(f["offsets"], C.c_int64)
        cap = max(batch, 1)
        lib = N.load()
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            free0 = torch.cuda.mem_get_info()[0]
            h = lib.ppll_stage_create(
                L, len(self.layers), in_w, out_w, relu, offs, f["theta"].numel(), cap,
                N.BF16 if self.precision == "bf16" else N.F32, f["theta"].data_ptr(),
                f["grad"].data_ptr(), f["mom"].data_ptr(),
                N.ptr(f["theta_lp"]), f["lr"].data_ptr(), f["state"].data_ptr(),
                self.schedule.total_steps, f["loss"].data_ptr(), f["state"][2:].data_ptr(),
                float(self.optimizer.mu), float(self.optimizer.weight_decay))
        if not h:
            raise N.NativeError("ppll_stage_create failed: " +
                                lib.ppll_last_error().decode(errors="replace"))
        self._native_bytes = max(0, free0 - torch.cuda.mem_get_info(self.device)[0])
        self._native, self._native_batch = h, cap
        return h

    def close(self) -> None:
        if self._native is not None:
            N.load().ppll_stage_destroy(self._native)
            self._native = None
            self._native_batch = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- generic stage interface used by the runtime ------------------------
    @property
    def in_shape(self) -> tuple:
        return (self.input_width,)

    @property
    def out_shape(self) -> tuple:
        return (self.output_width,)

    @property
    def in_features(self) -> int:
        return int(np.prod(self.in_shape))

    @property
    def out_features(self) -> int:
        return int(np.prod(self.out_shape))

    def launch_step(self, B, x_ptr, y_ptr, out_ptr, stream) -> None:
        """Enqueue one local step (``ppll_stage_step``) on ``stream``."""
        N.check(N.load().ppll_stage_step(self.native(B), B, x_ptr, y_ptr, out_ptr, stream),
                f"stage {self.stage_index} step")

    def launch_forward(self, B, x_ptr, h_ptr, logits_ptr, stream) -> None:
        N.check(N.load().ppll_stage_forward(self.native(B), B, x_ptr, h_ptr, logits_ptr, stream),
                f"stage {self.stage_index} forward")

    # -- the E2E / naive-PP baselines (runtime.py:248-284, 359-382) ---------
    supports_e2e = True

    def launch_block_forward(self, B, x_ptr, h_ptr, stream) -> None:
        N.check(N.load().ppll_stage_block_forward(self.native(B), B, x_ptr, h_ptr, stream),
                f"stage {self.stage_index} block forward")

    def launch_block_backward(self, B, x_ptr, gout_ptr, y_ptr, gin_ptr, stream) -> None:
        N.check(N.load().ppll_stage_block_backward(self.native(B), B, x_ptr, gout_ptr, y_ptr,
                                                   gin_ptr, stream),
                f"stage {self.stage_index} block backward")

    def error_word(self) -> int:
        """Sticky device error bits (synchronises this module's device)."""
        return int(self._flat["state"][2].item())

    def clear_error(self) -> None:
        self._flat["state"][2].zero_()

    def device_step(self) -> int:
        return int(self._flat["state"][0].item())

    def loss_history(self, start: int, count: int) -> list:
        """Device losses of steps [start, start+count) as Python floats."""
        return [float(v) for v in self._flat["loss"][start:start + count].double().cpu()]

    def raise_for_error(self, stage=None) -> None:
        e = self.error_word()
        if not e:
            return
        self.clear_error()
        if e & N.ERRBIT_LABEL:
            exc = LabelOutOfRange("labels must lie in [0, num_classes)")
        elif e & (N.ERRBIT_LOSS | N.ERRBIT_PARAM | N.ERRBIT_GRAD):
            exc = NonFiniteError("local step produced non-finite values")
        elif e & N.ERRBIT_SYNC:
            exc = TimeoutError("a device grid barrier timed out (stage results invalid)")
        else:
            exc = StepOutOfRange(f"step outside [0, {self.schedule.total_steps}]")
        if stage is None:
            raise exc
        raise WorkerPanic(stage, repr(exc)) from exc

    def __repr__(self) -> str:
        depth = "none" if self.aux is None else self.aux.depth
        return (f"LocalModule(stage={self.stage_index}, layers={len(self.layers)}, "
                f"aux_depth={depth}, precision={self.precision}, device={self.device})")


def _init_layer_host(rng, fan_in, fan_out):
    """blocks.py:190-195 — W ~ U(±1/√fan_in) drawn before b (PCG64, fp64)."""
    bound = 1.0 / math.sqrt(fan_in)
    W = rng.uniform(-bound, bound, size=(fan_in, fan_out))
    b = rng.uniform(-bound, bound, size=(fan_out,))
    return W, b


def build_modules(spec: NetworkSpec, plan: PartitionPlan, d_prime: int, n: int,
                  hyper: Hyperparams, devices: Sequence | None = None,
                  only: Sequence[int] | None = None) -> list:
    """One LocalModule per stage of ``plan`` (blocks.py:198-237).

    Initial values are drawn on the host with the reference's generator and
    draw order (``default_rng(seed + j)``, block layers then aux layers, W
    before b) and uploaded once; ``devices[j]`` places stage j (default: the
    current CUDA device for every stage).  ``only`` builds just those stage
    indices (one process per GPU: each rank builds its own stages; a stage's
    init does not depend on the others, blocks.py:202-204).
    """
    if plan.boundaries[-1][1] != spec.n_layers:
        raise ConfigMismatch("partition plan does not cover the network")
    dims = spec.layer_dims
    classes = spec.num_classes
    last_stage = plan.n_stages - 1
    modules = []
    for j, (start, end) in enumerate(plan.boundaries):
        if only is not None and j not in only:
            continue
        device = torch.device(devices[j]) if devices is not None else default_device()
        if isinstance(device, torch.device) and device.type == "cuda" and device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        rng = np.random.default_rng(hyper.seed + j)
        host = []   # (W, b, relu_after)
        for i in range(start, end):
            W, b = _init_layer_host(rng, dims[i], dims[i + 1])
            host.append((W, b, i != spec.n_layers - 1))
        assigned = aux_depth(j, d_prime, n)
        n_block = len(host)
        hidden = None
        if j != last_stage:
            block_out = dims[end]
            hidden = hyper.aux_hidden_width or block_out
            widths = [block_out] + [hidden] * assigned + [classes]
            for i in range(len(widths) - 1):
                W, b = _init_layer_host(rng, widths[i], widths[i + 1])
                host.append((W, b, i != len(widths) - 2))
        modules.append(_materialise(j, host, n_block, assigned, hidden, hyper, device))
    return modules


def _materialise(j, host, n_block, assigned, hidden, hyper, device):
    offsets, cur = [], 0
    for W, b, _ in host:
        for a in (W, b):
            offsets.append(cur)
            cur += (a.size + _ALIGN - 1) // _ALIGN * _ALIGN
    total = max(cur, _ALIGN)
    flat_host = np.zeros(total, dtype=np.float64)
    k = 0
    for W, b, _ in host:
        for a in (W, b):
            flat_host[offsets[k]:offsets[k] + a.size] = a.ravel()
            k += 1
    theta = torch.from_numpy(flat_host).to(device=device, dtype=torch.float32)
    mom = torch.zeros_like(theta)
    grad = torch.zeros_like(theta)
    theta_lp = theta.to(torch.bfloat16) if hyper.precision == "bf16" else None
    sched = LrSchedule(hyper.lr0, hyper.lr_min, hyper.total_steps)
    flat = {
        "theta": theta, "mom": mom, "grad": grad, "theta_lp": theta_lp,
        "offsets": offsets,
        "lr": lr_table(sched, device),
        # [step_count, nesterov block-completion scratch, error word, pad]
        "state": torch.zeros(4, dtype=torch.int32, device=device),
        "loss": torch.zeros(hyper.total_steps + 2, dtype=torch.float32, device=device),
    }
    attach_local_optimizer(flat, hyper)
    layers, params, moms = [], [], []
    k = 0
    for W, b, relu_after in host:
        wv = theta[offsets[k]:offsets[k] + W.size].view(W.shape)
        bv = theta[offsets[k + 1]:offsets[k + 1] + b.size]
        tw, tb = Tensor(wv, track_grad=True), Tensor(bv, track_grad=True)
        moms += [mom[offsets[k]:offsets[k] + W.size].view(W.shape),
                 mom[offsets[k + 1]:offsets[k + 1] + b.size]]
        layers.append(LinearLayer(tw, tb, relu_after))
        params += [tw, tb]
        k += 2
    block, aux_layers = layers[:n_block], layers[n_block:]
    aux = AuxHead(assigned, hidden, aux_layers) if aux_layers else None
    opt = OptimizerState(params, hyper.momentum, hyper.weight_decay,
                         _flat=(theta, mom, grad, moms))
    return LocalModule(j, block, aux, opt, sched, assigned, flat=flat, device=device,
                       precision=hyper.precision)


# --------------------------------------------------------------------------
# forward-only entry points (blocks.py:249-263)
# --------------------------------------------------------------------------

def _as_input(module: LocalModule, x: Tensor) -> torch.Tensor:
    """[B, *in_shape] (or [B, in_features]) device tensor in the stage dtype,
    flattened to [B, in_features]."""
    t = x.dev
    ok = t.dim() >= 2 and (tuple(t.shape[1:]) == tuple(module.in_shape) or
                           (t.dim() == 2 and t.shape[1] == module.in_features))
    if not ok:
        raise DimensionMismatch(
            f"stage {module.stage_index} expects width {module.in_shape}, got {x.shape}")
    require_cuda(t, f"stage {module.stage_index}")
    if t.device != module.device or t.dtype != module.act_dtype:
        t = t.to(device=module.device, dtype=module.act_dtype)
    return t.reshape(t.shape[0], module.in_features).contiguous()


def _forward(module: LocalModule, x: Tensor, want_logits: bool):
    xin = _as_input(module, x)
    B = xin.shape[0]
    h = torch.empty((B,) + tuple(module.out_shape), dtype=module.act_dtype, device=module.device)
    logits = None
    if want_logits:
        logits = torch.empty((B, module.num_classes), dtype=module.act_dtype, device=module.device)
    if B:
        st = torch.cuda.current_stream(module.device).cuda_stream
        module.launch_forward(B, xin.data_ptr(), h.data_ptr(), N.ptr(logits), st)
    return h, logits


def block_forward(module: LocalModule, x: Tensor) -> Tensor:
    """Run the stage's block layers (blocks.py:249-255); forward only."""
    h, _ = _forward(module, x, False)
    return Tensor(h)


def aux_forward(module: LocalModule, h: Tensor) -> Tensor:
    """Local logits (blocks.py:258-263): the aux head, or ``h`` itself for the
    final stage.  ``h`` must be this module's block output."""
    if module.aux is None:
        return h
    t = h.dev
    if t.dim() != 2 or t.shape[1] != module.output_width:
        raise DimensionMismatch(f"aux head expects width {module.output_width}, got {h.shape}")
    x = t.to(module.act_dtype)
    for layer in module.aux.layers:
        out = torch.empty((x.shape[0], layer.out_width), dtype=module.act_dtype,
                          device=module.device)
        W = (module._flat["theta_lp"] if module.precision == "bf16" else module._flat["theta"])
        off = _param_offset(module, layer.W)
        st = torch.cuda.current_stream(module.device).cuda_stream
        code = N.BF16 if module.precision == "bf16" else N.F32
        N.check(N.load().ppll_linear_fwd(x.shape[0], layer.W.shape[0], layer.out_width,
                                         x.data_ptr(), layer.W.shape[0],
                                         W[off:].data_ptr(), layer.b.dev.data_ptr(),
                                         out.data_ptr(), layer.out_width, None, 0,
                                         int(layer.relu_after), code, st), "aux forward")
        x = out
    return Tensor(x)


def _param_offset(module, tensor) -> int:
    base = module._flat["theta"].data_ptr()
    return (tensor.dev.data_ptr() - base) // 4


def local_loss_and_update(module: LocalModule, x_in: Tensor, labels,
                          on_output: Callable | None = None) -> tuple:
    """One local training step (blocks.py:266-289): forward, push hook,
    local loss, backward, cosine-LR Nesterov update — one native call.

    ``x_in`` must be detached.  The returned ``x_out`` (also handed to
    ``on_output``) is written by the block's last forward epilogue, so it
    reflects the PRE-step parameters.  Returns ``(float loss, x_out)``; the
    float read synchronises the stream (the pipeline runtime does not).
    """
    if x_in.track_grad:
        raise ValueError("stage input must be detached")
    xin = _as_input(module, x_in)
    B = xin.shape[0]
    y = as_labels(labels, B, module.num_classes, module.device, check_range=False)
    if B < 1:
        raise DimensionMismatch("softmax_xent needs a non-empty batch")
    step = module.optimizer.step_count
    x_out = torch.empty((B,) + tuple(module.out_shape), dtype=module.act_dtype,
                        device=module.device)
    st = torch.cuda.current_stream(module.device).cuda_stream
    if step > module.schedule.total_steps:
        # reference order: forward + push happen, then cosine_lr raises (blocks.py:280-287)
        module.launch_forward(B, xin.data_ptr(), x_out.data_ptr(), None, st)
        out = Tensor(x_out)
        if on_output is not None:
            on_output(out)
        raise StepOutOfRange(f"step {step} outside [0, {module.schedule.total_steps}]")
    module.launch_step(B, xin.data_ptr(), y.data_ptr(), x_out.data_ptr(), st)
    out = Tensor(x_out)
    if on_output is not None:
        on_output(out)
    module.raise_for_error()
    module.optimizer.step_count += 1
    loss = float(module._flat["loss"][step].item())
    return loss, out


# --------------------------------------------------------------------------
# memory accounting (blocks.py:292-317) + measured device bytes
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class MemoryProxy:
    """Float counts standing in for device memory (blocks.py:292-302)."""

    params: int
    activations: int

    @property
    def total(self) -> int:
        return self.params + self.activations


def memory_footprint(module: LocalModule, batch_size: int) -> MemoryProxy:
    """Analytic per-stage memory proxy in float counts (blocks.py:305-317)."""
    if batch_size < 1:
        raise ValueError(f"batch_size must be >= 1, got {batch_size}")
    params = sum(p.size for p in module.parameters())
    widths = [module.input_width] + [layer.out_width for layer in module.layers]
    if module.aux is not None:
        widths += [layer.out_width for layer in module.aux.layers]
    return MemoryProxy(int(params), int(batch_size * sum(widths)))
