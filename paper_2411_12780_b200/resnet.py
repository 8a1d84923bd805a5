"""ResNet local-learning stages (north-star model family; no reference
implementation exists — SURVEY §0.2).

CIFAR ResNet (He et al.): stem conv3x3 + BN + ReLU, three groups of ``n``
basic blocks (16/32/64 channels; option-B 1x1-conv shortcut on
downsampling), global average pool + linear.  ``n=5`` is ResNet-32, ``n=18``
ResNet-110.  The units [stem, block_0, ...] are split contiguously into
gradient-isolated stages; each non-final stage gets an auxiliary head of
N_l = aux_depth(l, d', n) conv3x3-BN-ReLU layers + GAP + linear (the paper's
ResNet used MAN heads; this builder choice is documented in
DESIGN.md).  The local step keeps the reference's semantics
(blocks.py:266-289) and runs as ONE native call (``ppll_resnet_stage_step``);
the CPU restatement it is checked against is ``oracle/resnet_oracle.py``.
Activations are NHWC; stage 0 takes images [B, H, W, C].
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from .blocks import Hyperparams, LocalModule, attach_local_optimizer, aux_depth
from .errors import ConfigMismatch
from .optim import LrSchedule, OptimizerState, lr_table
from .tensor import Tensor, default_device

_ALIGN = 64


@dataclass(frozen=True)
class ResNetSpec:
    n: int = 5
    image: int = 32
    channels: int = 3
    widths: tuple = (16, 32, 64)
    classes: int = 10

    @property
    def n_blocks(self) -> int:
        return 3 * self.n


def block_geometry(spec: ResNetSpec, b: int):
    g = b // spec.n
    cout = spec.widths[g]
    first = b % spec.n == 0
    cin = spec.widths[g - 1] if (first and g > 0) else cout
    stride = 2 if (first and g > 0) else 1
    h_in = spec.image // (2 ** g) * (2 if stride == 2 else 1)
    return cin, cout, stride, h_in


def resnet_split(spec: ResNetSpec, s: int) -> list:
    """Even contiguous split of the units [stem, blocks...] (earlier stages
    take the remainder, like partition()'s earliest-cut tie-break)."""
    units = spec.n_blocks + 1
    if s < 1 or s > units:
        raise ConfigMismatch(f"cannot split {units} units into {s} stages")
    q, r = divmod(units, s)
    out, u = [], 0
    for j in range(s):
        sz = q + (1 if j < r else 0)
        out.append([x - 1 for x in range(u, u + sz) if x >= 1])
        u += sz
    return out


def _unit_cost(hwc: float) -> float:
    """Relative cost of a basic block whose output map has ``hwc`` elements
    per image: a fixed per-layer launch/latency part plus a part proportional
    to the activation bytes its memory-bound kernels (im2col, BN, col2im)
    move; constants fit to the measured stage cycles of the even ResNet-32
    split on B200 (0.15 ms per 8x8x64 block, 0.32 ms per 32x32x16 block)."""
    return 0.093 + 1.38e-5 * hwc


def balanced_resnet_split(spec: ResNetSpec, s: int, d_prime: int, n: int) -> list:
    """Contiguous split of the units [stem, blocks...] minimising the most
    expensive stage (minimax DP), each stage charged for its blocks, its aux
    head (aux_depth(j, d', n) convs at its output map, none on the final
    stage) and the stem on stage 0.  The even split gives the early,
    high-resolution stages 2.5x the cycle of the last one; this balances the
    one-stage-per-GPU pipeline (the cost model's idle prediction)."""
    units = spec.n_blocks + 1
    if s < 1 or s > units:
        raise ConfigMismatch(f"cannot split {units} units into {s} stages")
    ucost = [0.5 * _unit_cost(spec.image * spec.image * spec.widths[0])]
    geo = []
    for b in range(spec.n_blocks):
        cin, cout, stride, h_in = block_geometry(spec, b)
        h = h_in // stride
        ucost.append(_unit_cost(h * h * cout) + (0.03 if stride != 1 or cin != cout else 0.0))
        geo.append(h * h * cout)
    out_hwc = [spec.image * spec.image * spec.widths[0]] + geo

    def stage_cost(j, a, b_):          # units a..b_-1 on stage j
        c = sum(ucost[a:b_])
        if j < s - 1:
            c += aux_depth(j, d_prime, n) * 0.5 * _unit_cost(out_hwc[b_ - 1])
        return c

    INF = float("inf")
    best = [[INF] * (units + 1) for _ in range(s + 1)]
    cut = [[0] * (units + 1) for _ in range(s + 1)]
    best[0][0] = 0.0
    for j in range(1, s + 1):
        for i in range(j, units - (s - j) + 1):
            for k in range(j - 1, i):
                v = max(best[j - 1][k], stage_cost(j - 1, k, i))
                if v < best[j][i] - 1e-12:
                    best[j][i], cut[j][i] = v, k
    bounds, i = [], units
    for j in range(s, 0, -1):
        k = cut[j][i]
        bounds.append((k, i))
        i = k
    bounds.reverse()
    return [[x - 1 for x in range(a, b_) if x >= 1] for a, b_ in bounds]


def stage_out_geometry(spec: ResNetSpec, blocks):
    if not blocks:
        return spec.widths[0], spec.image
    cin, cout, stride, h_in = block_geometry(spec, blocks[-1])
    return cout, h_in // stride


def _kp(k, cin):
    return (k * k * cin + 7) // 8 * 8


def _conv_w(rng, k, cin, cout):
    bound = 1.0 / math.sqrt(k * k * cin)
    return rng.uniform(-bound, bound, size=(k * k * cin, cout))


class ResLocalModule(LocalModule):
    """One ResNet stage: [stem] + basic blocks + aux convs + head."""

    def __init__(self, stage_index, spec, blocks, groups, n_aux, optimizer, schedule,
                 assigned_aux_depth, *, flat, device, precision, final, in_geo, out_geo):
        self.spec = spec
        self.block_ids = blocks
        self.groups = groups
        self.n_aux_convs = n_aux
        self.has_stem = stage_index == 0
        self.in_geo, self.out_geo = in_geo, out_geo   # (C, H)
        super().__init__(stage_index, list(groups), None, optimizer, schedule,
                         assigned_aux_depth, flat=flat, device=device, precision=precision)
        self.final = final

    @property
    def in_shape(self) -> tuple:
        c, h = self.in_geo
        return (h, h, c)

    @property
    def out_shape(self) -> tuple:
        c, h = self.out_geo
        return (h, h, c)

    @property
    def input_width(self) -> int:
        return self.in_features

    @property
    def output_width(self) -> int:
        return self.out_features

    @property
    def num_classes(self) -> int:
        return self.spec.classes

    def parameters(self) -> list:
        return [t for _, _, t in self.groups]

    def block_parameters(self) -> list:
        return [t for g, _, t in self.groups if g == "stem" or g.startswith("block")]

    def all_layers(self) -> list:
        return []

    def native(self, batch: int):
        if self._native is not None and batch <= self._native_batch:
            return self._native
        self.close()
        f, sp = self._flat, self.spec
        geo = []
        for b in self.block_ids:
            geo += list(block_geometry(sp, b))
        cfg = (C.c_int * 8)(batch, sp.channels, sp.image, sp.classes, int(self.has_stem),
                            len(self.block_ids), self.n_aux_convs, sp.widths[0])
        geo_a = (C.c_int * max(1, len(geo)))(*geo) if geo else (C.c_int * 1)(0)
        og = (C.c_int * 2)(*self.out_geo)
        offs = f["offsets"]
        arr = (C.c_int64 * len(offs))(*offs)
        lib = N.load()
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            free0 = torch.cuda.mem_get_info()[0]
            h = lib.ppll_resnet_stage_create(
                cfg, geo_a, og, arr, f["theta"].numel(), N.BF16 if self.precision == "bf16" else N.F32,
                f["theta"].data_ptr(), f["grad"].data_ptr(), f["mom"].data_ptr(),
                N.ptr(f["theta_lp"]), f["lr"].data_ptr(), f["state"].data_ptr(),
                self.schedule.total_steps, f["loss"].data_ptr(), f["state"][2:].data_ptr(),
                float(self.optimizer.mu), float(self.optimizer.weight_decay))
        if not h:
            raise N.NativeError("ppll_resnet_stage_create failed: " +
                                lib.ppll_last_error().decode(errors="replace"))
        self._native_bytes = max(0, free0 - torch.cuda.mem_get_info(self.device)[0])
        self._native, self._native_batch = h, batch
        return h

    def close(self) -> None:
        if self._native is not None:
            N.load().ppll_resnet_stage_destroy(self._native)
            self._native = None
            self._native_batch = 0

    def launch_step(self, B, x_ptr, y_ptr, out_ptr, stream) -> None:
        N.check(N.load().ppll_resnet_stage_step(self.native(B), B, x_ptr, y_ptr, out_ptr, stream),
                f"resnet stage {self.stage_index} step")

    def launch_forward(self, B, x_ptr, h_ptr, logits_ptr, stream) -> None:
        N.check(N.load().ppll_resnet_stage_forward(self.native(B), B, x_ptr, h_ptr, logits_ptr,
                                                   stream), f"resnet stage {self.stage_index} forward")

    # -- the E2E / naive-PP baselines (runtime.py:248-284, 359-382) ---------
    def launch_block_forward(self, B, x_ptr, h_ptr, stream) -> None:
        N.check(N.load().ppll_resnet_stage_block_forward(self.native(B), B, x_ptr, h_ptr, stream),
                f"resnet stage {self.stage_index} block forward")

    def launch_block_backward(self, B, x_ptr, gout_ptr, y_ptr, gin_ptr, stream) -> None:
        N.check(N.load().ppll_resnet_stage_block_backward(self.native(B), B, x_ptr, gout_ptr,
                                                          y_ptr, gin_ptr, stream),
                f"resnet stage {self.stage_index} block backward")

    def __repr__(self) -> str:
        return (f"ResLocalModule(stage={self.stage_index}, blocks={self.block_ids}, "
                f"aux_convs={self.n_aux_convs}, precision={self.precision})")


def build_resnet_modules(spec: ResNetSpec, s: int, d_prime: int, n: int, hyper: Hyperparams,
                         devices: Sequence | None = None,
                         only: Sequence[int] | None = None, split: str | list = "even") -> list:
    """One ResLocalModule per stage.  Init (blocks.py:198-237 style):
    ``default_rng(seed + j)``; conv W ~ U(±1/√fan_in) drawn in layer order
    (stem, per block w1, w2[, ws], aux convs), then the head W and b; BN gamma=1,
    beta=0 (no draws).  ``split``: "even" (resnet_split), "cost"
    (balanced_resnet_split) or an explicit list of block-index lists."""
    if split == "even":
        split = resnet_split(spec, s)
    elif split == "cost":
        split = balanced_resnet_split(spec, s, d_prime, n)
    elif len(split) != s:
        raise ConfigMismatch(f"split has {len(split)} stages, expected {s}")
    mods = []
    for j, blocks in enumerate(split):
        if only is not None and j not in only:
            continue
        device = torch.device(devices[j]) if devices is not None else default_device()
        if device.type == "cuda" and device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        rng = np.random.default_rng(hyper.seed + j)
        host = []        # (group, key, array, alloc_elems)
        ones = lambda c: np.ones(c)     # noqa: E731
        zeros = lambda c: np.zeros(c)   # noqa: E731
        if j == 0:
            c0 = spec.widths[0]
            host += [("stem", "w", _conv_w(rng, 3, spec.channels, c0), _kp(3, spec.channels) * c0),
                     ("stem", "bn_g", ones(c0), None), ("stem", "bn_b", zeros(c0), None)]
        for i, b in enumerate(blocks):
            cin, cout, stride, _ = block_geometry(spec, b)
            host += [(f"block{i}", "w1", _conv_w(rng, 3, cin, cout), _kp(3, cin) * cout),
                     (f"block{i}", "bn1_g", ones(cout), None), (f"block{i}", "bn1_b", zeros(cout), None),
                     (f"block{i}", "w2", _conv_w(rng, 3, cout, cout), _kp(3, cout) * cout),
                     (f"block{i}", "bn2_g", ones(cout), None), (f"block{i}", "bn2_b", zeros(cout), None)]
            if stride != 1 or cin != cout:
                host += [(f"block{i}", "ws", _conv_w(rng, 1, cin, cout), _kp(1, cin) * cout),
                         (f"block{i}", "bns_g", ones(cout), None),
                         (f"block{i}", "bns_b", zeros(cout), None)]
        c_out, h_out = stage_out_geometry(spec, blocks)
        final = j == len(split) - 1
        n_aux = 0 if final else aux_depth(j, d_prime, n)
        for i in range(n_aux):
            host += [(f"aux{i}", "w", _conv_w(rng, 3, c_out, c_out), _kp(3, c_out) * c_out),
                     (f"aux{i}", "bn_g", ones(c_out), None), (f"aux{i}", "bn_b", zeros(c_out), None)]
        bound = 1.0 / math.sqrt(c_out)
        host += [("head", "w", rng.uniform(-bound, bound, size=(c_out, spec.classes)), None),
                 ("head", "b", rng.uniform(-bound, bound, size=(spec.classes,)), None)]
        offsets, cur = [], 0
        for _, _, a, alloc in host:
            offsets.append(cur)
            n_el = max(a.size, alloc or 0)
            cur += (n_el + _ALIGN - 1) // _ALIGN * _ALIGN
        flat_host = np.zeros(max(cur, _ALIGN))
        for (_, _, a, _), o in zip(host, offsets):
            flat_host[o:o + a.size] = a.ravel()
        theta = torch.from_numpy(flat_host).to(device=device, dtype=torch.float32)
        mom, grad = torch.zeros_like(theta), torch.zeros_like(theta)
        theta_lp = theta.to(torch.bfloat16) if hyper.precision == "bf16" else None
        sched = LrSchedule(hyper.lr0, hyper.lr_min, hyper.total_steps)
        # native offsets: stem(3) + 9 per block + 3 per aux + head(2)
        byname = {(g, k): o for (g, k, _, _), o in zip(host, offsets)}
        nat = [byname.get(("stem", k), -1) for k in ("w", "bn_g", "bn_b")]
        for i in range(len(blocks)):
            nat += [byname.get((f"block{i}", k), -1)
                    for k in ("w1", "bn1_g", "bn1_b", "w2", "bn2_g", "bn2_b", "ws", "bns_g", "bns_b")]
        for i in range(n_aux):
            nat += [byname[(f"aux{i}", k)] for k in ("w", "bn_g", "bn_b")]
        nat += [byname[("head", "w")], byname[("head", "b")]]
        flat = {"theta": theta, "mom": mom, "grad": grad, "theta_lp": theta_lp, "offsets": nat,
                "lr": lr_table(sched, device),
                "state": torch.zeros(4, dtype=torch.int32, device=device),
                "loss": torch.zeros(hyper.total_steps + 2, dtype=torch.float32, device=device)}
        attach_local_optimizer(flat, hyper)
        groups, moms = [], []
        for (g, k, a, _), o in zip(host, offsets):
            view = theta[o:o + a.size].view(a.shape)
            groups.append((g, k, Tensor(view, track_grad=True)))
            moms.append(mom[o:o + a.size].view(a.shape))
        opt = OptimizerState([t for _, _, t in groups], hyper.momentum, hyper.weight_decay,
                             _flat=(theta, mom, grad, moms))
        in_geo = (spec.channels, spec.image) if j == 0 else stage_out_geometry(spec, split[j - 1])
        mods.append(ResLocalModule(j, spec, blocks, groups, n_aux, opt, sched, aux_depth(j, d_prime, n),
                                   flat=flat, device=device, precision=hyper.precision,
                                   final=final, in_geo=in_geo, out_geo=(c_out, h_out)))
    return mods
