"""ViT local-learning stages (north-star model family; no reference
implementation exists — SURVEY §0.2).

A ViT (pre-LN transformer, patch embedding, cls token) is split into
gradient-isolated blocks of transformer layers.  Each non-final block gets an
auxiliary head of N_l = aux_depth(l, d', n) transformer layers + LayerNorm +
classifier on the cls token (blocks.py:99-106); the final
block ends in the task head.  The local step keeps the reference's semantics
(blocks.py:266-289: push before backward, no gradient into the detached
input, cosine-LR L2-Nesterov on every parameter) and runs as ONE native call
(``ppll_vit_stage_step``); the CPU restatement it is checked against is
``oracle/vit_oracle.py``.

``VitLocalModule`` exposes the same surface as ``LocalModule`` (stage_index,
optimizer, schedule, parameters(), block_parameters(), assigned_aux_depth),
so ``local_loss_and_update``, ``run_epoch`` and ``run_deterministic`` drive it
unchanged.
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
LAYER_KEYS = ("ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1",
              "w2", "b2")


@dataclass(frozen=True)
class VitSpec:
    """ViT shape (defaults: ViT-S/4 on CIFAR-shaped 3x32x32)."""

    image: int = 32
    channels: int = 3
    patch: int = 4
    dim: int = 384
    heads: int = 6
    mlp: int = 1536
    depth: int = 8
    classes: int = 10

    def __post_init__(self):
        if self.image % self.patch:
            raise ValueError("image size must be a multiple of the patch size")
        if self.dim % self.heads or self.dim // self.heads != 64:
            raise ValueError("head_dim must be 64")
        if self.dim % 32:
            raise ValueError("dim must be a multiple of 32")

    @property
    def n_patches(self) -> int:
        return (self.image // self.patch) ** 2

    @property
    def tokens(self) -> int:
        return self.n_patches + 1

    @property
    def patch_dim(self) -> int:
        return self.channels * self.patch * self.patch


def _lin(rng, fi, fo):
    """blocks.py:190-195 — W ~ U(±1/√fan_in) before b."""
    bound = 1.0 / math.sqrt(fi)
    return rng.uniform(-bound, bound, size=(fi, fo)), rng.uniform(-bound, bound, size=(fo,))


def _init_layer(rng, spec):
    D, F = spec.dim, spec.mlp
    p = {"ln1_g": np.ones(D), "ln1_b": np.zeros(D)}
    p["wqkv"], p["bqkv"] = _lin(rng, D, 3 * D)
    p["wo"], p["bo"] = _lin(rng, D, D)
    p["ln2_g"], p["ln2_b"] = np.ones(D), np.zeros(D)
    p["w1"], p["b1"] = _lin(rng, D, F)
    p["w2"], p["b2"] = _lin(rng, F, D)
    return p


def balanced_depths(depth: int, s: int) -> list:
    """Contiguous split of ``depth`` layers into ``s`` blocks, earlier blocks
    taking the remainder (like partition()'s earliest-cut tie-break)."""
    if s < 1 or s > depth:
        raise ConfigMismatch(f"cannot split depth {depth} into {s} blocks")
    q, r = divmod(depth, s)
    return [q + (1 if j < r else 0) for j in range(s)]


def vit_layer_cost(spec: "VitSpec", first: bool = False) -> float:
    """Training FLOPs of one transformer layer per image (forward, input
    gradient, weight gradient).  ``first``: the block's first layer, whose
    detached input needs no QKV input gradient (blocks.py:277-278)."""
    T, D, F = spec.tokens, spec.dim, spec.mlp
    fwd = 2.0 * T * (4 * D * D + 2 * D * F) + 4.0 * T * T * D
    return 3.0 * fwd - (2.0 * T * D * 3 * D if first else 0.0)


def balanced_vit_depths(spec: "VitSpec", s: int, d_prime: int, n: int,
                        layer_cost: float | None = None, aux_cost: float | None = None,
                        embed_cost: float | None = None) -> list:
    """Contiguous split of the ``depth`` layers into ``s`` blocks minimising
    the most expensive STAGE, each stage charged for its block layers, its
    aux head (aux_depth(j, d', n) transformer layers, none on the final
    stage, blocks.py:99-106,218-229) and the patch embedding on stage 0.
    ``balanced_depths`` splits by depth only, which leaves the final stage
    (no aux head) idle for a third of every cycle at d'=1; this split is what
    the one-stage-per-GPU pipeline needs for an idle fraction under 10 %.

    Like ``partition`` (blocks.py:75-96) it enumerates the cut positions in
    ``itertools.combinations`` order and keeps the first strict minimum, so
    ties go to the earliest cuts.  Costs default to the analytic training
    FLOPs per image; pass measured ones (``calibrate``) to override."""
    import itertools
    if s < 1 or s > spec.depth:
        raise ConfigMismatch(f"cannot split depth {spec.depth} into {s} blocks")
    full = vit_layer_cost(spec) if layer_cost is None else layer_cost
    first_saving = (vit_layer_cost(spec) - vit_layer_cost(spec, first=True)) * full \
        / vit_layer_cost(spec)
    aux = full if aux_cost is None else aux_cost
    emb = (3.0 * 2.0 * spec.n_patches * spec.patch_dim * spec.dim
           if embed_cost is None else embed_cost)

    def stage_cost(j, n_layers):
        c = n_layers * full - first_saving + (emb if j == 0 else 0.0)
        if j < s - 1:
            c += aux_depth(j, d_prime, n) * aux
        return c

    L = spec.depth
    best, best_load = None, math.inf
    for cuts in itertools.combinations(range(1, L), s - 1):
        edges = (0,) + cuts + (L,)
        load = max(stage_cost(j, b - a) for j, (a, b) in enumerate(zip(edges, edges[1:])))
        if load < best_load * (1 - 1e-12):
            best, best_load = edges, load
    return [b - a for a, b in zip(best, best[1:])]


def vit_stage_costs(spec: "VitSpec", depths: Sequence[int], d_prime: int, n: int) -> list:
    """The analytic per-stage cost ``balanced_vit_depths`` minimises."""
    s = len(depths)
    full = vit_layer_cost(spec)
    out = []
    for j, dj in enumerate(depths):
        c = (dj - 1) * full + vit_layer_cost(spec, first=True)
        if j == 0:
            c += 3.0 * 2.0 * spec.n_patches * spec.patch_dim * spec.dim
        if j < s - 1:
            c += aux_depth(j, d_prime, n) * full
        out.append(c)
    return out


class VitLocalModule(LocalModule):
    """One ViT stage: [patch embed] + block layers + aux layers + head."""

    shared_gpu_pdl = False   # see LocalModule.shared_gpu_pdl

    def __init__(self, stage_index, spec, groups, n_block, n_aux, optimizer, schedule,
                 assigned_aux_depth, *, flat, device, precision, final):
        self.spec = spec
        self.groups = groups                 # [(group, key, Tensor)] in buffer order
        self.n_block_layers = n_block
        self.n_aux_layers = n_aux
        self.has_patch = stage_index == 0
        super().__init__(stage_index, [g for g in groups], None, optimizer, schedule,
                         assigned_aux_depth, flat=flat, device=device, precision=precision)
        self.final = final

    # -- shapes --------------------------------------------------------------
    @property
    def in_shape(self) -> tuple:
        sp = self.spec
        return (sp.channels, sp.image, sp.image) if self.has_patch else (sp.tokens, sp.dim)

    @property
    def out_shape(self) -> tuple:
        return (self.spec.tokens, self.spec.dim)

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
        return [t for g, _, t in self.groups if g == "patch" or g.startswith("block")]

    def all_layers(self) -> list:
        return []

    # -- native executor -------------------------------------------------------
    def native(self, batch: int):
        if self._native is not None and batch <= self._native_batch:
            return self._native
        self.close()
        f = self._flat
        sp = self.spec
        cfg = (C.c_int * 12)(batch, sp.tokens, sp.dim, sp.heads, sp.mlp, sp.classes,
                             self.n_block_layers, self.n_aux_layers, int(self.has_patch),
                             sp.channels, sp.image, sp.patch)
        offs = f["offsets"]
        arr = (C.c_int64 * len(offs))(*offs)
        lib = N.load()
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            free0 = torch.cuda.mem_get_info()[0]
            h = lib.ppll_vit_stage_create(
                cfg, arr, f["theta"].numel(), N.BF16 if self.precision == "bf16" else N.F32,
                f["theta"].data_ptr(), f["grad"].data_ptr(), f["mom"].data_ptr(),
                N.ptr(f["theta_lp"]), f["lr"].data_ptr(), f["state"].data_ptr(),
                self.schedule.total_steps, f["loss"].data_ptr(), f["state"][2:].data_ptr(),
                float(self.optimizer.mu), float(self.optimizer.weight_decay))
        if not h:
            raise N.NativeError("ppll_vit_stage_create failed: " +
                                lib.ppll_last_error().decode(errors="replace"))
        self._native_bytes = max(0, free0 - torch.cuda.mem_get_info(self.device)[0])
        self._native, self._native_batch = h, batch
        return h

    def close(self) -> None:
        if self._native is not None:
            N.load().ppll_vit_stage_destroy(self._native)
            self._native = None
            self._native_batch = 0

    def launch_step(self, B, x_ptr, y_ptr, out_ptr, stream) -> None:
        N.check(N.load().ppll_vit_stage_step(self.native(B), B, x_ptr, y_ptr, out_ptr, stream),
                f"vit stage {self.stage_index} step")

    def launch_forward(self, B, x_ptr, h_ptr, logits_ptr, stream) -> None:
        N.check(N.load().ppll_vit_stage_forward(self.native(B), B, x_ptr, h_ptr, logits_ptr,
                                                stream), f"vit stage {self.stage_index} forward")

    # -- the E2E / naive-PP baselines (runtime.py:248-284, 359-382) ---------
    def launch_block_forward(self, B, x_ptr, h_ptr, stream) -> None:
        N.check(N.load().ppll_vit_stage_block_forward(self.native(B), B, x_ptr, h_ptr, stream),
                f"vit stage {self.stage_index} block forward")

    def launch_block_backward(self, B, x_ptr, gout_ptr, y_ptr, gin_ptr, stream) -> None:
        N.check(N.load().ppll_vit_stage_block_backward(self.native(B), B, x_ptr, gout_ptr, y_ptr,
                                                       gin_ptr, stream),
                f"vit stage {self.stage_index} block backward")

    def __repr__(self) -> str:
        return (f"VitLocalModule(stage={self.stage_index}, layers={self.n_block_layers}, "
                f"aux_layers={self.n_aux_layers}, precision={self.precision})")


def build_vit_modules(spec: VitSpec, depths: Sequence[int], d_prime: int, n: int,
                      hyper: Hyperparams, devices: Sequence | None = None,
                      only: Sequence[int] | None = None) -> list:
    """One VitLocalModule per block (``depths[j]`` transformer layers each).

    Init mirrors blocks.py:198-237: ``default_rng(seed + j)`` per stage; linear
    W ~ U(±1/√fan_in) then b; LayerNorm gamma=1, beta=0 (no draws); stage 0
    draws its patch projection, then cls and pos (0.02·N(0,1)); then block
    layers, aux layers, and the head classifier."""
    depths = [int(d) for d in depths]
    if sum(depths) != spec.depth or min(depths) < 1:
        raise ConfigMismatch(f"block depths {depths} must be >= 1 and sum to {spec.depth}")
    s = len(depths)
    mods = []
    for j, dj in enumerate(depths):
        if only is not None and j not in only:
            continue
        device = torch.device(devices[j]) if devices is not None else default_device()
        if device.type == "cuda" and device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        rng = np.random.default_rng(hyper.seed + j)
        host = []
        if j == 0:
            wpe, bpe = _lin(rng, spec.patch_dim, spec.dim)
            cls = 0.02 * rng.standard_normal(spec.dim)
            pos = 0.02 * rng.standard_normal((spec.tokens, spec.dim))
            host += [("patch", "wpe", wpe), ("patch", "bpe", bpe), ("patch", "cls", cls),
                     ("patch", "pos", pos)]
        for i in range(dj):
            L = _init_layer(rng, spec)
            host += [(f"block{i}", k, L[k]) for k in LAYER_KEYS]
        final = j == s - 1
        n_aux = 0 if final else aux_depth(j, d_prime, n)
        for i in range(n_aux):
            L = _init_layer(rng, spec)
            host += [(f"aux{i}", k, L[k]) for k in LAYER_KEYS]
        wh, bh = _lin(rng, spec.dim, spec.classes)
        host += [("head", "lnf_g", np.ones(spec.dim)), ("head", "lnf_b", np.zeros(spec.dim)),
                 ("head", "wh", wh), ("head", "bh", bh)]
        # flat buffers, 256-B aligned tensors
        offsets, cur = [], 0
        for _, _, a in host:
            offsets.append(cur)
            cur += (a.size + _ALIGN - 1) // _ALIGN * _ALIGN
        flat_host = np.zeros(max(cur, _ALIGN))
        for (_, _, a), o in zip(host, offsets):
            flat_host[o:o + a.size] = a.ravel()
        theta = torch.from_numpy(flat_host).to(device=device, dtype=torch.float32)
        mom, grad = torch.zeros_like(theta), torch.zeros_like(theta)
        theta_lp = theta.to(torch.bfloat16) if hyper.precision == "bf16" else None
        sched = LrSchedule(hyper.lr0, hyper.lr_min, hyper.total_steps)
        native_offs = (offsets[:4] if j == 0 else [-1] * 4) + offsets[(4 if j == 0 else 0):]
        flat = {"theta": theta, "mom": mom, "grad": grad, "theta_lp": theta_lp,
                "offsets": native_offs, "lr": lr_table(sched, device),
                "state": torch.zeros(4, dtype=torch.int32, device=device),
                "loss": torch.zeros(hyper.total_steps + 2, dtype=torch.float32, device=device)}
        attach_local_optimizer(flat, hyper)
        groups, moms = [], []
        for (g, k, a), o in zip(host, offsets):
            view = theta[o:o + a.size].view(a.shape)
            groups.append((g, k, Tensor(view, track_grad=True)))
            moms.append(mom[o:o + a.size].view(a.shape))
        opt = OptimizerState([t for _, _, t in groups], hyper.momentum, hyper.weight_decay,
                             _flat=(theta, mom, grad, moms))
        mods.append(VitLocalModule(j, spec, groups, dj, n_aux, opt, sched,
                                   aux_depth(j, d_prime, n), flat=flat, device=device,
                                   precision=hyper.precision, final=final))
    return mods
