"""Torch-CPU restatement of the PPLL local step — TEST / BASELINE INFRASTRUCTURE ONLY.

BASELINE.md §3: ResNet and ViT cannot run on the reference (it is MLP-only,
SURVEY §0.2), so the CPU column for those configs is a torch-CPU fp32
*restatement* of the same local-learning step, run with every host thread.
This module is that restatement.  It takes the stages built by the numpy
oracles (``vit_oracle.build_vit_stages`` / ``resnet_oracle.build_resnet_stages``
/ ``ppll_oracle.build_stages`` — the reference's seeded init order,
blocks.py:190-237) and runs the reference's step order (blocks.py:266-289):

  block forward -> x_out (pre-update, detached) -> aux forward -> mean
  softmax-CE (tensor.py:201-234) -> backward (autograd; no gradient into the
  detached stage input) -> cosine_lr(step_count) (optim.py:39-44) ->
  L2-in-gradient Nesterov on every parameter (optim.py:81-88).

Gradients come from torch.autograd instead of the oracles' manual backward;
``tests/test_torch_cpu.py`` pins this restatement to the float64 numpy oracles
(float64 mode, 1e-9) so the two derivations check each other.  Only
``tests/`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs
import it; the product path never does.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

LN_EPS = 1e-5
BN_EPS = 1e-5


def cosine_lr(step, lr0, lr_min, total_steps):
    """optim.py:39-44."""
    if step < 0 or step > total_steps:
        raise ValueError(f"step {step} outside [0, {total_steps}]")
    return lr_min + 0.5 * (lr0 - lr_min) * (1.0 + math.cos(math.pi * step / total_steps))


class TorchStage:
    """One stage: a flat parameter list in the oracle's ``param_list`` order
    plus the forward closures of its block / aux-and-head."""

    def __init__(self, index, params, block_fn, head_fn, dtype):
        self.index = index
        self.params = [torch.tensor(np.asarray(p), dtype=dtype).requires_grad_(True)
                       for p in params]
        self.momenta = [torch.zeros_like(p, requires_grad=False) for p in self.params]
        self.block_fn = block_fn
        self.head_fn = head_fn
        self.step_count = 0
        self.dtype = dtype


# --------------------------------------------------------------------------
# ViT (vit_oracle.py semantics: pre-LN, erf GELU, cls token + learned pos)
# --------------------------------------------------------------------------

_VIT_KEYS = 12      # vit_oracle.LAYER_KEYS


def _vit_layer(x, p, heads):
    ln1_g, ln1_b, wqkv, bqkv, wo, bo, ln2_g, ln2_b, w1, b1, w2, b2 = p
    B, T, D = x.shape
    dh = D // heads
    xn = F.layer_norm(x, (D,), ln1_g, ln1_b, LN_EPS)
    qkv = xn @ wqkv + bqkv
    q, k, v = (t.reshape(B, T, heads, dh).transpose(1, 2) for t in qkv.split(D, dim=-1))
    o = F.scaled_dot_product_attention(q, k, v)          # scale 1/sqrt(dh)
    x1 = x + o.transpose(1, 2).reshape(B, T, D) @ wo + bo
    xn2 = F.layer_norm(x1, (D,), ln2_g, ln2_b, LN_EPS)
    return x1 + F.gelu(xn2 @ w1 + b1) @ w2 + b2


def from_vit(st, dtype=torch.float32) -> TorchStage:
    """A vit_oracle.VitStage as a TorchStage (same parameter values/order)."""
    spec = st.spec
    has_patch = st.patch is not None
    nb, na = len(st.block), len(st.aux)
    off_blk = 4 if has_patch else 0
    off_aux = off_blk + _VIT_KEYS * nb
    off_head = off_aux + _VIT_KEYS * na

    def block_fn(P, x):
        if has_patch:
            wpe, bpe, cls, pos = P[:4]
            B, C, H, W = x.shape
            p = spec.patch
            pt = x.reshape(B, C, H // p, p, W // p, p).permute(0, 2, 4, 1, 3, 5)
            tok = pt.reshape(B, (H // p) * (W // p), C * p * p) @ wpe + bpe
            x = torch.cat([cls.expand(B, 1, spec.dim), tok], dim=1) + pos
        for i in range(nb):
            x = _vit_layer(x, P[off_blk + _VIT_KEYS * i: off_blk + _VIT_KEYS * (i + 1)],
                           spec.heads)
        return x

    def head_fn(P, h):
        x = h
        for i in range(na):
            x = _vit_layer(x, P[off_aux + _VIT_KEYS * i: off_aux + _VIT_KEYS * (i + 1)],
                           spec.heads)
        g, b, wh, bh = P[off_head:off_head + 4]
        return F.layer_norm(x[:, 0], (spec.dim,), g, b, LN_EPS) @ wh + bh

    return TorchStage(st.index, st.params(), block_fn, head_fn, dtype)


# --------------------------------------------------------------------------
# ResNet (resnet_oracle.py semantics: NHWC, train-mode BN, option-B shortcut)
# --------------------------------------------------------------------------

def _conv(x, w, k, cin, stride):
    """x NCHW; w stored [k*k*cin, cout] tap-major (resnet_oracle.im2col)."""
    wt = w.reshape(k, k, cin, -1).permute(3, 2, 0, 1)
    return F.conv2d(x, wt, stride=stride, padding=(k - 1) // 2)


def _bn(z, g, b):
    return F.batch_norm(z, None, None, g, b, training=True, eps=BN_EPS)


def from_resnet(st, dtype=torch.float32) -> TorchStage:
    spec = st.spec
    layout = []            # how to walk the flat parameter list
    if st.stem is not None:
        layout.append(("stem", 3))
    for geo, p in st.blocks:
        layout.append(("block", geo, "ws" in p))
    n_aux = len(st.aux)

    def block_fn(P, x):
        x = x.permute(0, 3, 1, 2)                            # NHWC -> NCHW view
        i = 0
        for item in layout:
            if item[0] == "stem":
                x = F.relu(_bn(_conv(x, P[0], 3, spec.channels, 1), P[1], P[2]))
                i = 3
                continue
            _, (cin, cout, stride, _), short = item
            w1, g1, b1, w2, g2, b2 = P[i:i + 6]
            i += 6
            a1 = F.relu(_bn(_conv(x, w1, 3, cin, stride), g1, b1))
            y2 = _bn(_conv(a1, w2, 3, cout, 1), g2, b2)
            if short:
                ws, gs, bs = P[i:i + 3]
                i += 3
                sc = _bn(_conv(x, ws, 1, cin, stride), gs, bs)
            else:
                sc = x
            x = F.relu(y2 + sc)
        return x.permute(0, 2, 3, 1)                         # back to NHWC

    def head_fn(P, h):
        x = h.permute(0, 3, 1, 2)
        base = len(P) - 2 - 3 * n_aux
        C = x.shape[1]
        for a in range(n_aux):
            w, g, b = P[base + 3 * a: base + 3 * a + 3]
            x = F.relu(_bn(_conv(x, w, 3, C, 1), g, b))
        return x.mean(dim=(2, 3)) @ P[-2] + P[-1]

    return TorchStage(st.index, st.params(), block_fn, head_fn, dtype)


# --------------------------------------------------------------------------
# MLP (ppll_oracle.py / blocks.py:240-263)
# --------------------------------------------------------------------------

def from_mlp(st, dtype=torch.float32) -> TorchStage:
    relu_b = [r for _, _, r in st.block]
    relu_a = [r for _, _, r in st.aux]
    nb = len(relu_b)

    def _chain(P, x, relus, off):
        for i, r in enumerate(relus):
            x = x @ P[off + 2 * i] + P[off + 2 * i + 1]
            if r:
                x = F.relu(x)
        return x

    return TorchStage(st.index, st.params(),
                      lambda P, x: _chain(P, x, relu_b, 0),
                      lambda P, h: _chain(P, h, relu_a, 2 * nb) if relu_a else h,
                      dtype)


# --------------------------------------------------------------------------
# the local step (blocks.py:266-289)
# --------------------------------------------------------------------------

def local_step(ts: TorchStage, x_in, y, lr0, lr_min, total_steps, mu, wd, opt="nesterov",
               betas=(0.9, 0.999), eps=1e-8):
    """One local step; returns (loss, x_out detached, logits detached).
    ``opt="adamw"``: torch.optim.AdamW's rule (decoupled weight decay,
    bias-corrected moments, t = step_count + 1) instead of the reference's
    Nesterov — the checker of the device's AdamW local update (north_star's
    "local SGD/Adam update"; the reference has no Adam)."""
    x_in = torch.as_tensor(x_in).to(ts.dtype).detach()
    y = torch.as_tensor(np.asarray(y)).long()
    P = ts.params
    h = ts.block_fn(P, x_in)
    x_out = h.detach()                       # pushed before the update
    logits = ts.head_fn(P, h)
    loss = F.cross_entropy(logits, y)        # mean over the batch
    grads = torch.autograd.grad(loss, P)
    lr = cosine_lr(ts.step_count, lr0, lr_min, total_steps)
    if opt == "adamw":
        if not hasattr(ts, "momenta2"):
            ts.momenta2 = [torch.zeros_like(p, requires_grad=False) for p in P]
        b1, b2 = betas
        t = ts.step_count + 1
        with torch.no_grad():
            for p, m, v, g in zip(P, ts.momenta, ts.momenta2, grads):
                p.mul_(1.0 - lr * wd)
                m.mul_(b1).add_(g, alpha=1.0 - b1)
                v.mul_(b2).addcmul_(g, g, value=1.0 - b2)
                p.sub_(lr * (m / (1.0 - b1 ** t)) / ((v / (1.0 - b2 ** t)).sqrt() + eps))
        ts.step_count += 1
        return float(loss.detach()), x_out, logits.detach()
    with torch.no_grad():
        for p, v, g in zip(P, ts.momenta, grads):
            if wd != 0.0:
                g = g + wd * p
            v.mul_(mu).add_(g)
            p.sub_(lr * (g + mu * v))
    ts.step_count += 1
    return float(loss.detach()), x_out, logits.detach()


# --------------------------------------------------------------------------
# the paper's E2E baseline (reference runtime.py:248-284)
# --------------------------------------------------------------------------

def e2e_step(stages, x_in, y, lr0, lr_min, total_steps, mu, wd):
    """One end-to-end backprop step through every stage's BLOCK (aux heads
    unused): the final stage's block ends in its task head (the final stage
    has no aux layers, so ``head_fn`` is that head); the mean softmax-CE of
    the final logits is differentiated w.r.t. every parameter on the path and
    each stage takes the reference's L2-in-gradient Nesterov step on those
    parameters only (runtime.py:276-281); parameters off the path (aux heads)
    are left untouched.  Every stage's step counter advances.  Returns the
    loss."""
    x = torch.as_tensor(x_in).to(stages[0].dtype).detach()
    y = torch.as_tensor(np.asarray(y)).long()
    h = x
    for ts in stages:
        h = ts.block_fn(ts.params, h)
    logits = stages[-1].head_fn(stages[-1].params, h)
    loss = F.cross_entropy(logits, y)
    allp = [p for ts in stages for p in ts.params]
    grads = torch.autograd.grad(loss, allp, allow_unused=True)
    k = 0
    for ts in stages:
        lr = cosine_lr(ts.step_count, lr0, lr_min, total_steps)
        with torch.no_grad():
            for p, v in zip(ts.params, ts.momenta):
                g = grads[k]
                k += 1
                if g is None:
                    continue
                if wd != 0.0:
                    g = g + wd * p
                v.mul_(mu).add_(g)
                p.sub_(lr * (g + mu * v))
        ts.step_count += 1
    return float(loss.detach())
