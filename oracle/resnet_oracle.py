"""CPU oracle for PPLL ResNet local-learning stages — TEST INFRASTRUCTURE ONLY.

No reference implementation of convolutional blocks exists (SURVEY §0.2 /
§8c: "parity unpinned by the reference").  This numpy float64 restatement
follows the reference's local-step semantics where they apply (blocks.py
:266-289 step order; optim.py:71-89 L2-Nesterov on every parameter incl.
BN affine; cosine LR; per-stage ``default_rng(seed + j)`` init, W before b;
aux depth blocks.py:99-106; no aux on the final stage) and is pinned against
torch.autograd in float64 (tests/test_resnet_oracle.py).

Builder decisions: CIFAR ResNet (He et al.) with 3 groups of n
basic blocks (16/32/64 channels), option-B shortcut (1x1 stride-2 conv + BN)
on downsampling, BatchNorm in training mode (batch statistics, biased
variance, eps 1e-5; gamma=1, beta=0, no running stats), conv weights
U(±1/sqrt(fan_in)) without bias; head = global average pool + linear;
aux head for stage l = aux_depth(l, d', n) x [conv3x3 + BN + ReLU] at the
boundary resolution, then GAP + linear.  Layout NHWC; a conv weight is
stored [kh*kw*C_in, C_out] (tap-major rows) so a conv is im2col · W.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ppll_oracle import aux_depth, cosine_lr, nesterov_update
from ppll_oracle import softmax_xent as _xent

BN_EPS = 1e-5


@dataclass(frozen=True)
class ResNetSpec:
    n: int = 5                 # blocks per group: 5 -> ResNet-32, 18 -> ResNet-110
    image: int = 32
    channels: int = 3
    widths: tuple = (16, 32, 64)
    classes: int = 10

    @property
    def n_blocks(self) -> int:
        return 3 * self.n


def block_geometry(spec: ResNetSpec, b: int):
    """(C_in, C_out, stride, H_in) of basic block b (0-based)."""
    g = b // spec.n
    cout = spec.widths[g]
    first = b % spec.n == 0
    cin = spec.widths[g - 1] if (first and g > 0) else cout
    stride = 2 if (first and g > 0) else 1
    h_in = spec.image // (2 ** g) * (2 if stride == 2 else 1)
    return cin, cout, stride, h_in


def resnet_split(spec: ResNetSpec, s: int) -> list:
    """Contiguous split of the units [stem, block0, ..., block_{3n-1}] into s
    stages, as even as possible (earlier stages take the remainder).
    Returns per stage the list of block indices (stage 0 also has the stem)."""
    units = spec.n_blocks + 1
    if s < 1 or s > units:
        raise ValueError(f"cannot split {units} units into {s} stages")
    q, r = divmod(units, s)
    sizes = [q + (1 if j < r else 0) for j in range(s)]
    out, u = [], 0
    for sz in sizes:
        out.append([x - 1 for x in range(u, u + sz) if x >= 1])
        u += sz
    return out


def stage_out_geometry(spec: ResNetSpec, blocks):
    """(C, H) of the activation leaving a stage."""
    if not blocks:
        return spec.widths[0], spec.image
    cin, cout, stride, h_in = block_geometry(spec, blocks[-1])
    return cout, h_in // stride


# --------------------------------------------------------------------------
# parameters
# --------------------------------------------------------------------------

def _conv_w(rng, k, cin, cout):
    bound = 1.0 / math.sqrt(k * k * cin)
    return rng.uniform(-bound, bound, size=(k * k * cin, cout))


def _bn(c):
    return {"g": np.ones(c), "b": np.zeros(c)}


def init_block(rng, cin, cout, stride):
    p = {"w1": _conv_w(rng, 3, cin, cout), "bn1": _bn(cout),
         "w2": _conv_w(rng, 3, cout, cout), "bn2": _bn(cout)}
    if stride != 1 or cin != cout:
        p["ws"] = _conv_w(rng, 1, cin, cout)
        p["bns"] = _bn(cout)
    return p


@dataclass
class ResStage:
    index: int
    spec: ResNetSpec
    stem: dict | None           # {"w": [27, 16], "bn"}
    blocks: list                # (geometry, params)
    aux: list                   # [(w [9C, C], bn)]
    head: dict                  # {"w": [C, classes], "b": [classes]}
    final: bool
    momenta: list = field(default_factory=list)
    step_count: int = 0

    def param_list(self):
        out = []
        if self.stem is not None:
            out += [("stem", "w", self.stem["w"]), ("stem", "bn_g", self.stem["bn"]["g"]),
                    ("stem", "bn_b", self.stem["bn"]["b"])]
        for i, (_, p) in enumerate(self.blocks):
            for k in ("w1", "bn1", "w2", "bn2", "ws", "bns"):
                if k not in p:
                    continue
                if k.startswith("bn"):
                    out += [(f"block{i}", k + "_g", p[k]["g"]), (f"block{i}", k + "_b", p[k]["b"])]
                else:
                    out.append((f"block{i}", k, p[k]))
        for i, (w, bn) in enumerate(self.aux):
            out += [(f"aux{i}", "w", w), (f"aux{i}", "bn_g", bn["g"]), (f"aux{i}", "bn_b", bn["b"])]
        out += [("head", "w", self.head["w"]), ("head", "b", self.head["b"])]
        return out

    def params(self):
        return [a for _, _, a in self.param_list()]


def build_resnet_stages(spec: ResNetSpec, s: int, d_prime: int, n_int: int, seed: int,
                        split=None):
    """``split``: per stage the list of block indices (default: the even
    ``resnet_split``; the product's cost-balanced split is passed in
    explicitly by the tests that use it)."""
    split = resnet_split(spec, s) if split is None else [list(b) for b in split]
    if len(split) != s:
        raise ValueError(f"split has {len(split)} stages, expected {s}")
    stages = []
    for j, blocks in enumerate(split):
        rng = np.random.default_rng(seed + j)
        stem = None
        if j == 0:
            stem = {"w": _conv_w(rng, 3, spec.channels, spec.widths[0]), "bn": _bn(spec.widths[0])}
        bl = []
        for b in blocks:
            cin, cout, stride, h = block_geometry(spec, b)
            bl.append(((cin, cout, stride, h), init_block(rng, cin, cout, stride)))
        c_out, _ = stage_out_geometry(spec, blocks)
        final = j == s - 1
        aux = [] if final else [(_conv_w(rng, 3, c_out, c_out), _bn(c_out))
                                for _ in range(aux_depth(j, d_prime, n_int))]
        bound = 1.0 / math.sqrt(c_out)
        head = {"w": rng.uniform(-bound, bound, size=(c_out, spec.classes)),
                "b": rng.uniform(-bound, bound, size=(spec.classes,))}
        st = ResStage(j, spec, stem, bl, aux, head, final)
        st.momenta = [np.zeros_like(p) for p in st.params()]
        stages.append(st)
    return stages


# --------------------------------------------------------------------------
# primitives (NHWC)
# --------------------------------------------------------------------------

def im2col(x, k, stride):
    """x [N,H,W,C] -> [N·Ho·Wo, k·k·C] (tap-major (r, s, c)), pad (k-1)/2."""
    N, H, W, C = x.shape
    p = (k - 1) // 2
    xp = np.pad(x, ((0, 0), (p, p), (p, p), (0, 0)))
    Ho, Wo = (H + 2 * p - k) // stride + 1, (W + 2 * p - k) // stride + 1
    cols = np.empty((N, Ho, Wo, k, k, C))
    for r in range(k):
        for s_ in range(k):
            cols[:, :, :, r, s_, :] = xp[:, r:r + stride * Ho:stride, s_:s_ + stride * Wo:stride, :]
    return cols.reshape(N * Ho * Wo, k * k * C), (N, Ho, Wo)


def col2im(dcol, shape_in, k, stride):
    N, H, W, C = shape_in
    p = (k - 1) // 2
    Ho, Wo = (H + 2 * p - k) // stride + 1, (W + 2 * p - k) // stride + 1
    d = dcol.reshape(N, Ho, Wo, k, k, C)
    dxp = np.zeros((N, H + 2 * p, W + 2 * p, C))
    for r in range(k):
        for s_ in range(k):
            dxp[:, r:r + stride * Ho:stride, s_:s_ + stride * Wo:stride, :] += d[:, :, :, r, s_, :]
    return dxp[:, p:p + H, p:p + W, :]


def conv_fwd(x, w, k, stride):
    cols, (N, Ho, Wo) = im2col(x, k, stride)
    return (cols @ w).reshape(N, Ho, Wo, -1), cols


def conv_bwd(dy, cols, w, x_shape, k, stride):
    d2 = dy.reshape(-1, dy.shape[-1])
    dw = cols.T @ d2
    dx = col2im(d2 @ w.T, x_shape, k, stride)
    return dx, dw


def bn_fwd(z, g, b):
    """training-mode BatchNorm over N·H·W per channel (biased variance)."""
    C = z.shape[-1]
    z2 = z.reshape(-1, C)
    mu = z2.mean(0)
    var = ((z2 - mu) ** 2).mean(0)
    rstd = 1.0 / np.sqrt(var + BN_EPS)
    xh = (z - mu) * rstd
    return xh * g + b, (xh, rstd)


def bn_bwd(dy, cache, g):
    xh, rstd = cache
    C = dy.shape[-1]
    d2, x2 = dy.reshape(-1, C), xh.reshape(-1, C)
    P = d2.shape[0]
    dg = (d2 * x2).sum(0)
    db = d2.sum(0)
    dx = (g * rstd / P) * (P * dy - db - xh * dg)
    return dx, dg, db


def block_fwd(x, geo, p):
    cin, cout, stride, _ = geo
    z1, c1 = conv_fwd(x, p["w1"], 3, stride)
    y1, b1 = bn_fwd(z1, p["bn1"]["g"], p["bn1"]["b"])
    a1 = np.maximum(y1, 0.0)
    z2, c2 = conv_fwd(a1, p["w2"], 3, 1)
    y2, b2 = bn_fwd(z2, p["bn2"]["g"], p["bn2"]["b"])
    if "ws" in p:
        zs, cs = conv_fwd(x, p["ws"], 1, stride)
        sc, bs = bn_fwd(zs, p["bns"]["g"], p["bns"]["b"])
    else:
        sc, cs, bs = x, None, None
    out = np.maximum(y2 + sc, 0.0)
    return out, (x, c1, b1, a1, c2, b2, cs, bs, out)


def block_bwd(dout, cache, geo, p):
    cin, cout, stride, _ = geo
    x, c1, b1, a1, c2, b2, cs, bs, out = cache
    g = {}
    dsum = dout * (out > 0)
    dz2, g["bn2_g"], g["bn2_b"] = bn_bwd(dsum, b2, p["bn2"]["g"])
    da1, g["w2"] = conv_bwd(dz2, c2, p["w2"], a1.shape, 3, 1)
    dy1 = da1 * (a1 > 0)
    dz1, g["bn1_g"], g["bn1_b"] = bn_bwd(dy1, b1, p["bn1"]["g"])
    dx, g["w1"] = conv_bwd(dz1, c1, p["w1"], x.shape, 3, stride)
    if "ws" in p:
        dzs, g["bns_g"], g["bns_b"] = bn_bwd(dsum, bs, p["bns"]["g"])
        dxs, g["ws"] = conv_bwd(dzs, cs, p["ws"], x.shape, 1, stride)
        dx = dx + dxs
    else:
        dx = dx + dsum
    return dx, g


def aux_layer_fwd(x, w, bn):
    z, c = conv_fwd(x, w, 3, 1)
    y, b = bn_fwd(z, bn["g"], bn["b"])
    return np.maximum(y, 0.0), (x, c, b, y)


def aux_layer_bwd(dout, cache, w, bn):
    x, c, b, y = cache
    dy = dout * (y > 0)
    dz, dg, db = bn_bwd(dy, b, bn["g"])
    dx, dw = conv_bwd(dz, c, w, x.shape, 3, 1)
    return dx, dw, dg, db


def head_fwd(x, hd):
    pooled = x.mean(axis=(1, 2))
    return pooled @ hd["w"] + hd["b"], pooled


def head_bwd(dlog, pooled, hd, x_shape):
    N, H, W, C = x_shape
    g = {"w": pooled.T @ dlog, "b": dlog.sum(0)}
    dp = dlog @ hd["w"].T
    dx = np.broadcast_to(dp[:, None, None, :] / (H * W), x_shape).copy()
    return dx, g


# --------------------------------------------------------------------------
# one local step (blocks.py:266-289 order)
# --------------------------------------------------------------------------

def local_grads(st: ResStage, x_in, y):
    """x_in: NHWC float64.  Returns (loss, x_out, logits, grads in param order)."""
    x = x_in
    stem_cache = None
    if st.stem is not None:
        z, cs = conv_fwd(x, st.stem["w"], 3, 1)
        yb, bb = bn_fwd(z, st.stem["bn"]["g"], st.stem["bn"]["b"])
        stem_cache = (x, cs, bb, np.maximum(yb, 0.0), yb)
        x = stem_cache[3]
    caches = []
    for geo, p in st.blocks:
        x, c = block_fwd(x, geo, p)
        caches.append(c)
    x_out = x.copy()
    aux_caches = []
    for w, bn in st.aux:
        x, c = aux_layer_fwd(x, w, bn)
        aux_caches.append(c)
    logits, pooled = head_fwd(x, st.head)
    loss, dlog = _xent(logits, y)
    dx, gh = head_bwd(dlog, pooled, st.head, x.shape)
    g_aux = []
    for (w, bn), c in zip(reversed(st.aux), reversed(aux_caches)):
        dx, dw, dg, db = aux_layer_bwd(dx, c, w, bn)
        g_aux.append((dw, dg, db))
    g_aux.reverse()
    g_blk = []
    for (geo, p), c in zip(reversed(st.blocks), reversed(caches)):
        dx, g = block_bwd(dx, c, geo, p)
        g_blk.append(g)
    g_blk.reverse()
    grads = []
    if st.stem is not None:
        xs, cs, bb, a, yb = stem_cache
        dz, dg, db = bn_bwd(dx * (yb > 0), bb, st.stem["bn"]["g"])
        dwst = cs.T @ dz.reshape(-1, dz.shape[-1])
        grads += [dwst, dg, db]
    for (geo, p), g in zip(st.blocks, g_blk):
        for k in ("w1", "bn1", "w2", "bn2", "ws", "bns"):
            if k not in p:
                continue
            grads += [g[k + "_g"], g[k + "_b"]] if k.startswith("bn") else [g[k]]
    for dw, dg, db in g_aux:
        grads += [dw, dg, db]
    grads += [gh["w"], gh["b"]]
    return loss, x_out, logits, grads


def local_step(st: ResStage, x_in, y, lr0, lr_min, total_steps, mu, wd):
    loss, x_out, logits, grads = local_grads(st, x_in, y)
    lr = cosine_lr(st.step_count, lr0, lr_min, total_steps)
    for p, v, g in zip(st.params(), st.momenta, grads):
        nesterov_update(p, v, g, lr, mu, wd)
    st.step_count += 1
    return loss, x_out, logits
