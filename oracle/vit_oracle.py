"""CPU oracle for PPLL ViT local-learning stages — TEST INFRASTRUCTURE ONLY.

The reference (locopipe) is MLP-only; ViT blocks have NO reference
implementation (SURVEY §0.2, §8c "parity unpinned by the reference").  This
numpy float64 restatement follows the reference's local-step semantics
exactly where they apply:

  * step order  blocks.py:266-289 — block forward; x_out (pre-update) pushed;
    aux forward; mean softmax-CE (tensor.py:201-234); backward with NO
    gradient into the detached stage input; cosine_lr(step_count)
    (optim.py:39-44); L2-in-gradient Nesterov on EVERY stage parameter,
    including biases / LayerNorm / embeddings (optim.py:81-88);
  * init        blocks.py:190-237 — per-stage ``default_rng(seed + j)``, each
    linear W ~ U(±1/sqrt(fan_in)) drawn before its b, block before aux;
  * aux depth   blocks.py:99-106 — N_l = max(0, d' - floor(l/n)) transformer
    layers, then LayerNorm + linear classifier on the cls token (PAPER.md
    :265-271); the final stage's head is the task head (no aux).

Builder decisions (documented in DESIGN.md): pre-LN transformer layers
(LN → MHSA → +res; LN → FC1 → GELU(erf) → FC2 → +res), LayerNorm eps 1e-5
(gamma=1, beta=0, no draws), cls/pos ~ 0.02·N(0,1) drawn right after the
patch projection, attention scale 1/sqrt(head_dim).

Its manual backward is pinned against torch.autograd in float64
(tests/test_vit_oracle.py); only tests/, smoke() and bench.py's CPU legs
import this module.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ppll_oracle import aux_depth, cosine_lr, nesterov_update
from ppll_oracle import softmax_xent as _xent

LN_EPS = 1e-5


@dataclass(frozen=True)
class VitSpec:
    image: int = 32
    channels: int = 3
    patch: int = 4
    dim: int = 384
    heads: int = 6
    mlp: int = 1536
    depth: int = 8
    classes: int = 10

    @property
    def n_patches(self) -> int:
        return (self.image // self.patch) ** 2

    @property
    def tokens(self) -> int:
        return self.n_patches + 1

    @property
    def patch_dim(self) -> int:
        return self.channels * self.patch * self.patch


# --------------------------------------------------------------------------
# parameters
# --------------------------------------------------------------------------

LAYER_KEYS = ("ln1_g", "ln1_b", "wqkv", "bqkv", "wo", "bo", "ln2_g", "ln2_b", "w1", "b1",
              "w2", "b2")


def _lin(rng, fi, fo):
    bound = 1.0 / math.sqrt(fi)
    W = rng.uniform(-bound, bound, size=(fi, fo))
    b = rng.uniform(-bound, bound, size=(fo,))
    return W, b


def init_layer(rng, spec):
    D, F = spec.dim, spec.mlp
    p = {"ln1_g": np.ones(D), "ln1_b": np.zeros(D)}
    p["wqkv"], p["bqkv"] = _lin(rng, D, 3 * D)
    p["wo"], p["bo"] = _lin(rng, D, D)
    p["ln2_g"], p["ln2_b"] = np.ones(D), np.zeros(D)
    p["w1"], p["b1"] = _lin(rng, D, F)
    p["w2"], p["b2"] = _lin(rng, F, D)
    return p


@dataclass
class VitStage:
    index: int
    spec: VitSpec
    patch: dict | None          # {"wpe","bpe","cls","pos"} on stage 0
    block: list                 # list of layer dicts
    aux: list                   # aux transformer layers (empty on the final stage)
    head: dict                  # {"lnf_g","lnf_b","wh","bh"}
    final: bool
    momenta: list = field(default_factory=list)
    step_count: int = 0

    def param_list(self):
        """Flat parameter order (also the device buffer order)."""
        out = []
        if self.patch is not None:
            out += [("patch", k, self.patch[k]) for k in ("wpe", "bpe", "cls", "pos")]
        for i, L in enumerate(self.block):
            out += [(f"block{i}", k, L[k]) for k in LAYER_KEYS]
        for i, L in enumerate(self.aux):
            out += [(f"aux{i}", k, L[k]) for k in LAYER_KEYS]
        out += [("head", k, self.head[k]) for k in ("lnf_g", "lnf_b", "wh", "bh")]
        return out

    def params(self):
        return [a for _, _, a in self.param_list()]


def build_vit_stages(spec: VitSpec, depths, d_prime, n, seed):
    """One stage per entry of ``depths`` (transformer layers per block)."""
    if sum(depths) != spec.depth:
        raise ValueError("stage depths must sum to the network depth")
    stages = []
    s = len(depths)
    for j, dj in enumerate(depths):
        rng = np.random.default_rng(seed + j)
        patch = None
        if j == 0:
            wpe, bpe = _lin(rng, spec.patch_dim, spec.dim)
            cls = 0.02 * rng.standard_normal(spec.dim)
            pos = 0.02 * rng.standard_normal((spec.tokens, spec.dim))
            patch = {"wpe": wpe, "bpe": bpe, "cls": cls, "pos": pos}
        block = [init_layer(rng, spec) for _ in range(dj)]
        final = j == s - 1
        aux = [] if final else [init_layer(rng, spec) for _ in range(aux_depth(j, d_prime, n))]
        wh, bh = _lin(rng, spec.dim, spec.classes)
        head = {"lnf_g": np.ones(spec.dim), "lnf_b": np.zeros(spec.dim), "wh": wh, "bh": bh}
        st = VitStage(j, spec, patch, block, aux, head, final)
        st.momenta = [np.zeros_like(p) for p in st.params()]
        stages.append(st)
    return stages


# --------------------------------------------------------------------------
# primitives (forward returns a cache for the manual backward)
# --------------------------------------------------------------------------

def gelu(x):
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def gelu_grad(x):
    from scipy.special import erf
    cdf = 0.5 * (1.0 + erf(x / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return cdf + x * pdf


def ln_fwd(x, g, b):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xh = (x - mu) * rstd
    return xh * g + b, (xh, rstd)


def ln_bwd(dy, cache, g):
    xh, rstd = cache
    dg = (dy * xh).reshape(-1, xh.shape[-1]).sum(0)
    db = dy.reshape(-1, xh.shape[-1]).sum(0)
    dxh = dy * g
    dx = rstd * (dxh - dxh.mean(-1, keepdims=True) - xh * (dxh * xh).mean(-1, keepdims=True))
    return dx, dg, db


def patchify(img, p):
    """[B, C, H, W] -> [B, P, C*p*p] with (c, py, px) inner order, patches row-major."""
    B, C, H, W = img.shape
    x = img.reshape(B, C, H // p, p, W // p, p).transpose(0, 2, 4, 1, 3, 5)
    return x.reshape(B, (H // p) * (W // p), C * p * p)


def attn_fwd(qkv, B, T, H, dh):
    D = H * dh
    q = qkv[..., :D].reshape(B, T, H, dh).transpose(0, 2, 1, 3)
    k = qkv[..., D:2 * D].reshape(B, T, H, dh).transpose(0, 2, 1, 3)
    v = qkv[..., 2 * D:].reshape(B, T, H, dh).transpose(0, 2, 1, 3)
    s = q @ k.transpose(0, 1, 3, 2) / math.sqrt(dh)
    s = s - s.max(-1, keepdims=True)
    e = np.exp(s)
    P = e / e.sum(-1, keepdims=True)
    o = P @ v
    return o.transpose(0, 2, 1, 3).reshape(B, T, D), (q, k, v, P)


def attn_bwd(do, cache, B, T, H, dh):
    q, k, v, P = cache
    D = H * dh
    do = do.reshape(B, T, H, dh).transpose(0, 2, 1, 3)
    dv = P.transpose(0, 1, 3, 2) @ do
    dP = do @ v.transpose(0, 1, 3, 2)
    dS = P * (dP - (dP * P).sum(-1, keepdims=True))
    sc = 1.0 / math.sqrt(dh)
    dq = dS @ k * sc
    dk = dS.transpose(0, 1, 3, 2) @ q * sc
    out = np.empty((B, T, 3 * D))
    out[..., :D] = dq.transpose(0, 2, 1, 3).reshape(B, T, D)
    out[..., D:2 * D] = dk.transpose(0, 2, 1, 3).reshape(B, T, D)
    out[..., 2 * D:] = dv.transpose(0, 2, 1, 3).reshape(B, T, D)
    return out


def layer_fwd(x, L, spec):
    B, T, D = x.shape
    H = spec.heads
    xn1, c1 = ln_fwd(x, L["ln1_g"], L["ln1_b"])
    qkv = xn1 @ L["wqkv"] + L["bqkv"]
    o, ca = attn_fwd(qkv, B, T, H, D // H)
    x1 = x + o @ L["wo"] + L["bo"]
    xn2, c2 = ln_fwd(x1, L["ln2_g"], L["ln2_b"])
    u = xn2 @ L["w1"] + L["b1"]
    h = gelu(u)
    x2 = x1 + h @ L["w2"] + L["b2"]
    return x2, (x, xn1, c1, qkv, o, ca, x1, xn2, c2, u, h)


def layer_bwd(dx2, cache, L, spec):
    x, xn1, c1, qkv, o, ca, x1, xn2, c2, u, h = cache
    B, T, D = x.shape
    H = spec.heads
    g = {}
    f = lambda a: a.reshape(-1, a.shape[-1])  # noqa: E731
    g["w2"] = f(h).T @ f(dx2)
    g["b2"] = f(dx2).sum(0)
    du = (dx2 @ L["w2"].T) * gelu_grad(u)
    g["w1"] = f(xn2).T @ f(du)
    g["b1"] = f(du).sum(0)
    dxn2 = du @ L["w1"].T
    dx1_ln, g["ln2_g"], g["ln2_b"] = ln_bwd(dxn2, c2, L["ln2_g"])
    dx1 = dx2 + dx1_ln
    g["wo"] = f(o).T @ f(dx1)
    g["bo"] = f(dx1).sum(0)
    do = dx1 @ L["wo"].T
    dqkv = attn_bwd(do, ca, B, T, H, D // H)
    g["wqkv"] = f(xn1).T @ f(dqkv)
    g["bqkv"] = f(dqkv).sum(0)
    dxn1 = dqkv @ L["wqkv"].T
    dx_ln, g["ln1_g"], g["ln1_b"] = ln_bwd(dxn1, c1, L["ln1_g"])
    return dx1 + dx_ln, g


def patch_fwd(img, P, spec):
    B = img.shape[0]
    pt = patchify(img, spec.patch)
    tok = pt @ P["wpe"] + P["bpe"]
    x = np.empty((B, spec.tokens, spec.dim))
    x[:, 0] = P["cls"]
    x[:, 1:] = tok
    return x + P["pos"], pt


def patch_bwd(dx, pt, P):
    g = {}
    dtok = dx[:, 1:]
    g["wpe"] = pt.reshape(-1, pt.shape[-1]).T @ dtok.reshape(-1, dtok.shape[-1])
    g["bpe"] = dtok.reshape(-1, dtok.shape[-1]).sum(0)
    g["cls"] = dx[:, 0].sum(0)
    g["pos"] = dx.sum(0)
    return g


def head_fwd(x, Hd):
    cls = x[:, 0]
    z, c = ln_fwd(cls, Hd["lnf_g"], Hd["lnf_b"])
    return z @ Hd["wh"] + Hd["bh"], (z, c)


def head_bwd(dlog, cache, Hd, x_shape):
    z, c = cache
    g = {"wh": z.T @ dlog, "bh": dlog.sum(0)}
    dz = dlog @ Hd["wh"].T
    dcls, g["lnf_g"], g["lnf_b"] = ln_bwd(dz, c, Hd["lnf_g"])
    dx = np.zeros(x_shape)
    dx[:, 0] = dcls
    return dx, g


# --------------------------------------------------------------------------
# one local step (blocks.py:266-289 order)
# --------------------------------------------------------------------------

def stage_forward(st: VitStage, x_in):
    """Block forward; returns (block output, caches)."""
    caches = {}
    x = x_in
    if st.patch is not None:
        x, caches["patch"] = patch_fwd(x_in, st.patch, st.spec)
    caches["block"] = []
    for L in st.block:
        x, c = layer_fwd(x, L, st.spec)
        caches["block"].append(c)
    return x, caches


def local_grads(st: VitStage, x_in, y):
    """Forward + loss + manual backward.  Returns (loss, x_out, logits, grads)
    with grads in ``param_list`` order."""
    h, caches = stage_forward(st, x_in)
    x_out = h.copy()
    x = h
    aux_caches = []
    for L in st.aux:
        x, c = layer_fwd(x, L, st.spec)
        aux_caches.append(c)
    logits, hc = head_fwd(x, st.head)
    loss, dlog = _xent(logits, y)
    dx, gh = head_bwd(dlog, hc, st.head, x.shape)
    g_aux = []
    for L, c in zip(reversed(st.aux), reversed(aux_caches)):
        dx, g = layer_bwd(dx, c, L, st.spec)
        g_aux.append(g)
    g_aux.reverse()
    g_blk = []
    for L, c in zip(reversed(st.block), reversed(caches["block"])):
        dx, g = layer_bwd(dx, c, L, st.spec)
        g_blk.append(g)
    g_blk.reverse()
    grads = []
    if st.patch is not None:
        gp = patch_bwd(dx, caches["patch"], st.patch)
        grads += [gp[k] for k in ("wpe", "bpe", "cls", "pos")]
    for g in g_blk + g_aux:
        grads += [g[k] for k in LAYER_KEYS]
    grads += [gh[k] for k in ("lnf_g", "lnf_b", "wh", "bh")]
    return loss, x_out, logits, grads


def local_step(st: VitStage, x_in, y, lr0, lr_min, total_steps, mu, wd):
    loss, x_out, logits, grads = local_grads(st, x_in, y)
    lr = cosine_lr(st.step_count, lr0, lr_min, total_steps)
    for p, v, g in zip(st.params(), st.momenta, grads):
        nesterov_update(p, v, g, lr, mu, wd)
    st.step_count += 1
    return loss, x_out, logits
