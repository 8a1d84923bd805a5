"""CPU oracle for the PPLL local-learning hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy float64 restatement of the reference
``locopipe`` algorithm for the north-star path (one PPLL local step per
stage, the cosine-LR Nesterov update, the seeded stage initialisation, the
minimax partition, and the deterministic round-robin scheduler's integer
bookkeeping).  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2411_12780_b200``) never imports or calls it and
fails loudly when its CUDA library is missing.

Parity pinning: every function here is checked bit-for-bit (or to 1e-12)
against golden vectors produced by the reference itself
(``tests/golden/gen_golden.py`` imports ``/root/reference/pkg/src/locopipe``
in the build container and commits ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Citations are ``path:line`` relative to ``/root/reference/pkg/src/locopipe``.
"""
from __future__ import annotations

import itertools
import math
from collections import Counter, deque
from dataclasses import dataclass, field

import numpy as np


# --------------------------------------------------------------------------
# structure: partition (blocks.py:75-96), aux depth (blocks.py:99-106)
# --------------------------------------------------------------------------

def layer_params(dims, i):
    """blocks.py:53-55 — weights + bias of layer i."""
    return dims[i] * dims[i + 1] + dims[i + 1]


def partition(dims, s):
    """blocks.py:75-96 — contiguous minimax split of layer parameter counts;
    ``itertools.combinations`` order makes the first strict minimum the
    earliest-cut tie-break."""
    n = len(dims) - 1
    if s < 1 or s > n:
        raise ValueError(f"bad stage count {s} for {n} layers")
    costs = [layer_params(dims, i) for i in range(n)]
    best_cuts, best_load = None, math.inf
    for cuts in itertools.combinations(range(1, n), s - 1):
        edges = (0,) + cuts + (n,)
        load = max(sum(costs[a:b]) for a, b in zip(edges, edges[1:]))
        if load < best_load:
            best_load, best_cuts = load, cuts
    edges = (0,) + best_cuts + (n,)
    return tuple(zip(edges, edges[1:]))


def aux_depth(l, d_prime, n):
    """blocks.py:99-106 — max(0, d' - floor(l / n))."""
    return max(0, d_prime - l // n)


# --------------------------------------------------------------------------
# seeded init (blocks.py:190-237)
# --------------------------------------------------------------------------

@dataclass
class OracleStage:
    """One stage: list of (W, b, relu_after) for block then aux layers."""
    index: int
    block: list            # [(W [in,out], b [out], relu_after)]
    aux: list              # same, empty for the final stage
    momenta: list          # np arrays parallel to params()
    step_count: int = 0

    def params(self):
        out = []
        for W, b, _ in self.block + self.aux:
            out += [W, b]
        return out


def _init_layer(rng, fan_in, fan_out, relu_after):
    """blocks.py:190-195 — W ~ U(+-1/sqrt(fan_in)) drawn before b."""
    bound = 1.0 / math.sqrt(fan_in)
    W = rng.uniform(-bound, bound, size=(fan_in, fan_out))
    b = rng.uniform(-bound, bound, size=(fan_out,))
    return [W, b, relu_after]


def build_stages(dims, boundaries, d_prime, n, seed, aux_hidden_width=None):
    """blocks.py:198-237 — per-stage ``default_rng(seed + j)``; block layers,
    then aux layers; no aux head on the final stage; ReLU after every layer
    except the network's final layer and each aux classifier."""
    n_layers = len(dims) - 1
    classes = dims[-1]
    last = len(boundaries) - 1
    stages = []
    for j, (start, end) in enumerate(boundaries):
        rng = np.random.default_rng(seed + j)
        block = [_init_layer(rng, dims[i], dims[i + 1], i != n_layers - 1)
                 for i in range(start, end)]
        aux = []
        if j != last:
            assigned = aux_depth(j, d_prime, n)
            block_out = dims[end]
            hidden = aux_hidden_width or block_out
            widths = [block_out] + [hidden] * assigned + [classes]
            aux = [_init_layer(rng, widths[i], widths[i + 1], i != len(widths) - 2)
                   for i in range(len(widths) - 1)]
        st = OracleStage(j, block, aux, [])
        st.momenta = [np.zeros_like(p) for p in st.params()]
        stages.append(st)
    return stages


# --------------------------------------------------------------------------
# optimizer (optim.py:39-44, 71-89)
# --------------------------------------------------------------------------

def cosine_lr(step, lr0, lr_min, total_steps):
    """optim.py:39-44."""
    if step < 0 or step > total_steps:
        raise ValueError(f"step {step} outside [0, {total_steps}]")
    span = lr0 - lr_min
    return lr_min + 0.5 * span * (1.0 + math.cos(math.pi * step / total_steps))


def nesterov_update(theta, v, g, lr, mu, wd):
    """optim.py:81-88 — L2-in-gradient, lookahead-folded Nesterov; in place."""
    if wd != 0.0:
        g = g + wd * theta
    v *= mu
    v += g
    theta -= lr * (g + mu * v)


# --------------------------------------------------------------------------
# one local step (blocks.py:240-289; tensor.py:137-234)
# --------------------------------------------------------------------------

def _forward(layers, x):
    """blocks.py:240-246 — matmul, bias_add, relu; keep inputs for backward."""
    acts = [x]
    h = x
    for W, b, relu_after in layers:
        h = h @ W + b
        if relu_after:
            h = np.maximum(h, 0.0)
        acts.append(h)
    return h, acts


def softmax_xent(z, y):
    """tensor.py:201-234 — mean CE with max subtraction; returns (loss, dz)."""
    B, C = z.shape
    y = np.asarray(y)
    if y.min() < 0 or y.max() >= C:
        raise ValueError("label out of range")
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    denom = e.sum(axis=1, keepdims=True)
    logp = (z - m) - np.log(denom)
    loss = -logp[np.arange(B), y].mean()
    gz = e / denom
    gz[np.arange(B), y] -= 1.0
    return float(loss), gz * (1.0 / B)


def _backward(layers, acts, g, first_input_detached=True):
    """Reverse replay of tensor.py:137-180 adjoints: bias grad = row sum,
    dW = x^T g, dx = g W^T masked by the producing ReLU (x > 0; 0 at 0)."""
    grads = [None] * (2 * len(layers))
    for li in reversed(range(len(layers))):
        W, b, relu_after = layers[li]
        if relu_after:
            g = g * (acts[li + 1] > 0.0)
        x = acts[li]
        grads[2 * li] = x.T @ g
        grads[2 * li + 1] = g.sum(axis=0)
        if li > 0 or not first_input_detached:
            g = g @ W.T
    return grads, g


def local_step(stage, x, y, lr0, lr_min, total_steps, mu, wd):
    """blocks.py:266-289 — forward, detach (x_out is pre-update), aux forward,
    softmax-CE, backward, cosine_lr(step_count), Nesterov over all params.
    Returns (loss, x_out, logits)."""
    h, acts_b = _forward(stage.block, x)
    x_out = h.copy()
    if stage.aux:
        logits, acts_a = _forward(stage.aux, h)
    else:
        logits, acts_a = h, [h]
    loss, gz = softmax_xent(logits, y)
    layers = stage.block + stage.aux
    acts = acts_b + acts_a[1:]
    grads, _ = _backward(layers, acts, gz)
    lr = cosine_lr(stage.step_count, lr0, lr_min, total_steps)
    for p, v, g in zip(stage.params(), stage.momenta, grads):
        nesterov_update(p, v, g, lr, mu, wd)
    stage.step_count += 1
    return loss, x_out, logits


def sequential_ppll(stages, batches, lr0, lr_min, total_steps, mu, wd):
    """The sequential local-learning schedule: for each batch,
    for each stage in order.  Bitwise equal to every PPLL schedule because each
    stage consumes FIFO and pushes before its update (blocks.py:279-288)."""
    losses = [[] for _ in stages]
    for x, y in batches:
        h = np.asarray(x, dtype=np.float64)
        for j, st in enumerate(stages):
            loss, h, _ = local_step(st, h, y, lr0, lr_min, total_steps, mu, wd)
            losses[j].append(loss)
    return losses


def e2e_step(stages, x, y, lr0, lr_min, total_steps, mu, wd):
    """The paper's baselines E2E (runtime.py:248-284) and naive PP
    (runtime.py:359-382, 423-465), which compute the same numbers: block
    forward through every stage, the task loss on the final stage's output
    (no aux heads), backward through all blocks with the boundary gradients
    flowing stage to stage (no dX into the network input), then the
    cosine-LR Nesterov step over each stage's BLOCK parameters only; every
    stage's step_count advances.  Returns the loss."""
    h = np.asarray(x, dtype=np.float64)
    acts = []
    for st in stages:
        h, a = _forward(st.block, h)
        acts.append(a)
    loss, g = softmax_xent(h, y)
    grads = [None] * len(stages)
    for j in reversed(range(len(stages))):
        grads[j], g = _backward(stages[j].block, acts[j], g, first_input_detached=(j == 0))
    for j, st in enumerate(stages):
        lr = cosine_lr(st.step_count, lr0, lr_min, total_steps)
        nb = 2 * len(st.block)
        for p, v, gg in zip(st.params()[:nb], st.momenta[:nb], grads[j]):
            nesterov_update(p, v, gg, lr, mu, wd)
        st.step_count += 1
    return loss


# --------------------------------------------------------------------------
# deterministic round-robin scheduler bookkeeping (runtime.py:475-533)
# --------------------------------------------------------------------------

@dataclass
class RoundRobinTrace:
    rounds: int = 0
    batches_processed: list = field(default_factory=list)
    staleness: Counter = field(default_factory=Counter)
    high_water: list = field(default_factory=list)
    order: list = field(default_factory=list)   # (round, stage, batch_id)


def roundrobin_trace(n_stages, n_batches, capacity):
    """runtime.py:475-533 with the compute elided: integer bookkeeping only
    (source top-up to M, stage j runs iff input non-empty and downstream has
    room, staleness vs producer_progress, high water, virtual wall = rounds)."""
    s, M = n_stages, capacity
    bufs = [deque() for _ in range(s)]
    closed = [False] * s
    progress = [-1] * s
    done = [False] * s
    next_id = 0
    tr = RoundRobinTrace(batches_processed=[0] * s, high_water=[0] * s)
    while not all(done):
        tr.rounds += 1
        while next_id <= n_batches and len(bufs[0]) < M:
            if next_id == n_batches:
                closed[0] = True
                next_id += 1
                break
            progress[0] = next_id
            bufs[0].append(next_id)
            tr.high_water[0] = max(tr.high_water[0], len(bufs[0]))
            next_id += 1
        for j in range(s):
            if done[j]:
                continue
            if not bufs[j]:
                if closed[j]:
                    done[j] = True
                    if j < s - 1:
                        closed[j + 1] = True
                continue
            last = j == s - 1
            if not last and len(bufs[j + 1]) >= M:
                continue
            bid = bufs[j].popleft()
            tr.staleness[max(0, progress[j] - bid)] += 1
            if not last:
                progress[j + 1] = bid
                bufs[j + 1].append(bid)
                tr.high_water[j + 1] = max(tr.high_water[j + 1], len(bufs[j + 1]))
            tr.order.append((tr.rounds, j, bid))
            tr.batches_processed[j] += 1
    return tr
