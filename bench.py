"""PPLL throughput benchmark (BASELINE.json metric: images/sec training,
device-timed, at 1/2/4/8 B200, plus the pipeline idle fraction).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                    [--workload vit_s|mlp_m]

Workloads (BASELINE.json configs):
  vit_s  (default, configs[1]) ViT-small: patch 4, depth 8, D=384, 6 heads,
         MLP 1536, CIFAR-shaped 3x32x32, batch 128, split into 4
         gradient-isolated blocks of 2 layers, aux head = N_l transformer
         layers (d'=1, n=3) + LN + classifier.
  mlp_m  the reference-runnable MLP analog 3072-1024x4-10, 4 stages, d'=2,
         n=3, batch 128 (SURVEY §8 'M').

One "step" = one synthetic batch pushed through every stage's local step
(forward -> push -> aux -> softmax-CE -> backward -> cosine-LR Nesterov).
``value`` is device-timed (CUDA events) with inputs already resident in HBM
(a 64-batch pool cycled; per-step working set > 126 MB L2, no flush);
``e2e`` is the same metric through the public API (``run_epoch`` on host
numpy batches: pinned staging + H2D inside the timed region, loss history
D2H).  ``--impl reference`` times the reference algorithm's CPU path (the
numpy oracle port in oracle/) on the host cores.

Multi-GPU (torchrun, one rank per GPU): round 1 runs independent replicas of
the whole stage pipeline per GPU (weak scaling); the NVLink stage-sharded
pipeline is the next milestone.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "vit_s": dict(kind="vit", spec=dict(image=32, channels=3, patch=4, dim=384, heads=6,
                                        mlp=1536, depth=8, classes=10),
                  s=4, d_prime=1, interval=3, batch=128),
    # configs[0]: ResNet-32 / 4 blocks, CIFAR-shaped, batch 128
    "resnet32": dict(kind="resnet", spec=dict(n=5, image=32, channels=3, widths=(16, 32, 64),
                                              classes=10),
                     s=4, d_prime=1, interval=3, batch=128, data_shape="CIFAR-10",
                     split="cost"),
    # configs[2]: ResNet-110 / 8 blocks, SVHN-shaped, batch 256
    "resnet110": dict(kind="resnet", spec=dict(n=18, image=32, channels=3, widths=(16, 32, 64),
                                               classes=10),
                      s=8, d_prime=1, interval=3, batch=256, data_shape="SVHN",
                      split="cost"),
    # configs[3]: ViT-base / 8 blocks, STL-10-shaped 96x96, patch 16 (T = 37), batch 128
    "vit_b": dict(kind="vit", spec=dict(image=96, channels=3, patch=16, dim=768, heads=12,
                                        mlp=3072, depth=12, classes=10),
                  s=8, d_prime=1, interval=3, batch=128, data_shape="STL-10"),
    "mlp_m": dict(kind="mlp", dims=(3072, 1024, 1024, 1024, 1024, 10), s=4, d_prime=2,
                  interval=3, batch=128),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML every
    10 ms (a first sample at entry), nvidia-smi every 200 ms if NVML is absent."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append([str(sm), str(mx)] +
                         ["Active" if bits & b else "Not Active" for b in self.BITS])

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self._sample_nvml()
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.01 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def vit_depths(wl):
    """Layers per ViT block: cost-balanced (``balanced_vit_depths``: block
    layers + aux head + patch embedding per stage) unless the workload says
    ``split="even"``."""
    from paper_2411_12780_b200.vit import VitSpec, balanced_depths, balanced_vit_depths
    spec = VitSpec(**wl["spec"])
    if wl.get("split", "cost") == "even":
        return balanced_depths(spec.depth, wl["s"])
    return balanced_vit_depths(spec, wl["s"], wl["d_prime"], wl["interval"])


def resnet_blocks(wl):
    from paper_2411_12780_b200.resnet import ResNetSpec, balanced_resnet_split, resnet_split
    spec = ResNetSpec(**wl["spec"])
    if wl.get("split", "even") == "cost":
        return balanced_resnet_split(spec, wl["s"], wl["d_prime"], wl["interval"])
    return resnet_split(spec, wl["s"])


def describe(wl, name):
    if wl["kind"] == "resnet":
        sp = wl["spec"]
        return (f"{name}: PPLL ResNet-{6 * sp['n'] + 2} (CIFAR basic blocks 16/32/64, option-B "
                f"shortcut, train-mode BN), {wl['s']} gradient-isolated blocks, aux = "
                f"aux_depth(l,{wl['d_prime']},{wl['interval']}) conv3x3-BN-ReLU + GAP + linear, "
                f"{wl['data_shape']}-shaped {sp['image']}x{sp['image']}x3 NHWC, batch {wl['batch']}")
    if wl["kind"] == "vit":
        sp = wl["spec"]
        size = "base" if sp["dim"] >= 768 else "small"
        return (f"{name}: PPLL ViT-{size}/{sp['patch']} depth {sp['depth']} D={sp['dim']} "
                f"heads={sp['heads']} MLP={sp['mlp']}, {wl['s']} gradient-isolated blocks "
                f"(layers {vit_depths(wl)}), aux = aux_depth(l,"
                f"{wl['d_prime']},{wl['interval']}) transformer layers + LN + classifier, "
                f"{wl.get('data_shape', 'CIFAR-10')}-shaped {sp['channels']}x{sp['image']}x"
                f"{sp['image']}, {sp['classes']} classes, batch {wl['batch']}")
    return (f"{name}: PPLL MLP {'-'.join(map(str, wl['dims']))}, {wl['s']} gradient-isolated "
            f"stages, d'={wl['d_prime']}, n={wl['interval']}, CIFAR-shaped 3x32x32 inputs, "
            f"batch {wl['batch']}")


def cfg_dict(wl, args):
    extra = {}
    if wl["kind"] == "resnet":
        extra["stage_split"] = (f"{wl.get('split', 'even')} split, blocks per stage "
                                f"{[len(b) for b in resnet_blocks(wl)]} (stem on stage 0)")
    elif wl["kind"] == "vit":
        extra["stage_split"] = f"{wl.get('split', 'cost')} split, layers per stage {vit_depths(wl)}"
    return extra | {"workload": describe(wl, args.workload),
            "global_batch": wl["batch"], "stages": wl["s"], "d_prime": wl["d_prime"],
            "buffer_capacity": args.capacity, "precision": args.precision,
            "placement": "all stages on one GPU, one CUDA stream per stage",
            "l2": "no flush between steps; per-step working set (64-batch resident input "
                  "pool + per-stage params/momenta/grads/activations) exceeds the 126 MB L2"}


def bench_phases(steps: int, warmup: int, s: int) -> dict:
    """Local steps every module takes in one N=1 bench run, phase by phase
    (main() consumes exactly these; the cosine-LR horizon ``total_steps`` is
    sized from them — cosine_lr raises StepOutOfRange past it, optim.py:39-44)."""
    return {"warmup": warmup, "launch_probe": 1, "timed": steps, "sequential_warmup": 3,
            "sequential": max(10, steps // 3), "e2e_warmup": 2 * s + 2,
            "e2e": max(100, steps)}


def sharded_phases(steps: int, warmup: int) -> dict:
    """The same for the N>1 (one process per GPU) path."""
    return {"warmup": warmup, "timed": steps, "e2e": max(60, steps)}


def step_budget(phases: dict) -> int:
    return sum(phases.values()) + 16


# ---------------------------------------------------------------------------
# the reference arm / CPU baseline: the reference algorithm on host cores
# ---------------------------------------------------------------------------

def cpu_reference(wl, n_batches, warmup=1, time_budget=None):
    """Images/s of the reference algorithm on the host cores, sequential
    local-learning schedule (bitwise the PPLL result), at the
    workload's full batch and stage split; the number of steps (not the
    batch) is time-bounded.  MLP: the numpy float64 oracle port of the
    reference (pinned to its golden vectors).  ViT / ResNet (no reference
    implementation exists): the torch-CPU fp32 restatement (oracle/torch_cpu.py,
    BASELINE.md §3), every host thread to torch's intra-op pool."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    cores = len(os.sched_getaffinity(0))
    torch.set_num_threads(cores)
    B = wl["batch"]
    rng = np.random.default_rng(0)
    if wl["kind"] == "mlp":
        import ppll_oracle as orc
        dims = wl["dims"]
        stages = orc.build_stages(dims, orc.partition(dims, wl["s"]), wl["d_prime"],
                                  wl["interval"], 42)
        data = [(rng.standard_normal((B, dims[0])), rng.integers(0, dims[-1], B))
                for _ in range(2)]
        kind = "numpy float64 oracle port of the reference (sequential schedule)"

        def step(x, y):
            orc.sequential_ppll(stages, [(x, y)], 0.05, 0.001, 10 ** 6, 0.9, 1e-4)
    else:
        import torch_cpu as tc
        if wl["kind"] == "resnet":
            import resnet_oracle as ro
            spec = ro.ResNetSpec(**wl["spec"])
            stages = [tc.from_resnet(st) for st in ro.build_resnet_stages(
                spec, wl["s"], wl["d_prime"], wl["interval"], 42, split=resnet_blocks(wl))]
            shape = (B, spec.image, spec.image, spec.channels)
        else:
            import vit_oracle as vo
            spec = vo.VitSpec(**wl["spec"])
            stages = [tc.from_vit(st) for st in vo.build_vit_stages(
                spec, vit_depths(wl), wl["d_prime"], wl["interval"], 42)]
            shape = (B, spec.channels, spec.image, spec.image)
        data = [(torch.tensor(rng.standard_normal(shape), dtype=torch.float32),
                 rng.integers(0, spec.classes, B)) for _ in range(2)]
        kind = "torch-CPU fp32 restatement (oracle/torch_cpu.py, sequential schedule)"

        def step(x, y):
            h = x
            for st in stages:
                _, h, _ = tc.local_step(st, h, y, 0.05, 0.001, 10 ** 6, 0.9, 1e-4)
    for i in range(warmup):
        step(*data[i % 2])
    t0 = time.perf_counter()
    done = 0
    for i in range(n_batches):
        step(*data[i % 2])
        done += 1
        if time_budget and time.perf_counter() - t0 > time_budget:
            break
    dt = time.perf_counter() - t0
    return {"value": done * B / dt, "unit": "images/s", "cores": cores, "kind": "port",
            "sample": f"{done} steps x batch {B} through all {wl['s']} stages, {kind}, "
                      f"{cores} threads, {dt:.1f} s",
            "steps": done, "seconds": dt, "dtype": "f64" if wl["kind"] == "mlp" else "fp32"}


def run_reference_arm(args, wl, rank):
    if rank != 0:
        return
    warm = min(args.warmup, 1)
    cpu = cpu_reference(wl, args.steps, warmup=warm, time_budget=120.0)
    ips = cpu["value"]
    line = {
        "impl": "reference", "metric": "images/sec training (device-timed) at 1/2/4/8 B200; "
        "pipeline idle fraction", "value": ips, "unit": "images/s",
        "n_gpus": args.gpus, "steps": cpu["steps"], "warmup": warm,
        "ms_per_step": 1e3 * cpu["seconds"] / max(cpu["steps"], 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cpu["dtype"], "data": "synthetic",
        "config": cfg_dict(wl, args),
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": ips, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def build(wl, precision, device, total_steps):
    import paper_2411_12780_b200 as lp
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=total_steps, seed=42,
                           precision=precision)
    if wl["kind"] == "mlp":
        spec = lp.NetworkSpec(wl["dims"])
        return lp.build_modules(spec, lp.partition(spec, wl["s"]), wl["d_prime"],
                                wl["interval"], hyper, devices=[device] * wl["s"])
    if wl["kind"] == "resnet":
        return lp.build_resnet_modules(lp.ResNetSpec(**wl["spec"]), wl["s"], wl["d_prime"],
                                       wl["interval"], hyper, devices=[device] * wl["s"],
                                       split=resnet_blocks(wl))
    spec = lp.VitSpec(**wl["spec"])
    return lp.build_vit_modules(spec, vit_depths(wl), wl["d_prime"],
                                wl["interval"], hyper, devices=[device] * wl["s"])


def sharded_stages(wl, world):
    """Stage count at N GPUs: the configured s, or N when N exceeds it (the
    paper's LPP: one block per GPU; ViT-S depth 8 on 8 GPUs = 1 layer/block)."""
    return max(wl["s"], world)


def run_sharded(args, wl, rank, world, local, dev):
    """N > 1: stages sharded over ranks (stage j on rank floor(j·N/s)),
    cross-GPU boundaries are CUDA-IPC rings written by the producer's epilogue
    over NVLink; device-timed, max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2411_12780_b200 as lp
    from paper_2411_12780_b200 import _native as N
    from paper_2411_12780_b200.distributed import (DistributedPipeline, gather_metrics,
                                                   stage_placement)
    s = sharded_stages(wl, world)
    placement = stage_placement(s, world)
    mine = [j for j in range(s) if placement[j] == rank]
    B = wl["batch"]
    total = step_budget(sharded_phases(args.steps, args.warmup))
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=total, seed=42,
                           precision=args.precision)
    if wl["kind"] == "mlp":
        spec = lp.NetworkSpec(wl["dims"])
        s = min(s, spec.n_layers)
        placement = stage_placement(s, world)
        mine = [j for j in range(s) if placement[j] == rank]
        mods = lp.build_modules(spec, lp.partition(spec, s), wl["d_prime"], wl["interval"],
                                hyper, devices=[dev] * s, only=mine)
    elif wl["kind"] == "resnet":
        spec = lp.ResNetSpec(**wl["spec"])
        mods = lp.build_resnet_modules(spec, s, wl["d_prime"], wl["interval"], hyper,
                                       split=resnet_blocks(dict(wl, s=s)),
                                       devices=[dev] * s, only=mine)
    else:
        spec = lp.VitSpec(**wl["spec"])
        mods = lp.build_vit_modules(spec, vit_depths(dict(wl, s=s)), wl["d_prime"],
                                    wl["interval"], hyper, devices=[dev] * s, only=mine)
    pipe = DistributedPipeline(mods, placement, rank, None, capacity=args.capacity, max_batch=B,
                               use_graphs=not args.no_graphs)
    in_shape = None
    if rank == placement[0]:
        in_shape = tuple(mods[0].in_shape)
    shapes = [None] * world
    dist.all_gather_object(shapes, in_shape)
    in_shape = next(x for x in shapes if x is not None)
    n_cls = wl["dims"][-1] if wl["kind"] == "mlp" else spec.classes
    gen = torch.Generator(device=dev).manual_seed(1234)
    pool = None
    if rank == placement[0]:
        pool = (torch.randn((64, B) + in_shape, device=dev, generator=gen),
                torch.randint(0, n_cls, (64, B), device=dev, generator=gen))

    def batches(k, off=0):
        if pool is None:
            return None
        return ((pool[0][(off + i) % 64], pool[1][(off + i) % 64]) for i in range(k))

    pipe.run(batches(args.warmup), args.warmup, B)
    launches0 = N.launch_count() + pipe.replayed_kernels
    dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        res = pipe.run(batches(args.steps, 11), args.steps, B)
    launches = N.launch_count() + pipe.replayed_kernels - launches0
    met = gather_metrics(res, s, args.steps, args.steps * B, None)
    errs = [None] * world
    dist.all_gather_object(errs, res["errors"])
    value = met.images / met.wall_time
    idle = met.idle_fraction
    # e2e: host numpy batches through the same sharded pipeline (rank 0 H2D)
    rng = np.random.default_rng(7)
    # inputs in pinned host memory (the contract's e2e: H2D from pinned buffers)
    host = [(torch.from_numpy(rng.standard_normal((B,) + in_shape).astype(np.float32)).pin_memory(),
             torch.from_numpy(rng.integers(0, n_cls, B)).pin_memory()) for _ in range(8)]
    e2e_steps = sharded_phases(args.steps, args.warmup)["e2e"]
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    r2 = pipe.run((host[i % 8] for i in range(e2e_steps)) if rank == placement[0] else None,
                  e2e_steps, B)
    m2 = gather_metrics(r2, s, e2e_steps, e2e_steps * B, None)
    e2e_dt = time.perf_counter() - t0
    dts = [None] * world
    dist.all_gather_object(dts, e2e_dt)
    e2e_dt = max(dts)
    launch_counts = [None] * world
    dist.all_gather_object(launch_counts, launches)
    xfer = _guard("boundary_transfer", boundary_transfer, pipe, mods, placement, rank, world, B,
                  dev)
    seq = None
    if rank == 0:
        seq = _guard("sequential_same_split", sequential_same_split, args, wl, s, dev, 40)
    roof = None
    if rank == 0:   # the dominant kernel, timed alone on rank 0's GPU (same as N = 1)
        hbm, tf_burst, _, peak_kind = peaks()
        if wl["kind"] == "vit":
            roof = _guard("roofline_gemm", roofline_gemm, wl, tf_burst, hbm, dev)
        elif wl["kind"] == "resnet" and args.precision == "bf16":
            roof = _guard("roofline_conv", roofline_conv, wl, tf_burst, hbm, dev)
        if isinstance(roof, dict):
            roof["peak_kind"] = peak_kind
    if rank == 0:
        line = {
            "metric": "images/sec training (device-timed) at 1/2/4/8 B200; pipeline idle fraction",
            "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * met.wall_time / args.steps,
            "higher_is_better": True, "scaling": "strong" if s == wl["s"] else "weak",
            "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (seeded N(0,1) CIFAR-shaped inputs, uniform labels; "
                    "random-init weights drawn like the reference)",
            "config": cfg_dict(dict(wl, s=s), args) | {
                "global_batch": B, "stages": s, "placement": f"stage->rank {placement}",
                "parallelism": f"pp{world} (PPLL stages sharded over GPUs; CUDA-IPC rings, "
                               f"producer epilogue stores over NVLink)"},
            "idle_fraction": {"per_stage": [round(x, 4) for x in idle],
                              "mean": round(sum(idle) / len(idle), 4)},
            "e2e": {"value": e2e_steps * B / e2e_dt, "unit": "images/s",
                    "h2d_bytes_per_step": B * int(np.prod(in_shape)) * 4 + B * 8,
                    "d2h_bytes_per_step": 4 * s,
                    "api": "DistributedPipeline.run on pinned host batches (rank 0 H2D)"},
            "roofline": roof, "cpu_baseline": None,
            "sequential_same_split": seq,
            "boundary_transfer": xfer,
            "gpu_launches": int(sum(launch_counts)),
            "clocks": clk.summary(),
            "stage_errors": errs,
            "final_losses": [h[-1] if h else None for h in met.loss_history],
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    pipe.close()
    dist.destroy_process_group()


def boundary_transfer(pipe, mods, placement, rank, world, B, dev, reps=50):
    """Queue-transfer evidence for the N > 1 line (north_star: "NVLink GB/s for
    queue transfers"; SURVEY §8e baseline "ncclSend/ncclRecv on a comm
    stream").  For every cross-rank boundary j -> j+1 the producer moves one
    ring slot's payload (B x features activation + B int64 labels) to the
    consumer's ring, all boundaries concurrently, ``reps`` times:
      * ``p2p_ring``: a copy into the consumer's CUDA-IPC-mapped slot (the
        path the pipeline's fused epilogue stores take, over NVLink);
      * ``nccl``: torch.distributed NCCL isend/irecv of the same bytes (the
        baseline), through a separate NCCL group.
    Device-timed with CUDA events, max over ranks; GB/s per boundary."""
    import torch
    import torch.distributed as dist
    from paper_2411_12780_b200 import _native as N
    lib = N.load()
    s = len(placement)
    cross = [j for j in range(s - 1) if placement[j] != placement[j + 1]]
    if not cross:
        return None
    feat = {}
    for j in cross:
        if placement[j] == rank:
            feat[j] = mods_by_stage(mods)[j].out_features
    sizes = [None] * world
    dist.all_gather_object(sizes, feat)
    allfeat = {}
    for d in sizes:
        allfeat.update(d)
    esz = 2 if mods[0].precision == "bf16" else 4
    nbytes = {j: B * allfeat[j] * esz + 8 * B for j in cross}
    out = {"boundaries": cross, "bytes_per_boundary": nbytes, "reps": reps}
    st = torch.cuda.current_stream(dev)

    def timed(fn):
        fn()                                                  # warm-up
        torch.cuda.synchronize(dev)
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        b.synchronize()
        t = [None] * world
        dist.all_gather_object(t, a.elapsed_time(b) / 1e3)
        return max(t)

    # (1) the IPC ring: producer copies into the peer-mapped slot
    src = {j: torch.empty(nbytes[j], dtype=torch.uint8, device=dev)
           for j in cross if placement[j] == rank}

    def p2p():
        for j, buf in src.items():
            N.check(lib.ppll_copy_async(pipe.x_peer[j + 1], buf.data_ptr(), nbytes[j],
                                        st.cuda_stream), "p2p copy")
    try:
        t = timed(p2p)
        out["p2p_ring"] = {"seconds": t, "GBps_per_boundary": {
            str(j): nbytes[j] * reps / t / 1e9 for j in cross},
            "path": "cudaMemcpyAsync into the consumer's CUDA-IPC-mapped ring slot"}
    except Exception as e:                                     # noqa: BLE001
        out["p2p_ring"] = {"error": f"{type(e).__name__}: {e}"}
    # (2) the NCCL baseline
    try:
        g = dist.new_group(backend="nccl")
        dst = {j: torch.empty(nbytes[j], dtype=torch.uint8, device=dev)
               for j in cross if placement[j + 1] == rank}

        def nccl():
            ops = []
            for j in cross:
                if placement[j] == rank:
                    ops.append(dist.P2POp(dist.isend, src[j], placement[j + 1], g))
                if placement[j + 1] == rank:
                    ops.append(dist.P2POp(dist.irecv, dst[j], placement[j], g))
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        t = timed(nccl)
        out["nccl_sendrecv"] = {"seconds": t, "GBps_per_boundary": {
            str(j): nbytes[j] * reps / t / 1e9 for j in cross},
            "path": "torch.distributed batch_isend_irecv over an NCCL group"}
    except Exception as e:                                     # noqa: BLE001
        out["nccl_sendrecv"] = {"error": f"{type(e).__name__}: {e}"}
    return out


def backprop_baselines(wl, args, dev, batches, ppll_ips):
    """The paper's baselines on the same GPU and workload (reference
    runtime.py:248-284 E2E, :359-382 NaivePP): end-to-end backprop through all
    blocks on one stream, and the same computation as a naive pipeline (one
    stream per stage; stage j's forward of batch t+1 waits for its backward of
    t — the bubble PPLL removes).  Fresh modules (own cosine horizon);
    device-timed by the run's CUDA events (EpochMetrics.wall_time)."""
    import torch
    import paper_2411_12780_b200 as lp
    n, w = max(10, args.steps // 2), 3
    mods = build(wl, args.precision, dev, 2 * (n + w) + 16)
    cfg = lp.RunConfig(buffer_capacity=args.capacity, timing=True)
    out = {}
    for mode, key in ((lp.RunMode.E2E, "e2e_backprop_images_per_s"),
                      (lp.RunMode.NAIVE_PP, "naive_pp_images_per_s")):
        lp.run_epoch(mode, mods, batches(w, 21), cfg)
        torch.cuda.synchronize(dev)
        met = lp.run_epoch(mode, mods, batches(n, 25), cfg)
        out[key] = met.images / met.wall_time
    out["ppll_over_naive_pp"] = ppll_ips / out["naive_pp_images_per_s"]
    out["note"] = ("same GPU, same batches; E2E on one stream, naive PP one stream per stage "
                   "(the paper compares PPLL / PP on one GPU per stage)")
    for m in mods:
        m.close()
    return out


def mods_by_stage(mods):
    return {m.stage_index: m for m in mods}


def sequential_same_split(args, wl, s, dev, steps):
    """The paper's S=1 reference for the SAME s-stage split the sharded run
    uses (all stages on one stream of rank 0's GPU): the speed-up at N GPUs is
    value / this, model split held fixed (an s=8 sequential
    baseline whenever N=8 switches to LPP)."""
    import torch
    import paper_2411_12780_b200 as lp
    wl_s = dict(wl, s=s)
    mods = build(wl_s, args.precision, dev, steps + 16)
    B = wl["batch"]
    in_shape = tuple(mods[0].in_shape)
    gen = torch.Generator(device=dev).manual_seed(99)
    pool_x = torch.randn((8, B) + in_shape, device=dev, generator=gen)
    pool_y = torch.randint(0, mods[-1].num_classes, (8, B), device=dev, generator=gen)
    seq = lp.DevicePipeline(mods, lp.RunConfig(buffer_capacity=args.capacity,
                                               use_graphs=not args.no_graphs, timing=False))
    cur = torch.cuda.current_stream(dev)
    seq.streams = [cur] * len(mods)
    seq.src_stream = cur
    seq.run((pool_x[i % 8], pool_y[i % 8]) for i in range(3))
    torch.cuda.synchronize(dev)
    n = max(10, steps - 3)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    seq.run((pool_x[i % 8], pool_y[i % 8]) for i in range(n))
    b.record()
    b.synchronize()
    for m in mods:
        m.close()
    return {"images_per_s": n * B / (a.elapsed_time(b) * 1e-3), "stages": s,
            "placement": "all stages on one stream of rank 0's GPU"}


def _time_kernel(fn, dev, reps=20):
    """Mean CUDA-event duration of fn() on torch's current stream with a cold
    L2: every launch follows a read of a 512 MB buffer (clean lines, so the
    timed kernel does not pay for write-backs of a dirty flush).  Events
    bracket the whole loop of (flush, kernel) pairs and the same loop of
    flushes alone; the per-launch time is the difference / reps (single-launch
    event pairs are too coarse for 10-20 us kernels)."""
    import torch
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)
    for _ in range(3):
        fn(st.cuda_stream)

    def loop(with_kernel):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            torch.sum(flush, dim=(0,), out=sink[0])
            if with_kernel:
                fn(st.cuda_stream)
        b.record(st)
        b.synchronize()
        return a.elapsed_time(b)

    loop(True)
    both = min(loop(True) for _ in range(3))
    alone = min(loop(False) for _ in range(3))
    return max(both - alone, 1e-6) / reps * 1e-3


def engine_calibration(tf_burst, dev):
    """The same tcgen05 engine on a large square GEMM (8192^3, bf16 fwd):
    what it reaches when the problem is big enough to amortise its fixed
    per-launch cost (the ViT-S layer GEMMs are 2.5-10 GFLOP each)."""
    import torch
    from paper_2411_12780_b200 import _native as N
    n = 8192
    X = torch.randn(n, n, device=dev).bfloat16()
    W = (torch.randn(n, n, device=dev) * 0.01).bfloat16()
    Y = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    lib = N.load()
    dt = _time_kernel(lambda s: lib.ppll_linear_fwd(n, n, n, X.data_ptr(), n, W.data_ptr(), None,
                                                    Y.data_ptr(), n, None, 0, 0, N.BF16, s),
                      dev, reps=10)
    fl = 2.0 * n ** 3
    return {"gemm": f"{n}x{n}x{n} fwd", "us": round(dt * 1e6, 1),
            "tflops": round(fl / dt / 1e12, 1), "tensor_frac": round(fl / dt / 1e12 / tf_burst, 3)}


def roofline_nesterov(mods, hbm, dev):
    """Fused Nesterov update of the largest stage (HBM-bound, 22 B/param)."""
    import torch
    from paper_2411_12780_b200 import _native as N
    m = max(mods, key=lambda mm: mm._flat["theta"].numel())
    f = m._flat
    n = f["theta"].numel()
    lib = N.load()
    g = torch.zeros_like(f["grad"])
    th, v = f["theta"].clone(), f["mom"].clone()
    lpb = f["theta_lp"].clone() if f["theta_lp"] is not None else None
    dt = _time_kernel(lambda s: lib.ppll_nesterov_step(n, th.data_ptr(), v.data_ptr(),
                                                       g.data_ptr(), N.ptr(lpb), None, None, 0,
                                                       0.0, 0.9, 1e-4, None, s), dev)
    per = 20 + (2 if lpb is not None else 0)
    return {"kernel": "nesterov_kernel (fused Nesterov-SGD over the largest stage's flat "
                      "parameter buffer)", "bound": "hbm", "achieved": n * per / dt / 1e9,
            "peak": hbm, "unit": "GB/s", "frac": n * per / dt / 1e9 / hbm,
            # the committed capture is of ResNet-32's largest stage (373,056 params)
            "traffic": _traffic_of("nesterov_kernel") if (n == 373056 and lpb is not None) else None,
            "algorithmic_bytes_per_launch": n * per, "params": n, "bytes_per_param": per,
            "launch_us": dt * 1e6}


def roofline_attention(wl, hbm, dev, sets=4, reps=5):
    """Second roofline entry of the ViT line: the tcgen05 attention kernels
    (attn_tc_fwd_kernel / the persistent attn_tc_bwd_kernel) at the workload's
    geometry.  `sets` independent input/output sets (~45 MB each for the
    backward, > L2 together) are cycled by back-to-back launches captured in a
    CUDA graph (PDL edges, as in the stage graphs), so every launch reads
    inputs the previous launches did not leave in L2; per-launch time = graph
    time / launches.  HBM-bound: algorithmic bytes = qkv read + o (+ lse)
    written (forward); qkv, o, dO (+ lse) read + dqkv (+ the fused bias
    partials) written (backward)."""
    import torch
    from paper_2411_12780_b200 import _native as N
    sp = wl["spec"]
    B, T = wl["batch"], (sp["image"] // sp["patch"]) ** 2 + 1
    H = sp["heads"]
    D = 64 * H
    M = B * T
    geo_vit_s = (B, T, H) == (128, 65, 6)   # the geometry of profiles/r02_ncu_traffic.csv
    lib = N.load()
    bufs = []
    for _ in range(sets):
        qkv = (torch.randn(M, 3 * D, device=dev) * 0.5).bfloat16()
        bufs.append(dict(qkv=qkv, dout=(torch.randn(M, D, device=dev) * 0.5).bfloat16(),
                         o=torch.empty(M, D, device=dev, dtype=torch.bfloat16),
                         lse=torch.empty(B * H * T, device=dev), dqkv=torch.empty_like(qkv),
                         bias=torch.empty(B, 3 * D, device=dev)))
    st = torch.cuda.Stream(dev)

    def fwd(bf, s):
        lib.ppll_attn_fwd_bf16(B, T, H, bf["qkv"].data_ptr(), bf["o"].data_ptr(),
                               bf["lse"].data_ptr(), s)

    def bwd(bf, s):
        lib.ppll_attn_bwd_bf16(B, T, H, bf["qkv"].data_ptr(), bf["o"].data_ptr(),
                               bf["dout"].data_ptr(), bf["lse"].data_ptr(), bf["dqkv"].data_ptr(),
                               bf["bias"].data_ptr(), s)

    def per_launch(fn):
        with torch.cuda.stream(st):
            for bf in bufs:
                fn(bf, st.cuda_stream)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                for bf in bufs:
                    fn(bf, st.cuda_stream)
        with torch.cuda.stream(st):
            g.replay()
        torch.cuda.synchronize(dev)
        best = float("inf")
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):      # replay on the stream the events bracket
                a.record(st)
                g.replay()
                b.record(st)
            b.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3 / (reps * len(bufs)))
        return best

    t_f = per_launch(fwd)
    t_b = per_launch(bwd)
    # the same launches on one resident input set (inputs in L2, as when the
    # attention directly follows the GEMM that produced its inputs)
    bufs = bufs[:1]
    w_f, w_b = per_launch(fwd), per_launch(bwd)
    by_f = 2 * M * 3 * D + 2 * M * D + 4 * B * H * T
    by_b = 2 * M * 3 * D + 2 * 2 * M * D + 4 * B * H * T + 2 * M * 3 * D + 4 * B * 3 * D
    return {"kernel": "attn_tc_bwd_kernel (persistent, one CTA per resident slot; the ViT "
                      "layer's attention backward), back-to-back launches over "
                      f"{sets} input sets (> L2) from one CUDA graph",
            "bound": "hbm", "achieved": by_b / t_b / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": by_b / t_b / 1e9 / hbm,
            "traffic": _traffic_of("attn_tc_bwd") if geo_vit_s else None,
            "traffic_source": "profiles/r02_ncu_traffic.csv (ViT-S geometry only)",
            "algorithmic_bytes_per_launch": by_b, "launch_us": t_b * 1e6,
            "geometry": {"batch": B, "tokens": T, "heads": H, "head_dim": 64},
            "forward": {"kernel": "attn_tc_fwd_kernel", "achieved": by_f / t_f / 1e9,
                        "frac": by_f / t_f / 1e9 / hbm, "algorithmic_bytes_per_launch": by_f,
                        "traffic": _traffic_of("attn_tc_fwd") if geo_vit_s else None,
                        "launch_us": t_f * 1e6},
            "warm_l2": {"how": "same graph on one input set (L2-resident inputs)",
                        "bwd_launch_us": w_b * 1e6, "bwd_frac": by_b / w_b / 1e9 / hbm,
                        "fwd_launch_us": w_f * 1e6, "fwd_frac": by_f / w_f / 1e9 / hbm}}


def vit_layer_gemms(wl, dev):
    """The 12 tcgen05 GEMM launches of one ViT transformer layer's local step
    (vit_stage.cu: forward QKV / proj / FC1 / FC2, dgrad and wgrad of each) at
    the workload's batch, with the step's exact fused epilogues, as callables
    on a stream plus their algorithmic FLOPs and bytes (operands read once,
    outputs written once, epilogue side inputs read once)."""
    import torch
    from paper_2411_12780_b200 import _native as N
    sp = wl["spec"]
    M = wl["batch"] * ((sp["image"] // sp["patch"]) ** 2 + 1)
    D, F = sp["dim"], sp["mlp"]
    lib = N.load()
    g = torch.Generator(device=dev).manual_seed(0)
    bf = lambda *sh: (torch.randn(*sh, device=dev, generator=g) * 0.5).bfloat16()  # noqa: E731
    keep = []
    out = []

    def t(*sh):
        x = bf(*sh)
        keep.append(x)
        return x

    def fwd(name, K, Nn, act, res, pre, dual=False):
        X, W, Y = t(M, K), t(K, Nn), t(M, Nn)
        b = torch.zeros(Nn, device=dev)
        R = t(M, Nn) if res else None
        P = t(M, Nn) if pre else None
        Y2 = t(M, Nn) if dual else None
        keep.append(b)
        by = 2 * (M * K + K * Nn + M * Nn * (1 + (res is True) + (pre is True) + dual)) + 4 * Nn
        out.append((name, 2.0 * M * K * Nn, by, lambda s: lib.ppll_linear_fwd_ex(
            M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(), N.ptr(R), Nn, act, N.ptr(P),
            Nn, Y.data_ptr(), Nn, N.ptr(Y2), Nn, N.BF16, s)))

    def dgrad(name, K, Nn, mask_mode):
        dY, W, dX = t(M, Nn), t(K, Nn), t(M, K)
        Mk = t(M, K) if mask_mode else None
        by = 2 * (M * Nn + K * Nn + M * K * (1 + (mask_mode != 0)))
        out.append((name, 2.0 * M * K * Nn, by, lambda s: lib.ppll_linear_dgrad_ex(
            M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(), N.ptr(Mk), K, mask_mode, dX.data_ptr(),
            K, N.BF16, s)))

    def wgrad(name, K, Nn):
        X, dY = t(M, K), t(M, Nn)
        dW = torch.empty(K, Nn, device=dev)
        keep.append(dW)
        by = 2 * (M * K + M * Nn) + 4 * K * Nn
        out.append((name, 2.0 * M * K * Nn, by, lambda s: lib.ppll_linear_wgrad(
            M, K, Nn, X.data_ptr(), K, dY.data_ptr(), Nn, dW.data_ptr(), None, N.BF16, s)))

    fwd(f"qkv fwd {M}x{D}x{3 * D} +bias", D, 3 * D, 0, False, False)
    fwd(f"proj fwd {M}x{D}x{D} +bias+residual", D, D, 0, True, False)
    fwd(f"fc1 fwd {M}x{D}x{F} +bias, GELU, gelu' store", D, F, 3, False, True)
    fwd(f"fc2 fwd {M}x{F}x{D} +bias+residual", F, D, 0, True, False)
    dgrad(f"fc2 dgrad {M}x{F}x{D} *gelu'", F, D, 3)
    dgrad(f"fc1 dgrad {M}x{D}x{F}", D, F, 0)
    dgrad(f"proj dgrad {M}x{D}x{D}", D, D, 0)
    dgrad(f"qkv dgrad {M}x{D}x{3 * D}", D, 3 * D, 0)
    wgrad(f"fc2 wgrad {F}x{D} over {M}", F, D)
    wgrad(f"fc1 wgrad {D}x{F} over {M}", D, F)
    wgrad(f"proj wgrad {D}x{D} over {M}", D, D)
    wgrad(f"qkv wgrad {D}x{3 * D} over {M}", D, 3 * D)
    return out, keep


def _ncu_traffic(tag):
    """Per-launch DRAM bytes of the layer GEMMs from the committed ncu capture
    (profiles/r01_ncu_vit_layer_gemms.csv: dram__bytes_read.sum +
    dram__bytes_write.sum, one row per launch in vit_layer_gemms order)."""
    path = os.path.join(ROOT, "profiles", "r01_ncu_vit_layer_gemms.csv")
    try:
        import csv
        rows = [r for r in csv.reader(open(path)) if len(r) > 12]
        hdr = next(r for r in rows if "Metric Name" in r)
        vals = {}
        for r in rows:
            if r is hdr:
                continue
            d = dict(zip(hdr, r))
            if d.get("Metric Name") not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                continue
            if "gemm_tc" not in d.get("Kernel Name", ""):   # input set-up kernels
                continue
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1)
            key = int(d["ID"])
            vals[key] = vals.get(key, 0.0) + float(d["Metric Value"].replace(",", "")) * scale
        return [vals[k] for k in sorted(vals)]
    except Exception:
        return None


def _ncu_launch_traffic(fname="r02_ncu_traffic.csv"):
    """[(kernel name, dram read + write bytes)] per launch, in launch order, from
    a committed `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` CSV
    (profiles/r02_ncu_traffic.csv: tools/traffic_probe.py, one launch of each
    roofline kernel at the bench geometry, caches flushed before each)."""
    path = os.path.join(ROOT, "profiles", fname)
    try:
        import csv
        rows = [r for r in csv.reader(open(path)) if len(r) > 12]
        hdr = next(r for r in rows if "Metric Name" in r)
        vals, names = {}, {}
        for r in rows:
            if r is hdr:
                continue
            d = dict(zip(hdr, r))
            if d.get("Metric Name") not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                continue
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1)
            key = int(d["ID"])
            names[key] = d.get("Kernel Name", "")
            vals[key] = vals.get(key, 0.0) + float(d["Metric Value"].replace(",", "")) * scale
        return [(names[k], vals[k]) for k in sorted(vals)]
    except Exception:
        return []


def _traffic_of(substr, nth=None):
    """Traffic of the launches whose kernel name contains `substr` (the nth, or
    the mean over all of them); None when the capture holds none."""
    hits = [b for n, b in _ncu_launch_traffic() if substr in n]
    if not hits:
        return None
    if nth is not None:
        return hits[nth] if nth < len(hits) else None
    return sum(hits) / len(hits)


def gemm_sequence(gemms, dev, reps=20):
    """The layer's 12 GEMM launches as they follow each other in a stage step
    (forward QKV, proj, FC1, FC2; then per linear layer, top first, its dgrad
    and wgrad), captured once into a CUDA graph (programmatic-dependent-launch
    edges, as in the stage graphs) and replayed back to back.  Each launch
    reads inputs the others do not touch; one replay streams ~0.4 GB of
    operands and outputs, so no launch finds its inputs in the 126 MB L2 from
    the previous replay (inputs larger than L2, no flush).  Returns the mean
    sequence time and, per launch, its marginal time (sequence minus the
    sequence without that launch)."""
    import torch
    order = [0, 1, 2, 3, 4, 8, 5, 9, 6, 10, 7, 11]
    st = torch.cuda.Stream(dev)

    def graph(idx):
        with torch.cuda.stream(st):
            for i in idx:
                gemms[i][3](st.cuda_stream)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in idx:
                gemms[i][3](st.cuda_stream)
        return g

    def timed(g):
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize(dev)
        best = float("inf")
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                a.record(st)
                for _ in range(reps):
                    g.replay()
                b.record(st)
            b.synchronize()
            best = min(best, a.elapsed_time(b) / reps * 1e-3)
        return best

    full = timed(graph(order))
    marginal = {}
    for i in order:
        marginal[i] = full - timed(graph([k for k in order if k != i]))
    return full, marginal


def gemm_sequence_step_streams(gemms, dev, reps=20):
    """The same 12 launches with the stage step's stream structure
    (vit_stage.cu): forward and the data-gradient chain on the step's stream,
    each weight gradient forked onto the stage's side stream when its input
    gradient is ready (events, captured as graph edges) and joined before the
    optimizer.  Returns the mean time of one layer's 12 GEMMs as the step
    executes them."""
    import torch
    st, side = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def enqueue():
        for i in (0, 1, 2, 3):
            gemms[i][3](st.cuda_stream)
        for dg, wg in ((4, 8), (5, 9), (6, 10), (7, 11)):
            ev = torch.cuda.Event()
            ev.record(st)
            side.wait_event(ev)
            gemms[wg][3](side.cuda_stream)
            gemms[dg][3](st.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(side)
        st.wait_event(ev)

    with torch.cuda.stream(st):
        enqueue()
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        enqueue()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize(dev)
    best = float("inf")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            for _ in range(reps):
                g.replay()
            b.record(st)
        b.synchronize()
        best = min(best, a.elapsed_time(b) / reps * 1e-3)
    return best


def roofline_gemm(wl, tf_burst, hbm, dev):
    """The dominant kernel of the ViT step: the tcgen05 GEMM engine
    (gemm_tc_kernel / gemm_tc_cluster_kernel, ~55 % of the step in the ncu
    launch list).  Each of one layer's 12 GEMM launches is timed alone with
    CUDA events after an L2 flush; the engine's achieved rate is Σ algorithmic
    FLOPs / Σ launch time, against the measured bf16 peak.  Per launch the
    table also gives the bound it is held to: max(FLOPs / tensor peak,
    algorithmic bytes / HBM peak)."""
    gemms, keep = vit_layer_gemms(wl, dev)
    table, tot_fl, tot_t, tot_b = [], 0.0, 0.0, 0.0
    for name, fl, by, fn in gemms:
        dt = _time_kernel(fn, dev)
        t_roof = max(fl / (tf_burst * 1e12), by / (hbm * 1e9))
        table.append({"gemm": name, "us": round(dt * 1e6, 2), "tflops": round(fl / dt / 1e12, 1),
                      "tensor_frac": round(fl / dt / 1e12 / tf_burst, 3),
                      "bound": "tensor" if fl / (tf_burst * 1e12) >= by / (hbm * 1e9) else "hbm",
                      "roofline_frac": round(t_roof / dt, 3)})
        tot_fl += fl
        tot_t += dt
        tot_b += by
    seq_t, marg = gemm_sequence(gemms, dev)
    for i, row in enumerate(table):
        row["us_in_sequence"] = round(marg[i] * 1e6, 2)
    try:
        step_t = gemm_sequence_step_streams(gemms, dev)
    except Exception as e:  # noqa: BLE001 — auxiliary figure
        step_t = None
        print(f"[bench] step-stream GEMM sequence failed: {e}", file=sys.stderr)
    del keep
    sp = wl["spec"]
    is_vit_s = sp["dim"] == 384 and sp["image"] == 32
    # the committed ncu capture is of the ViT-S layer; other geometries get null
    traffic = _ncu_traffic("vit_layer") if is_vit_s else None
    label = "ViT-S" if is_vit_s else f"ViT (D={sp['dim']}, {sp['image']}px/{sp['patch']})"
    return {"kernel": f"gemm_tc (tcgen05 engine): the 12 GEMM launches of one {label} layer's "
                      "local step with the step's fused epilogues, in step order, replayed back "
                      "to back from one CUDA graph (PDL edges; inputs larger than L2, no flush)",
            "bound": "tensor", "achieved": tot_fl / seq_t / 1e12, "peak": tf_burst,
            "unit": "TFLOP/s", "frac": tot_fl / seq_t / 1e12 / tf_burst,
            "launch_us_in_sequence": seq_t / len(table) * 1e6,
            "in_step_streams": None if step_t is None else {
                "how": "the same 12 launches with the step's streams: forward + dgrad chain on "
                       "the step stream, each wgrad forked to the side stream (vit_stage.cu)",
                "achieved": tot_fl / step_t / 1e12, "frac": tot_fl / step_t / 1e12 / tf_burst,
                "layer_us": step_t * 1e6},
            "cold_alone": {"how": "each launch alone after a clean 512 MB L2 flush (round-1 "
                                  "method)", "achieved": tot_fl / tot_t / 1e12,
                           "frac": tot_fl / tot_t / 1e12 / tf_burst,
                           "launch_us": tot_t / len(table) * 1e6},
            "traffic": (sum(traffic) / len(traffic) if traffic and len(traffic) == len(table)
                        else None),
            "algorithmic_bytes_per_launch": tot_b / len(table),
            "algorithmic_flops_per_launch": tot_fl / len(table),
            "launch_us": seq_t / len(table) * 1e6, "launches": len(table),
            "roofline_frac_vs_max_bound": sum(
                max(fl / (tf_burst * 1e12), by / (hbm * 1e9)) for _, fl, by, _ in gemms) / seq_t,
            "per_gemm": table, "engine_calibration": engine_calibration(tf_burst, dev)}


def _graph_per_launch(fns, dev, reps=4):
    """Per-launch time of fns (callables on a stream), launched back to back
    `reps` times each from one CUDA graph (the stage graphs' PDL edges) and
    replayed on the stream the timing events bracket."""
    import torch
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        for fn in fns:
            fn(st.cuda_stream)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            for fn in fns:
                fn(st.cuda_stream)
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize(dev)
    best = float("inf")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            g.replay()
            b.record(st)
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3 / (reps * len(fns)))
    return best


def roofline_conv(wl, tf_burst, hbm, dev):
    """ResNet: the implicit-GEMM tcgen05 convolutions — the 3x3 stride-1
    forward / input-gradient conv (conv3x3_tc_kernel) and its weight gradient
    (conv3x3_wgrad_tc_kernel) — at the three CIFAR stage resolutions and the
    workload batch.  Each shape is launched back to back from one CUDA graph
    over enough input/output sets (> 160 MB together, more than the 126 MB L2)
    that every launch reads its activations from HBM; achieved = Σ algorithmic
    bytes / Σ launch time over the three resolutions (the aggregate the step
    sees), per-shape rows alongside.  HBM-bound: bytes = input + output
    activations + weights once (forward), x + dZ read + dW written (weight
    gradient); AI ≈ 9·C/2 FLOP/B is below the ridge."""
    import torch
    from paper_2411_12780_b200 import _native as N
    lib = N.load()
    B = wl["batch"]
    table, tot_t, tot_b, tot_f = [], 0.0, 0.0, 0.0
    wg_t, wg_b = 0.0, 0.0
    trs = []
    nws = lib.ppll_conv3x3_wgrad_ws_floats(B, 32, 32, 64, 64)
    ws = torch.empty(nws, device=dev)
    for C, H in zip(wl["spec"]["widths"], (32, 16, 8)):
        P = B * H * H
        nsets = max(2, int((160 << 20) // (2 * 2 * P * C)) + 1)
        sets = [(torch.randn(B, H, H, C, device=dev).bfloat16(),
                 torch.empty(B, H, H, C, device=dev, dtype=torch.bfloat16)) for _ in range(nsets)]
        w = (torch.randn(9 * C, C, device=dev) / (3 * C ** 0.5)).bfloat16()
        dw = torch.empty(9 * C, C, device=dev)
        fwd = [lambda s, x=x, y=y: lib.ppll_conv3x3_bf16(B, H, H, C, C, x.data_ptr(), w.data_ptr(),
                                                         y.data_ptr(), 0, s) for x, y in sets]
        wgr = [lambda s, x=x, y=y: lib.ppll_conv3x3_wgrad_bf16(B, H, H, C, C, x.data_ptr(),
                                                               y.data_ptr(), dw.data_ptr(),
                                                               ws.data_ptr(), nws, s)
               for x, y in sets]
        dt = _graph_per_launch(fwd, dev)
        dtw = _graph_per_launch(wgr, dev)
        fl, by = 2.0 * P * 9 * C * C, 2.0 * (2 * P * C + 9 * C * C)
        byw = 2.0 * 2 * P * C + 4.0 * 9 * C * C
        # ncu DRAM bytes of this shape (tools/traffic_probe.py captures batch 128)
        tr = _traffic_of("conv3x3_tc_kernel", len(table)) if B == 128 else None
        trs.append(tr)
        table.append({"conv": f"{C}->{C} 3x3 @ {H}x{H}, batch {B}", "us": round(dt * 1e6, 2),
                      "traffic": tr, "algorithmic_bytes": by,
                      "gbs": round(by / dt / 1e9, 1), "tflops": round(fl / dt / 1e12, 1),
                      "hbm_frac": round(by / dt / 1e9 / hbm, 3),
                      "wgrad_us": round(dtw * 1e6, 2), "wgrad_gbs": round(byw / dtw / 1e9, 1),
                      "wgrad_hbm_frac": round(byw / dtw / 1e9 / hbm, 3)})
        tot_t += dt
        tot_b += by
        tot_f += fl
        wg_t += dtw
        wg_b += byw
        del sets
    return {"kernel": "conv3x3_tc_kernel (implicit-GEMM tcgen05 conv, TMA 4-D window gathers), "
                      "the three CIFAR stage resolutions, back-to-back launches from HBM",
            "bound": "hbm", "achieved": tot_b / tot_t / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": tot_b / tot_t / 1e9 / hbm,
            "traffic": (sum(trs) / len(trs) if trs and all(t is not None for t in trs) else None),
            "traffic_source": "profiles/r02_ncu_traffic.csv (ncu dram__bytes_read.sum + "
                              "dram__bytes_write.sum per launch, caches flushed; batch 128)",
            "algorithmic_bytes_per_launch": tot_b / 3, "algorithmic_flops_per_launch": tot_f / 3,
            "tflops": tot_f / tot_t / 1e12, "launch_us": tot_t / 3 * 1e6, "per_conv": table,
            "weight_gradient": {"kernel": "conv3x3_wgrad_tc_kernel (implicit GEMM, wide split-K "
                                          "form + fixed-order reduction)",
                                "achieved": wg_b / wg_t / 1e9, "frac": wg_b / wg_t / 1e9 / hbm,
                                "launch_us": wg_t / 3 * 1e6}}


def cost_model(wl, args, dev, measured_seq_ips, measured_ips):
    """calibrate the reference's batch-time model with
    stage profiles measured on this GPU (lp.calibrate on scratch modules of
    the same workload), then simulate the PPLL schedule with one stage per
    GPU.  The single-GPU sequential schedule it implies (Σ cycles) is checked
    against the measured one; the one-stage-per-GPU prediction is what the
    N = s scaling run should approach."""
    import paper_2411_12780_b200 as lp
    mods = build(wl, args.precision, dev, 10 ** 6)
    B = wl["batch"]
    prof = lp.calibrate(mods, B)
    s = len(prof)
    r = lp.simulate_schedule(prof, lp.CommModel(0.0), "ppll", 8 * s, args.capacity)
    seq = sum(p.cycle for p in prof)
    for m in mods:
        m.close()
    return {"stage_cycle_ms": [round(p.cycle * 1e3, 4) for p in prof],
            "stage_push_ms": [round(p.f * 1e3, 4) for p in prof],
            "comm": "0 (the producer's last GEMM epilogue stores the boundary activation "
                    "into the consumer's ring slot; no separate transfer)",
            "predicted_sequential_images_per_s": B / seq,
            "measured_sequential_images_per_s": measured_seq_ips,
            "predicted_one_stage_per_gpu": {
                "n_gpus": s, "steady_batch_ms": r.steady_batch_time * 1e3,
                "images_per_s": B / r.steady_batch_time,
                "idle_fraction": [round(x, 4) for x in r.idle_fraction(s)]},
            "measured_single_gpu_pipeline_images_per_s": measured_ips}


def _guard(name, fn, *a, **k):
    """Auxiliary legs (rooflines, cost model, CPU baseline) must not take the
    bench line down with them: a failure is reported in the line instead."""
    try:
        return fn(*a, **k)
    except Exception as e:          # noqa: BLE001
        print(f"[bench] {name} failed: {type(e).__name__}: {e}", file=sys.stderr, flush=True)
        return {"error": f"{type(e).__name__}: {e}"}


def workload_from_args(args) -> dict:
    wl = dict(WORKLOADS[args.workload])
    if args.batch:
        wl["batch"] = args.batch
    if args.d_prime is not None:
        wl["d_prime"] = args.d_prime
    if args.stages:
        wl["s"] = args.stages
    if args.split:
        wl["split"] = args.split
    return wl


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="vit_s", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--capacity", type=int, default=2)
    ap.add_argument("--batch", type=int, default=0, help="override the workload batch (C5 sweep)")
    ap.add_argument("--d-prime", type=int, default=None, help="max aux depth d' (PAPER.md:271)")
    ap.add_argument("--stages", type=int, default=0, help="override the stage count (C5 sweep)")
    ap.add_argument("--split", default=None, choices=["even", "cost"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true")
    args = ap.parse_args(argv)
    args.warmup = max(3, args.warmup)
    return args


def main():
    args = parse_args()
    wl = workload_from_args(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PPLL_BENCH_SHARE_GPU") == "1":   # test hook: all ranks on cuda:0
        local = 0

    if args.impl == "reference":
        run_reference_arm(args, wl, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2411_12780_b200 as lp
    from paper_2411_12780_b200 import _native as N

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # control plane only (IPC handles, metrics); the data path is P2P
        dist.init_process_group("gloo")
        return run_sharded(args, wl, rank, world, local, dev)
    hbm, tf_burst, tf_sus, peak_kind = peaks()
    B = wl["batch"]
    ph = bench_phases(args.steps, args.warmup, wl["s"])
    mods = build(wl, args.precision, dev, step_budget(ph))
    in_shape = tuple(mods[0].in_shape)
    n_cls = mods[-1].num_classes
    cfg = lp.RunConfig(buffer_capacity=args.capacity, use_graphs=not args.no_graphs,
                       timing=True)
    pipe = lp.DevicePipeline(mods, cfg)
    gen = torch.Generator(device=dev).manual_seed(1234)
    pool_x = torch.randn((64, B) + in_shape, device=dev, generator=gen)
    pool_y = torch.randint(0, n_cls, (64, B), device=dev, generator=gen)

    def batches(k, off=0):
        for i in range(k):
            yield pool_x[(off + i) % 64], pool_y[(off + i) % 64]

    pipe.run(batches(ph["warmup"]))                   # warm-up (+ graph capture)
    before = N.launch_count()
    probe = lp.DevicePipeline(mods, lp.RunConfig(buffer_capacity=args.capacity,
                                                 use_graphs=False, timing=False))
    probe.run(batches(ph["launch_probe"], 7))
    launches_per_step = N.launch_count() - before
    torch.cuda.synchronize(dev)

    # ---- the timed region: PPLL pipeline, inputs resident in HBM ----
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        met = pipe.run(batches(ph["timed"], 11))
    torch.cuda.synchronize(dev)
    wall = met.wall_time
    value = met.images / wall
    idle = met.idle_fraction

    # ---- the sequential local-learning schedule on one stream (paper's S=1) ----
    seq = lp.DevicePipeline(mods, lp.RunConfig(buffer_capacity=args.capacity,
                                               use_graphs=not args.no_graphs, timing=False))
    cur = torch.cuda.current_stream(dev)
    seq.streams = [cur] * len(mods)
    seq.src_stream = cur
    seq.run(batches(ph["sequential_warmup"]))
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nseq = ph["sequential"]
    a.record()
    seq.run(batches(nseq, 5))
    b.record()
    b.synchronize()
    seq_ips = nseq * B / (a.elapsed_time(b) * 1e-3)

    # ---- e2e through the public API: pinned host batches ----
    rng = np.random.default_rng(7)
    host = [(torch.from_numpy(rng.standard_normal((B,) + in_shape).astype(np.float32)).pin_memory(),
             torch.from_numpy(rng.integers(0, n_cls, B)).pin_memory()) for _ in range(8)]
    # one untimed epoch first (pipeline staging / graphs are cached per module
    # set), then enough batches that the epoch's fill and drain amortise
    lp.run_epoch(lp.RunMode.PPLL, mods, (host[i % 8] for i in range(ph["e2e_warmup"])), cfg)
    e2e_steps = ph["e2e"]
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    m2 = lp.run_epoch(lp.RunMode.PPLL, mods, (host[i % 8] for i in range(e2e_steps)), cfg)
    _ = [sum(h) for h in m2.loss_history]           # losses read back (D2H)
    e2e_dt = time.perf_counter() - t0
    e2e = {"value": e2e_steps * B / e2e_dt, "unit": "images/s",
           "h2d_bytes_per_step": B * int(np.prod(in_shape)) * 4 + B * 8,
           "d2h_bytes_per_step": 4 * wl["s"],
           "api": "paper_2411_12780_b200.run_epoch(RunMode.PPLL, modules, pinned host batches)"}
    used = [m.optimizer.step_count for m in mods]
    assert max(used) <= step_budget(ph), (used, ph)

    roof_attn = None
    if wl["kind"] == "vit":
        roof = _guard("roofline_gemm", roofline_gemm, wl, tf_burst, hbm, dev)
        roof_extra = _guard("roofline_nesterov", roofline_nesterov, mods, hbm, dev)
        with ClockSampler(local) as clk_attn:   # the attention entry is latency-bound: clock-sensitive
            roof_attn = _guard("roofline_attention", roofline_attention, wl, hbm, dev)
        if isinstance(roof_attn, dict):
            roof_attn["clocks"] = clk_attn.summary()
    elif wl["kind"] == "resnet" and args.precision == "bf16":
        roof = _guard("roofline_conv", roofline_conv, wl, tf_burst, hbm, dev)
        roof_extra = _guard("roofline_nesterov", roofline_nesterov, mods, hbm, dev)
    else:
        roof = _guard("roofline_nesterov", roofline_nesterov, mods, hbm, dev)
        roof_extra = None
    if isinstance(roof, dict):
        roof["peak_kind"] = peak_kind

    cmodel = _guard("cost_model", cost_model, wl, args, dev, seq_ips, value)
    bp = _guard("backprop_baselines", backprop_baselines, wl, args, dev, batches, value)

    cpu = None
    if not args.no_cpu_baseline:
        cpu = _guard("cpu_baseline", cpu_reference, wl, 10 ** 6, warmup=1, time_budget=20.0)
        if isinstance(cpu, dict) and "value" in cpu:
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}

    line = {
        "metric": "images/sec training (device-timed) at 1/2/4/8 B200; pipeline idle fraction",
        "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic (seeded N(0,1) CIFAR-shaped inputs, "
        "uniform labels; random-init weights drawn like the reference)",
        "config": cfg_dict(wl, args) | {"parallelism": "pp-streams"},
        "idle_fraction": {"per_stage": [round(x, 4) for x in idle],
                          "mean": round(sum(idle) / len(idle), 4)},
        "sequential_schedule_images_per_s": seq_ips,
        "backprop_baselines": bp,
        "e2e": e2e, "roofline": roof, "roofline_optimizer": roof_extra,
        "roofline_attention": roof_attn,
        "cpu_baseline": cpu,
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clk.summary(),
        "staleness": {str(k): v for k, v in sorted(met.staleness.items())},
        "cost_model": cmodel,
        "step_budget": {"phases": ph, "total_steps": step_budget(ph), "used": used},
        "final_losses": [h[-1] for h in met.loss_history],
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
