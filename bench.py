"""PPLL throughput benchmark (BASELINE.json metric: images/sec training,
device-timed, at 1/2/4/8 B200, plus the pipeline idle fraction).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One "step" = one synthetic batch pushed through every stage's local step
(forward -> push -> aux -> softmax-CE -> backward -> cosine-LR Nesterov).
``value`` is device-timed (CUDA events) with inputs already resident in HBM
(a 64-batch pool cycled so the working set exceeds the 126 MB L2); ``e2e``
is the same metric through the public API (``run_epoch`` on host numpy
batches: pinned staging + H2D inside the timed region, loss history D2H).
``--impl reference`` times the reference algorithm's CPU path (the numpy
oracle port, oracle/ppll_oracle.py) on the host cores.

Multi-GPU (torchrun, one rank per GPU): round 1 runs independent replicas of
the whole stage pipeline per GPU ("replicas", weak scaling); the NVLink
stage-sharded pipeline is the next milestone.
"""
from __future__ import annotations

import argparse
import json
import math
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
    # the reference-runnable CIFAR-shaped MLP analog (SURVEY §8 'M'): 4 stages,
    # d'=2, n=3, B=128; inputs 3072 = 3x32x32
    "mlp_m": dict(dims=(3072, 1024, 1024, 1024, 1024, 10), s=4, d_prime=2, interval=3,
                  batch=128),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

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


# ---------------------------------------------------------------------------
# the reference arm / CPU baseline: the oracle port on host cores
# ---------------------------------------------------------------------------

def cpu_reference(wl, n_batches, warmup=1, time_budget=None):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ppll_oracle as orc
    dims = wl["dims"]
    bnd = orc.partition(dims, wl["s"])
    stages = orc.build_stages(dims, bnd, wl["d_prime"], wl["interval"], 42)
    rng = np.random.default_rng(0)
    B = wl["batch"]
    data = [(rng.standard_normal((B, dims[0])), rng.integers(0, dims[-1], B))
            for _ in range(4)]
    T = 10 ** 6
    for i in range(warmup):
        orc.sequential_ppll(stages, [data[i % 4]], 0.05, 0.001, T, 0.9, 1e-4)
    t0 = time.perf_counter()
    done = 0
    per_step = []
    for i in range(n_batches):
        ts = time.perf_counter()
        orc.sequential_ppll(stages, [data[i % 4]], 0.05, 0.001, T, 0.9, 1e-4)
        per_step.append(time.perf_counter() - ts)
        done += 1
        if time_budget and time.perf_counter() - t0 > time_budget:
            break
    dt = time.perf_counter() - t0
    return done * B / dt, done, dt, per_step


def run_reference_arm(args, wl, rank, world):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    ips, done, dt, per = cpu_reference(wl, args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": "images/sec training (PPLL local-learning step, "
        "all stages, sequential schedule)", "value": ips, "unit": "images/s",
        "n_gpus": args.gpus, "steps": done, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / max(done, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg_dict(wl, args),
        "cpu_baseline": {"value": ips, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": f"{done} batches of {wl['batch']} images through all "
                                   f"{wl['s']} stages (numpy fp64 oracle, BLAS threads = "
                                   f"all {cores} cores)"},
        "e2e": {"value": ips, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cfg_dict(wl, args):
    return {"workload": f"{args.workload}: PPLL MLP {'-'.join(map(str, wl['dims']))}, "
                        f"{wl['s']} gradient-isolated stages, d'={wl['d_prime']}, "
                        f"n={wl['interval']}, CIFAR-shaped 3x32x32 inputs",
            "global_batch": wl["batch"] * max(1, args.gpus), "stages": wl["s"],
            "buffer_capacity": args.capacity, "precision": args.precision,
            "placement": "all stages on each GPU (replicas)" if args.gpus > 1 else
                         "all stages on one GPU, one CUDA stream per stage",
            "l2": "no flush; per-step working set (64-batch input pool 100 MB + "
                  "params/momenta/grads ~190 MB) exceeds the 126 MB L2"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def build(wl, precision, device, total_steps):
    import paper_2411_12780_b200 as lp
    spec = lp.NetworkSpec(wl["dims"])
    plan = lp.partition(spec, wl["s"])
    hyper = lp.Hyperparams(lr0=0.05, lr_min=0.001, total_steps=total_steps, seed=42,
                           precision=precision)
    return lp.build_modules(spec, plan, wl["d_prime"], wl["interval"], hyper,
                            devices=[device] * wl["s"])


def dominant_kernel_roofline(mods, B, hbm, stream_dev):
    """Time the step's dominant kernel (the fused Nesterov update of the
    largest stage; see profiles/) with CUDA events on its launching stream,
    over R launches on the live stage buffers."""
    import torch
    from paper_2411_12780_b200 import _native as N
    m = max(mods, key=lambda mm: mm._flat["theta"].numel())
    f = m._flat
    n = f["theta"].numel()
    lib = N.load()
    st = torch.cuda.current_stream(stream_dev)
    g = torch.zeros_like(f["grad"])
    th, v = f["theta"].clone(), f["mom"].clone()
    lp_buf = f["theta_lp"].clone() if f["theta_lp"] is not None else None
    R = 20
    flush = torch.empty(64 << 20, dtype=torch.float32, device=stream_dev)   # 256 MB > L2
    for _ in range(3):
        lib.ppll_nesterov_step(n, th.data_ptr(), v.data_ptr(), g.data_ptr(), N.ptr(lp_buf),
                               None, None, 0, 0.0, 0.9, 1e-4, None, st.cuda_stream)
    times = []
    for _ in range(R):
        flush.zero_()                      # evict the operands from L2 between launches
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        lib.ppll_nesterov_step(n, th.data_ptr(), v.data_ptr(), g.data_ptr(), N.ptr(lp_buf),
                               None, None, 0, 0.0, 0.9, 1e-4, None, st.cuda_stream)
        b.record(st)
        b.synchronize()
        times.append(a.elapsed_time(b))
    dt = statistics.median(times) * 1e-3
    per_param = 20 + (2 if lp_buf is not None else 0)
    bytes_ = n * per_param
    return {"kernel": "nesterov_kernel (fused Nesterov-SGD, largest stage)",
            "bound": "hbm", "achieved": bytes_ / dt / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": bytes_ / dt / 1e9 / hbm, "traffic": None,
            "algorithmic_bytes_per_launch": bytes_, "params": n,
            "bytes_per_param": per_param, "launch_us": dt * 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mlp_m", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--capacity", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, wl, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2411_12780_b200 as lp
    from paper_2411_12780_b200 import _native as N

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    hbm, tf_burst, tf_sus, peak_kind = peaks()
    B = wl["batch"]
    total = args.warmup + 2 * args.steps + 8
    mods = build(wl, args.precision, dev, total)
    cfg = lp.RunConfig(buffer_capacity=args.capacity, use_graphs=not args.no_graphs,
                       timing=True)
    pipe = lp.DevicePipeline(mods, cfg)
    # resident synthetic pool: 64 CIFAR-shaped batches in HBM
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    pool_x = torch.randn(64, B, wl["dims"][0], device=dev, generator=gen)
    pool_y = torch.randint(0, wl["dims"][-1], (64, B), device=dev, generator=gen)

    def batches(k, off=0):
        for i in range(k):
            yield pool_x[(off + i) % 64], pool_y[(off + i) % 64]

    pipe.run(batches(args.warmup))                    # warm-up (graph capture)
    # kernels launched per step (graph replays launch the same sequence)
    before = N.launch_count()
    for j, m in enumerate(mods):
        pass
    probe = lp.DevicePipeline(mods, lp.RunConfig(buffer_capacity=args.capacity,
                                                 use_graphs=False, timing=False))
    probe.run(batches(1, 7))
    launches_per_step = N.launch_count() - before
    torch.cuda.synchronize(dev)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        met = pipe.run(batches(args.steps, 11))
    torch.cuda.synchronize(dev)
    wall = met.wall_time
    if world > 1:
        t = torch.tensor([wall], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
        dist.barrier()
    images = met.images * world
    value = images / wall
    idle = met.idle_fraction

    # ---- sequential local-learning schedule on one stream (paper's S=1) ----
    seq_cfg = lp.RunConfig(buffer_capacity=args.capacity, use_graphs=False, timing=False)
    seq = lp.DevicePipeline(mods, seq_cfg)
    seq.streams = [torch.cuda.current_stream(dev)] * len(mods)
    seq.src_stream = torch.cuda.current_stream(dev)
    seq.run(batches(3))
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nseq = max(10, args.steps // 4)
    a.record()
    seq.run(batches(nseq, 5))
    b.record()
    b.synchronize()
    seq_ips = nseq * B / (a.elapsed_time(b) * 1e-3)

    # ---- e2e through the public API: host numpy batches ----
    rng = np.random.default_rng(7 + rank)
    host = [(rng.standard_normal((B, wl["dims"][0])).astype(np.float32),
             rng.integers(0, wl["dims"][-1], B)) for _ in range(8)]
    e2e_steps = max(10, args.steps // 2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    m2 = lp.run_epoch(lp.RunMode.PPLL, mods, (host[i % 8] for i in range(e2e_steps)), cfg)
    _ = [sum(h) for h in m2.loss_history]           # losses are read back (D2H)
    e2e_dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_dt = float(t.item())
    e2e = {"value": e2e_steps * B * world / e2e_dt, "unit": "images/s",
           "h2d_bytes_per_step": B * wl["dims"][0] * 4 + B * 8,
           "d2h_bytes_per_step": 4 * wl["s"],
           "api": "paper_2411_12780_b200.run_epoch(RunMode.PPLL, modules, host numpy batches)"}

    roof = dominant_kernel_roofline(mods, B, hbm, dev)
    roof["peak_kind"] = peak_kind

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ips, done, dt, _ = cpu_reference(wl, 200, warmup=1, time_budget=15.0)
        cpu = {"value": ips, "unit": "images/s", "cores": len(os.sched_getaffinity(0)),
               "kind": "port",
               "sample": f"{done} batches x {B} images, all {wl['s']} stages, sequential "
                         f"schedule, numpy fp64 oracle ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": "images/sec training (device-timed) at 1/2/4/8 B200; pipeline idle fraction",
            "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic (seeded N(0,1) CIFAR-shaped inputs, "
            "uniform labels; random-init weights drawn like the reference)",
            "config": cfg_dict(wl, args) | {"parallelism": f"replicas{world}" if world > 1
                                            else "pp-streams"},
            "idle_fraction": {"per_stage": [round(x, 4) for x in idle],
                              "mean": round(sum(idle) / len(idle), 4)},
            "sequential_schedule_images_per_s": seq_ips,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
            "staleness": {str(k): v for k, v in sorted(met.staleness.items())},
            "final_losses": [h[-1] for h in met.loss_history],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
