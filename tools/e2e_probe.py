import time, sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench, paper_2411_12780_b200 as lp
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "vit_s"]
dev = torch.device("cuda", 0)
mods = bench.build(wl, "bf16", dev, 10**6)
B = wl["batch"]
rng = np.random.default_rng(7)
shape = tuple(mods[0].in_shape)
host = [(torch.from_numpy(rng.standard_normal((B,) + shape).astype(np.float32)).pin_memory(),
         torch.from_numpy(rng.integers(0, 10, B)).pin_memory()) for _ in range(8)]
for timing in (True, False, True, False):
    cfg = lp.RunConfig(buffer_capacity=2, timing=timing)
    lp.run_epoch(lp.RunMode.PPLL, mods, (host[i % 8] for i in range(20)), cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = lp.run_epoch(lp.RunMode.PPLL, mods, (host[i % 8] for i in range(150)), cfg)
    _ = [sum(h) for h in m.loss_history]
    dt = time.perf_counter() - t0
    print("timing", timing, "e2e img/s", round(150 * B / dt))
# host-only loop cost: time the enqueue part
import cProfile, pstats
cfg = lp.RunConfig(buffer_capacity=2, timing=True)
pr = cProfile.Profile(); pr.enable()
m = lp.run_epoch(lp.RunMode.PPLL, mods, (host[i % 8] for i in range(150)), cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
