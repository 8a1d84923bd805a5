"""bench.py's contract pieces that can be checked without a GPU: the local
step budget covers every phase main() runs (round 1 shipped a budget that
was 20 steps short -> StepOutOfRange on the driver's command), the argument
overrides, and the reference arm's JSON line at the workload's real batch."""
import ast
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("steps,warmup", [(20, 5), (3, 1), (300, 10), (1, 3), (1000, 50)])
@pytest.mark.parametrize("s", [1, 4, 8])
def test_step_budget_covers_every_phase(steps, warmup, s):
    args = bench.parse_args(["--steps", str(steps), "--warmup", str(warmup)])
    ph = bench.bench_phases(args.steps, args.warmup, s)
    # what main() consumes per module, phase by phase (warmup is clamped >= 3)
    consumed = (max(3, warmup) + 1 + steps + 3 + max(10, steps // 3) + (2 * s + 2)
                + max(100, steps))
    assert sum(ph.values()) == consumed
    assert bench.step_budget(ph) >= consumed
    sp = bench.sharded_phases(args.steps, args.warmup)
    assert bench.step_budget(sp) >= max(3, warmup) + steps + max(60, steps)


def test_main_runs_only_budgeted_phases():
    """Every pipeline run in main() takes its batch count from bench_phases."""
    src = open(os.path.join(ROOT, "bench.py")).read()
    tree = ast.parse(src)
    main = next(n for n in tree.body if isinstance(n, ast.FunctionDef) and n.name == "main")
    seg = ast.get_source_segment(src, main)
    keys = set(bench.bench_phases(20, 5, 4))
    for k in keys:
        assert f'ph["{k}"]' in seg, k
    # no step count derived from args.steps outside the phase table
    assert "args.steps //" not in seg and "max(100, args.steps)" not in seg


def test_overrides():
    args = bench.parse_args(["--workload", "vit_s", "--batch", "256", "--d-prime", "2",
                             "--stages", "2"])
    wl = bench.workload_from_args(args)
    assert (wl["batch"], wl["d_prime"], wl["s"]) == (256, 2, 2)
    assert bench.WORKLOADS["vit_s"]["batch"] == 128          # not mutated
    assert sum(bench.vit_depths(wl)) == 8


def test_reference_arm_line_reports_the_real_batch():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "resnet32", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["config"]["global_batch"] == 128
    assert "batch 128" in line["cpu_baseline"]["sample"]
    assert line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["value"] > 0


def test_roofline_traffic_capture_is_committed_and_parsed():
    """The `traffic` of the attention / conv / optimizer roofline entries comes
    from the committed ncu capture (profiles/r02_ncu_traffic.csv,
    tools/traffic_probe.py): one DRAM-bytes figure per roofline kernel, equal to
    the kernel's algorithmic reads (no HBM re-reads) within 2 %."""
    rows = bench._ncu_launch_traffic()
    names = [n for n, _ in rows]
    assert any("attn_tc_fwd" in n for n in names) and any("attn_tc_bwd" in n for n in names)
    assert sum("conv3x3_tc_kernel" in n for n in names) == 3
    assert any("nesterov_kernel" in n for n in names)
    B, T, D = 128, 65, 384
    M = B * T
    fwd_reads = 2 * M * 3 * D                                   # qkv
    bwd_reads = 2 * M * 3 * D + 2 * 2 * M * D + 4 * B * 6 * T   # qkv, o, dO, lse
    assert abs(bench._traffic_of("attn_tc_fwd") / fwd_reads - 1) < 0.02
    assert abs(bench._traffic_of("attn_tc_bwd") / bwd_reads - 1) < 0.02
    for i, (C, H) in enumerate(((16, 32), (32, 16), (64, 8))):
        x_bytes = 2 * 128 * H * H * C
        assert abs(bench._traffic_of("conv3x3_tc_kernel", i) / x_bytes - 1) < 0.12
    assert abs(bench._traffic_of("nesterov_kernel") / (3 * 4 * 373056) - 1) < 0.02
