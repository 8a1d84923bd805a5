"""Top stalled SASS instructions of one kernel in an ncu report (source page),
with their dominant stall reasons.

usage: python tools/ncu_stalls.py report.ncu-rep [n]
"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, data = rows[1], rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
iall, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[iall] or 0) for r in data)
agg = {c: sum(int(r[h.index(c)] or 0) for r in data) for c in reasons}
print(f"{len(data)} SASS instructions, {tot} samples; by reason: " +
      ", ".join(f"{k[6:]} {v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v))
for i, r in sorted(enumerate(data), key=lambda ir: -int(ir[1][iall] or 0))[:n]:
    top = sorted(((int(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:3]
    why = " ".join(f"{c}:{v}" for v, c in top if v)
    print(f"{i:5d} {r[iall]:>5} x{r[iex]:>7}  {r[isrc][:60]:60s} {why}")
