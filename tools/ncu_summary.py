"""One line per kernel launch from an ncu --set full report (.ncu-rep):
duration, DRAM bytes, tensor-pipe / SM / L2 / DRAM utilisation, issue
efficiency, registers, occupancy.

usage: python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

TC_ACTIVE = "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg"
METRICS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "MB_rd", 1e-6),
    ("dram__bytes_write.sum", "MB_wr", 1e-6),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%", 1),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "issue%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
]
SCALE = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print("# " + path.split("/")[-1] + " (ncu --set full --clock-control none)")
    print("kernel | " + " | ".join(m[1] for m in METRICS) + " | tensor_active%")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").split("(")[0][:72]
        vals = []
        for key, label, mul in METRICS:
            v = d.get(key)
            if v in (None, "", "n/a"):
                vals.append("-")
                continue
            try:
                x = float(v.replace(",", "")) * SCALE.get(u.get(key, ""), 1) * mul
                vals.append(f"{x:.2f}")
            except ValueError:
                vals.append(v)
        try:   # tcgen05 pipe active cycles / elapsed SM cycles
            tc = 100.0 * float(d[TC_ACTIVE]) / float(d["sm__cycles_elapsed.avg"].replace(",", ""))
            vals.append(f"{tc:.1f}")
        except (KeyError, ValueError, ZeroDivisionError):
            vals.append("-")
        print(f"{name} | " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
