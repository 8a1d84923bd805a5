"""Per-kernel summary of an ncu launch list with duration + DRAM bytes
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv):
share of time, launches, mean us, mean MB moved, achieved GB/s.

usage: python tools/launch_bytes.py launches.csv [top]
"""
import collections
import csv
import sys

SC = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3,
      "Mbyte": 1.0, "Gbyte": 1e3}


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    per = collections.defaultdict(dict)
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * SC.get(d["Metric Unit"], 1.0)
        per[(d["ID"], d["Kernel Name"].split("(")[0][:78])][d["Metric Name"]] = v
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, k), m in per.items():
        a = agg[k]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"# {sum(a[0] for a in agg.values())} launches, {tot:.1f} us (ncu, serialised)")
    print("share  launches  avg_us   avg_MB    GB/s  kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(top)]:
        print(f"{a[1] / tot * 100:5.1f}%  {a[0]:7d}  {a[1] / a[0]:7.2f}  {a[2] / a[0]:7.2f}  "
              f"{a[2] / a[1] * 1e3:6.0f}  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
