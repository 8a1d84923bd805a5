"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys

def main(path, top=25):
    top = int(top)
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        k = d["Kernel Name"].split("(")[0][:80]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# {len(data)} launches, {tot:.1f} us total (ncu, cold caches, serialised)")
    print("share  launches  avg_us  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{v[1] / tot * 100:5.1f}%  {v[0]:7d}  {v[1] / v[0]:7.2f}  {k}")

if __name__ == "__main__":
    main(*sys.argv[1:])
