"""Summarise an ncu CSV (time + DRAM bytes per launch) of one iteration by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
per = collections.defaultdict(dict)
for d in data:
    per[(d["ID"], d["Kernel Name"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, name), m in per.items():
    short = name.split("(")[0].replace("void ", "")[:48]
    a = agg[short]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tt = sum(v[1] for v in agg.values())
tb = sum(v[2] + v[3] for v in agg.values())
print(f"{sum(v[0] for v in agg.values())} launches; serialized kernel time {tt / 1e6:.3f} ms; "
      f"DRAM {tb / 1e6:.1f} MB")
print(f"{'kernel':48s} {'n':>5s} {'ms':>8s} {'share':>6s} {'DRAM MB':>9s} {'GB/s':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    mb = (v[2] + v[3]) / 1e6
    print(f"{k:48s} {v[0]:5d} {v[1] / 1e6:8.3f} {100 * v[1] / tt:5.1f}% {mb:9.1f} "
          f"{(v[2] + v[3]) / max(v[1], 1):8.1f}")
