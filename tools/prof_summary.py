"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"][:70]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{len(data)} launches, {tot / 1e6:.3f} ms total")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[1] / 1e6:10.3f} ms {100 * v[1] / tot:5.1f}% {v[0]:6d} {k}")
