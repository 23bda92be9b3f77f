"""Aggregate an ncu --metrics gpu__time_duration.sum CSV: per-kernel launches and time.
  python tools/launches.py launches.csv [first_launch_index] [last]"""
import csv, collections, sys
rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
r = list(csv.DictReader(rows))
r = [x for x in r if x.get("Metric Name") == "gpu__time_duration.sum"]
a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = int(sys.argv[3]) if len(sys.argv) > 3 else len(r)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for x in r[a:b]:
    k = x["Kernel Name"].split("(")[0].replace("void ", "")
    v = float(x["Metric Value"].replace(",", "")) * scale[x["Metric Unit"]]
    agg[k][0] += 1
    agg[k][1] += v
    agg[k][2] = max(agg[k][2], v)
tot = sum(v[1] for v in agg.values())
print(f"{len(r[a:b])} launches, {tot/1e3:.3f} ms kernel time")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:34s} {v[0]:5d} {v[1]/1e3:9.3f} ms {100*v[1]/tot:5.1f}%  max {v[2]:9.1f} us")
