"""Summarise an ncu launch list (gpu__time_duration + dram bytes) of N identical
hulls: per-kernel launches / time / share / DRAM bytes of the LAST hull.
    python tools/launch_summary.py launches.csv [hulls]"""
import collections
import csv
import sys

path = sys.argv[1]
hulls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
k = collections.OrderedDict()
for r in rows:
    k.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = r["Metric Value"]
items = list(k.items())
per = len(items) // hulls
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, name), m in items[len(items) - per:]:
    a = agg[name.split("(")[0].replace("void ", "")]
    a[0] += 1
    a[1] += float(m["gpu__time_duration.sum"].replace(",", ""))
    a[2] += sum(float(m.get(x, "0").replace(",", "")) for x in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s} {'GB/s':>7s}")
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:60]:60s} {a[0]:8d} {a[1]/1e6:9.3f} {a[1]/tot*100:5.1f}% {a[2]/1e9:8.3f} {a[2]/a[1]:7.1f}")
print(f"total {tot/1e6:.3f} ms over {per} launches")
