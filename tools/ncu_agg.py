"""Aggregate an ncu --csv metrics launch list per kernel:  python tools/ncu_agg.py file.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ix["Kernel Name"]][:70]
    v = r[ix["Metric Value"]].replace(",", "")
    try:
        agg.setdefault(k, collections.defaultdict(list))[r[ix["Metric Name"]]].append(float(v))
    except ValueError:
        pass
for k, d in agg.items():
    t = d["gpu__time_duration.sum"]
    extra = "  ".join(f"{m.split('__')[-1][:28]} {sum(x) / len(x) / 1e6:8.2f}M" for m, x in d.items()
                      if m != "gpu__time_duration.sum")
    print(f"{len(t):3d} x {sum(t) / len(t):10.1f} ns  {extra}  {k}")
