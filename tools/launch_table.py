"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/launch_table.py gpurun_out/launches.csv [frames]
"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = rows[0]
iN, iV = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    try:
        v = float(r[iV].replace(",", ""))
    except ValueError:
        continue
    name = re.sub(r"\(.*", "", r[iN])
    name = re.sub(r"^void ", "", name).replace("sgs::<unnamed>::", "")[:60]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'avg us':>8s} {'us/frame':>9s} {'share':>6s}")
for k, (c, s) in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"{k:60s} {c:8d} {s / c / 1e3:8.1f} {s / frames / 1e3:9.1f} {s / tot * 100:5.1f}%")
print(f"total {tot / frames / 1e3:.1f} us/frame over {frames:g} frames")
