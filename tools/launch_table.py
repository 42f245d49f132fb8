"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list (CSV log)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
d = collections.defaultdict(list)
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):4d} {sum(v) / 1e3:9.1f} us-tot {sum(v) / len(v) / 1e3:8.2f} us-avg  {k}")
