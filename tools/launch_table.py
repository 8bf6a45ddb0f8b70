"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    try:
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
    except (ValueError, IndexError):
        pass
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{sum(v) / tot * 100:5.1f}% {len(v):4d} {sum(v) / len(v) / 1e3:9.1f} us  {k}")
