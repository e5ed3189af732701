"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= mi:
        continue
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "")
    v = float(r[mi].replace(",", ""))
    v *= {"usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{k:40s} {v[0]:7d} {v[1] / 1e6:9.2f} ms  avg {v[1] / v[0] / 1e3:8.2f} us")
print("total", round(tot / 1e6, 3), "ms")
