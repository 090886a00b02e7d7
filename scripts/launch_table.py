"""summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel times of the last step"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
launches = []
for r in rows[hdr + 1:]:
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[r[ui]]
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    launches.append((name, v))
half = len(launches) // int(sys.argv[2]) if len(sys.argv) > 2 else 0
last = launches[-half:] if half else launches
agg = OrderedDict()
for n, v in last:
    agg[n] = agg.get(n, 0) + v
tot = sum(agg.values())
for n, v in agg.items():
    print(f"{v:10.1f} us {100 * v / tot:5.1f}%  {n[:100]}")
print(f"{tot:10.1f} us total, {len(last)} launches")
