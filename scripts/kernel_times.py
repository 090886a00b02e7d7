"""print an ncu gpu__time_duration launch list (one line per launch, us) -- companion of kernel_times.sh"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = 0.0
for r in rows[hdr + 1:]:
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    tot += v
    name = r[ki].split("(")[0].replace("void ", "").replace("p2p::", "").replace("<unnamed>::", "")
    print(f"{v:10.1f} us  {name[:90]}")
print(f"{tot:10.1f} us  total")
