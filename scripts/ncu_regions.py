"""Split a kernel's warp samples into loop bodies (backward branches) vs straight-line code, from the SASS
source page of an ncu report.  usage: python scripts/ncu_regions.py REPORT kernel-regex"""
import csv
import io
import re
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2])
body = None
for c in re.split(r'^"Kernel Name",', txt, flags=re.M)[1:]:
    name, rest = c.split("\n", 1)
    if pat.search(name):
        body = rest
        break
rows = list(csv.reader(io.StringIO(body)))
h = rows[0]
I = {k: i for i, k in enumerate(h)}
recs = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    recs.append(dict(addr=int(r[I["Address"]], 16), src=r[I["Source"]].strip(),
                     s=int(r[I["Warp Stall Sampling (All Samples)"]] or 0), ex=int(r[I["Instructions Executed"]] or 0)))
addr_idx = {x["addr"]: i for i, x in enumerate(recs)}
tot = sum(x["s"] for x in recs) or 1
loops = []
for i, x in enumerate(recs):
    m = re.search(r"BRA (0x[0-9a-f]+)", x["src"])
    if m and int(m.group(1), 16) in addr_idx and addr_idx[int(m.group(1), 16)] < i:
        j = addr_idx[int(m.group(1), 16)]
        loops.append((j, i))
# innermost loops only (no other loop strictly inside)
inner = [(a, b) for (a, b) in loops if not any(a <= c and d <= b and (c, d) != (a, b) for c, d in loops)]
inloop = set()
print(f"{'loop':>14s} {'instr':>6s} {'samples':>8s} {'exec/instr':>11s}  mix")
for a, b in sorted(inner):
    s = sum(recs[k]["s"] for k in range(a, b + 1))
    ex = max(recs[k]["ex"] for k in range(a, b + 1))
    mufu = sum("MUFU" in recs[k]["src"] for k in range(a, b + 1))
    for k in range(a, b + 1):
        inloop.add(k)
    if s / tot > 0.002:
        print(f"[{a:5d}-{b:5d}] {b - a + 1:6d} {100 * s / tot:7.2f}% {ex:11d}  MUFU:{mufu}")
out = sum(x["s"] for k, x in enumerate(recs) if k not in inloop)
print(f"innermost loops total {100 * (tot - out) / tot:.2f}%   straight-line / outer {100 * out / tot:.2f}%")
