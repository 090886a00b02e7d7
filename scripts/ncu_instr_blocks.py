"""Where do a kernel's executed instructions go?  Splits the SASS of the first launch matching a regex (ncu source
page, --import-source on) into basic blocks and prints the blocks by executed warp-instructions, with their opcode
mix and the share of all executed instructions.  usage: python scripts/ncu_instr_blocks.py REPORT [regex] [top]"""
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
chunks = re.split(r'^"Kernel Name",', txt, flags=re.M)
body = None
for c in chunks[1:]:
    name, rest = c.split("\n", 1)
    if pat.search(name):
        body = rest
        print("kernel:", name.strip().strip('",')[:150])
        break
if body is None:
    body = txt  # single-kernel report: no per-launch header
rows = list(csv.reader(io.StringIO(body)))
h = next(r for r in rows if r and r[0] == "Address")
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
ins = []
for r in rows[rows.index(h) + 1:]:
    if len(r) <= iex or not r[ia].startswith("0x"):
        continue
    ins.append((int(r[ia], 16), r[isrc].strip(), int(float(r[iex] or 0))))
targets = set()
for a, s, _ in ins:
    m = re.search(r"BRA\S* (0x[0-9a-f]+)", s)
    if m:
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for k, (a, s, e) in enumerate(ins):
    if a in targets and cur:
        blocks.append(cur)
        cur = []
    cur.append((k, s, e))
    if re.search(r"\bBRA\b|\bEXIT\b|\bRET\b", s):
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
total = sum(e for _, _, e in ins)
print(f"executed warp-instructions: {total:.4g}")
res = []
for b in blocks:
    ex = sum(e for _, _, e in b)
    ops = {}
    for _, s, _ in b:
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    res.append((ex, b[0][0], b[-1][0], max(e for _, _, e in b), ops))
res.sort(reverse=True)
for ex, k0, k1, mx, ops in res[:top]:
    mix = " ".join(f"{o}:{n}" for o, n in sorted(ops.items(), key=lambda z: -z[1])[:9])
    print(f"[{k0:5d}-{k1:5d}] {100 * ex / total:5.1f}%  runs={mx:<10d} n={k1 - k0 + 1:<4d} {mix}")
