"""Where does a kernel spend its warp samples?  Reads the SASS source page of an ncu --set full report
(--import-source on) for the first launch whose name matches a regex and prints
  * the sample share of each contiguous block (split at branch targets/branches), with its instruction mix;
  * the top instructions by samples with their dominant stall reasons;
  * executed-instruction counts per opcode class.
usage: python scripts/ncu_hot.py REPORT.ncu-rep [kernel-regex] [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
# the page holds one table per launch, each preceded by a "Kernel Name" line
chunks = re.split(r'^"Kernel Name",', txt, flags=re.M)
body = None
for c in chunks[1:]:
    name, rest = c.split("\n", 1)
    if pat.search(name):
        body = rest
        print("kernel:", name.strip().strip('",')[:160])
        break
if body is None:
    sys.exit("no launch matches")
rows = list(csv.reader(io.StringIO(body)))
h = rows[0]
I = {k: h.index(k) for k in h}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
recs = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    src = r[I["Source"]].strip()
    recs.append(dict(src=src, op=src.split()[0] if src else "", s=int(r[I["Warp Stall Sampling (All Samples)"]] or 0),
                     ex=int(r[I["Instructions Executed"]] or 0),
                     st={k: int(r[I[k]] or 0) for k in stalls}))
tot = sum(x["s"] for x in recs) or 1
print(f"instructions {len(recs)}  samples {tot}")


def opclass(src):
    s = re.sub(r"^@!?U?P\w+\s+", "", src)
    return s.split()[0].split(".")[0] if s else ""


# blocks: split after every branch / before every instruction following one
blocks, cur = [], []
for i, x in enumerate(recs):
    cur.append((i, x))
    if re.search(r"\bBRA\b|\bEXIT\b|\bRET\b|BSYNC", x["src"]):
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
print("\n-- blocks with >= 1% of samples --")
for b in blocks:
    s = sum(x["s"] for _, x in b)
    if s / tot < 0.01:
        continue
    mix = collections.Counter(opclass(x["src"]) for _, x in b)
    ex = max(x["ex"] for _, x in b)
    print(f"[{b[0][0]:5d}-{b[-1][0]:5d}] {100 * s / tot:5.1f}%  n={len(b):3d} exec={ex:>10d}  " +
          " ".join(f"{k}:{v}" for k, v in mix.most_common(8)))
print(f"\n-- top {top} instructions --")
for i, x in sorted(enumerate(recs), key=lambda t: -t[1]["s"])[:top]:
    st = sorted(x["st"].items(), key=lambda t: -t[1])[:3]
    print(f"{i:5d} {100 * x['s'] / tot:5.1f}%  {x['src'][:60]:60s} " +
          " ".join(f"{k[6:]}={v}" for k, v in st if v))
tot_st = collections.Counter()
for x in recs:
    tot_st.update(x["st"])
print("\n-- stall reasons --")
print(" ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in tot_st.most_common(10)))
ex = collections.Counter()
for x in recs:
    ex[opclass(x["src"])] += x["ex"]
print("\n-- executed warp instructions by opcode --")
print(" ".join(f"{k}:{v:.3g}" for k, v in ex.most_common(24)))

# lane utilisation of the MUFU-heavy blocks: thread instructions / (32 * warp instructions)
print("\n-- lane utilisation (thread-inst / 32 warp-inst) of blocks with MUFU --")
for b in blocks:
    idxs = [i for i, _ in b]
    if not any("MUFU" in recs[i]["src"] for i in idxs):
        continue
    wi = sum(recs[i]["ex"] for i in idxs)
    ti = sum(int(rows[1 + i][I["Thread Instructions Executed"]] or 0) for i in idxs)
    s = sum(recs[i]["s"] for i in idxs)
    if wi:
        print(f"[{idxs[0]:5d}-{idxs[-1]:5d}] samples {100 * s / tot:5.1f}%  lanes/warp-inst {ti / wi:5.2f}")
