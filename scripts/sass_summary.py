"""Per-kernel SASS opcode summary of the built libp2p.so (cuobjdump, no GPU): which kernels carry the Blackwell
data-movement / tensor instructions the design claims -- UBLKCP (1D TMA bulk copy), UTMALDG (TMA tensor load),
UTCHMMA / UTCQMMA (tcgen05.mma), LDTM / STTM (TMEM load / store), LDGSTS (cp.async), SYNCS (mbarrier),
FFMA2 / FADD2 / FMUL2 (packed FP32x2), MUFU.RSQ -- and their static counts.
usage: python scripts/sass_summary.py [libp2p.so] > profiles/r02_sass_summary.txt"""
import collections
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_2511_21535_b200/libp2p.so"
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
KEYS = ["UBLKCP", "UTMALDG", "UTMASTG", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS", "LDGSTS",
        "SYNCS", "FFMA2", "FADD2", "FMUL2", "MUFU.RSQ", "MUFU.RSQ64H", "DFMA", "SHFL", "REDUX", "MATCH", "ATOMG",
        "RED", "STG", "LDG", "LDS", "STS"]
cur, counts = None, collections.OrderedDict()
for line in txt.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        dm = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", dm.replace("p2p::", "").replace("(anonymous namespace)::", ""))[:90]
        counts.setdefault(cur, collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and cur:
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                counts[cur][k] += 1
                break
print(f"# SASS opcode summary of {so} (cuobjdump -sass; static instruction counts per kernel)")
print("# UBLKCP = cp.async.bulk (1D TMA), UTMALDG = TMA tensor load, UTCHMMA = tcgen05.mma, LDTM/STTM = TMEM access,")
print("# LDGSTS = cp.async, SYNCS = mbarrier ops, FFMA2/FADD2/FMUL2 = packed FP32x2")
for k, c in counts.items():
    if not c:
        continue
    print(f"{k}")
    print("    " + "  ".join(f"{o}:{n}" for o, n in sorted(c.items(), key=lambda z: KEYS.index(z[0]))))
