"""Instruction mix of the innermost MUFU loops of a kernel in libp2p.so (the eval hot loops).
usage: python scripts/sass_loop.py NAME_SUBSTRING [min_mufu]
Prints, for every backward branch whose body holds >= min_mufu MUFU instructions, the body length and opcode
counts -- the check that the hot loop holds only FFMA2/FADD2/FMUL2 + MUFU + LDS (+ loop control on the ALU pipe)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2511_21535_b200", "libp2p.so")
want = sys.argv[1]
min_mufu = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if want not in name:
        continue
    L = [re.sub(r"/\* 0x[0-9a-f]+ \*/", "", l).strip() for l in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4}\*/", l)]
    addr = [int(re.match(r"/\*([0-9a-f]+)\*/", l).group(1), 16) for l in L]
    print("==", name[:140])
    for i, l in enumerate(L):
        m = re.search(r"BRA (0x[0-9a-f]+)", l)
        if not m:
            continue
        t = int(m.group(1), 16)
        if t not in addr or addr.index(t) >= i:
            continue
        body = L[addr.index(t):i + 1]
        if sum("MUFU" in b for b in body) < min_mufu:
            continue
        ops = collections.Counter(re.sub(r"^/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?", "", b).split(" ")[0].split(".")[0]
                                  for b in body)
        print(f"  loop @{t:#x}: {len(body)} instr  " + " ".join(f"{k}:{v}" for k, v in ops.most_common()))
