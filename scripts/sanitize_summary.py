"""Summarise scripts/sanitize.sh logs: per (tool, case) the sanitizer's error count split into
  * product errors  -- every reported hazard / invalid access / uninitialised read, and leaks whose allocation
                       backtrace passes through libp2p.so (the library's own allocations);
  * driver leaks    -- blocks still referenced by the Python test driver's torch tensors at exit (allocation
                       backtrace in torch's CUDACachingAllocator / at::empty, never in libp2p.so).
usage: python scripts/sanitize_summary.py gpurun_out/sanitize > profiles/r02_sanitize_summary.txt"""
import glob
import os
import re
import sys


def blocks(text):
    """split a compute-sanitizer log into its reported records: a record starts at a top-level line (one space
    after the '=========' prefix) and collects the indented lines after it"""
    out, cur = [], []
    for line in text.splitlines():
        if not line.startswith("========="):
            continue
        body = line[len("========="):]
        if body.strip() == "":
            continue
        if body.startswith(" ") and not body.startswith("  "):
            if cur:
                out.append(cur)
            cur = [body]
        elif cur:
            cur.append(body)
    if cur:
        out.append(cur)
    return out


def main(d):
    rows = []
    for f in sorted(glob.glob(os.path.join(d, "*.log"))):
        tool, case = os.path.basename(f)[:-4].split("_", 1)
        text = open(f, errors="replace").read()
        summ = re.findall(r"ERROR SUMMARY: (\d+) error", text) or \
            re.findall(r"RACECHECK SUMMARY: (\d+) hazard", text)
        total = int(summ[-1]) if summ else -1
        rc = re.findall(r"^rc=(\d+)", text, re.M)
        done = f"case {case} done" in text
        recs = blocks(text)
        leaks_driver = leaks_lib = other = 0
        kinds = {}
        for r in recs:
            head = r[0].strip()
            if head.startswith("Leaked"):
                if any("libp2p.so" in x for x in r):
                    leaks_lib += 1
                else:
                    leaks_driver += 1
            elif head.startswith(("LEAK SUMMARY", "ERROR SUMMARY", "COMPUTE-SANITIZER", "RACECHECK SUMMARY")):
                continue
            elif any(head.startswith(k) for k in ("Uninitialized", "Invalid", "Race", "Barrier", "Program hit",
                                                  "Error", "Malloc", "Warning", "Cuda API", "Potential")):
                other += 1
                key = head.split(" at ")[0][:60]
                kinds[key] = kinds.get(key, 0) + 1
        rows.append((tool, case, total, other, leaks_lib, leaks_driver, done, rc[-1] if rc else "?", kinds))
    print("# compute-sanitizer over libp2p (scripts/sanitize.sh, scripts/sanitize_cases.py), summarised by "
          "scripts/sanitize_summary.py")
    print("# product = hazards / invalid or uninitialised accesses / libp2p-allocated leaks; driver leaks = the "
          "Python driver's torch tensors still referenced at exit (not library memory)")
    print(f"{'tool':10s} {'case':10s} {'sanitizer errors':>16s} {'product':>8s} {'lib leaks':>9s} "
          f"{'driver leaks':>12s} {'case ran':>8s}")
    for t, c, tot, oth, ll, ld, done, rc, kinds in rows:
        print(f"{t:10s} {c:10s} {tot:16d} {oth:8d} {ll:9d} {ld:12d} {str(done):>8s}")
        for k, v in kinds.items():
            print(f"{'':22s} {v:6d} x {k}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sanitize")
