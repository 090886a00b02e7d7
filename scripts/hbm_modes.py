"""HBM bandwidth by access mix on this B200 (write-only fill, read-only reduction, copy), CUDA events, best of 10.
Gives the write-dominated ceiling the restructure (a6: 16 R bytes written, ~0.15 of that read) is judged against.
usage: python scripts/hbm_modes.py"""
import json

import torch

n = 1 << 30  # 4 GiB of fp32
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
a.fill_(1.0)


def best(fn, nbytes, reps=10):
    t = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        t.append(s.elapsed_time(e))
    return nbytes / (min(t) * 1e-3) / 1e9


out = {"write_only_fill_GBs": best(lambda: b.fill_(2.0), 4 * n),
       "read_only_sum_GBs": best(lambda: a.sum(), 4 * n),
       "copy_GBs(read+write)": best(lambda: b.copy_(a), 8 * n)}
print(json.dumps(out))
