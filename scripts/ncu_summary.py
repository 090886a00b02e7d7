"""Summarise an ncu --set full report (one row per captured launch): duration, throughput, pipes, DRAM bytes."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
idx = {w: h.index(w) for w in want if w in h}
out = []
for r in rows[2:]:
    d = {w: r[i] for w, i in idx.items()}
    out.append(d)
    name = d.get("Kernel Name", "")[:70]
    print(f"== {name}")
    for w in want[1:]:
        if w in idx:
            print(f"   {w} = {d[w]} {u[idx[w]]}")
