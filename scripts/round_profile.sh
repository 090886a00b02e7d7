#!/bin/bash
# One GPU call that regenerates the round's measurement artifacts under gpurun_out/$TAG/:
#   ncu --set full of the hot kernels on c5w (-> eval DRAM traffic for bench.py's roofline.traffic),
#   the default bench line, the density sweep, the reference arm, Helmholtz, and the bench's ncu launch list.
# usage: bash scripts/round_profile.sh TAG
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
ncu --set full --import-source on --clock-control none \
    -k regex:"k_eval_gravity|k_restructure_gravity|k_nbr_count|k_nbr_fill|k_radix_pass|k_permute|k_bin_gravity" -c 10 \
    -o $O/full_c5w python scripts/profile_step.py c5w 1 redundant,indexed > $O/ncu_full.log 2>&1
python - "$O" <<'PY'
import csv, io, json, subprocess, sys
o = sys.argv[1]
raw = subprocess.run(["ncu", "-i", f"{o}/full_c5w.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ki, r, w = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for row in rows[2:]:
    if "k_eval_gravity<float, (int)0" in row[ki] or "k_eval_gravity<float, 0" in row[ki]:
        t = float(row[r]) * scale[units[r]] + float(row[w]) * scale[units[w]]
        d = {"_source": "profiles/r01_ncu_full_c5w.txt: ncu --set full (scripts/round_profile.sh), "
                        "k_eval_gravity<float,REDUNDANT,4> on the c5w tile, dram__bytes_read.sum + "
                        "dram__bytes_write.sum per launch (bytes)", "c5w": int(t)}
        json.dump(d, open("profiles/ncu_eval_traffic.json", "w"), indent=1)
        json.dump(d, open(f"{o}/ncu_eval_traffic.json", "w"), indent=1)
        print("eval traffic", t)
        break
PY
python bench.py > $O/bench_c5w.json 2> $O/bench_c5w.err
for w in c4-8 c4-16 c4-32 c4-64 c4-128 c3; do
    python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python scripts/bench_helmholtz.py c2a c2b > $O/bench_helmholtz.jsonl 2> $O/bench_helmholtz.err
P2P_HELM_SIMT=1 python scripts/bench_helmholtz.py c2a c2b >> $O/bench_helmholtz.jsonl 2>> $O/bench_helmholtz.err
for w in c5s c3dense; do python bench.py --workload $w --no-cpu-baseline --steps 5 > $O/bench_$w.json 2> $O/bench_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
echo done
python scripts/bench_pairrec.py > $O/bench_pairrec.jsonl 2> $O/bench_pairrec.err
python scripts/locality_model.py > $O/locality.jsonl 2> $O/locality.err
python scripts/dist_overhead.py > $O/dist_overhead.txt 2>&1
python scripts/hbm_modes.py > $O/hbm_modes.json 2>&1
python scripts/kprof.py c5w 5 > $O/kprof_c5w.txt 2>/dev/null
