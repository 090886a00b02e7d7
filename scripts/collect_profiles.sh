#!/bin/bash
# Copy one scripts/round_profile.sh run (gpurun_out/$TAG) into profiles/ as the round's r01_* artifacts and
# regenerate the ncu summaries.  usage: bash scripts/collect_profiles.sh TAG
O=gpurun_out/${1:?tag}
for w in c3 c3dense c4-128 c4-16 c4-32 c4-64 c4-8 c5s c5w reference; do cp $O/bench_$w.json profiles/r01_bench_$w.json; done
cp $O/bench_helmholtz.jsonl profiles/r01_bench_helmholtz.jsonl
cp $O/bench_pairrec.jsonl profiles/r01_bench_pairrec.jsonl
cp $O/locality.jsonl profiles/r01_locality_model.jsonl
cp $O/dist_overhead.txt profiles/r01_dist_overhead.txt
cp $O/ncu_launches_bench.csv profiles/r01_ncu_launches_bench.csv
cp $O/ncu_eval_traffic.json profiles/ncu_eval_traffic.json
cp $O/kprof_c5w.txt profiles/r01_kprof_c5w.txt
cp $O/hbm_modes.json profiles/r01_hbm_modes.json
[ -f $O/gpu_tests.log ] && cp $O/gpu_tests.log profiles/r01_gpu_tests.log
python scripts/launch_table.py profiles/r01_ncu_launches_bench.csv > profiles/r01_ncu_launches_bench_summary.txt
python scripts/ncu_summary.py $O/full_c5w.ncu-rep > profiles/r01_ncu_full_c5w.txt
{ echo "# scripts/ncu_hot.py on $O/full_c5w.ncu-rep (ncu --set full --import-source on, c5w tile, scripts/round_profile.sh)"
  echo "## eval (REDUNDANT)"; python scripts/ncu_hot.py $O/full_c5w.ncu-rep "k_eval_gravity<float, \(int\)0|k_eval_gravity<float, 0" 25
  echo; echo "## restructure"; python scripts/ncu_hot.py $O/full_c5w.ncu-rep "k_restructure_gravity" 15; } > profiles/r01_ncu_source_c5w.txt 2>&1
