set -x
O=gpurun_out/r02c; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubm scripts/ubench_evalmix.cu && /tmp/ubm > $O/ubench_evalmix.txt 2>&1
cat $O/ubench_evalmix.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
python scripts/kprof.py c5w 5 > $O/kprof_c5w.txt 2>$O/kprof.err; cat $O/kprof_c5w.txt; tail -3 $O/kprof.err
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -8 $O/gpu_tests.log
python bench.py > $O/bench_c5w.json 2> $O/bench_c5w.err; echo bench rc=$?
python -c "import json;d=json.load(open('$O/bench_c5w.json'));print(d['value'],d['ms_per_step'],d['phases'],d['roofline_hbm'])"
SAN_TIMEOUT=400 bash scripts/sanitize.sh memcheck initcheck > $O/sanitize_summary.txt 2>&1
cp -r gpurun_out/sanitize $O/
tail -40 $O/sanitize_summary.txt
