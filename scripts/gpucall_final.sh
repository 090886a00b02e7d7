# final light re-measurement at the round's last code: GPU tests + smoke, default bench line, c4-8, c3, fp64, kprof
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
python bench.py > $O/bench_c5w.json 2> $O/bench_c5w.err
python bench.py --precision fp64 --no-cpu-baseline --steps 10 > $O/bench_c5w_fp64.json 2> $O/bench_c5w_fp64.err
for w in c4-8 c3; do python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
python scripts/kprof.py c5w 5 > $O/kprof_c5w.txt 2>/dev/null
python scripts/summarize_bench.py $O/bench_*.json
