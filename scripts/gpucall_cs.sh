# counting sort: new parity tests, full GPU suite, per-kernel times (count vs radix), bench
O=gpurun_out/cs; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_count_sort.py -m gpu -q -x > $O/tests_cs.log 2>&1; tail -15 $O/tests_cs.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in c5w c4-8 c3 c4-128; do echo "== $w count"; python scripts/kprof.py $w 5 2>/dev/null | grep -v Memset; echo "== $w radix"; P2P_SORT=radix python scripts/kprof.py $w 5 2>/dev/null | grep -E 'total'; done
python bench.py --no-cpu-baseline --steps 10 > $O/bench_c5w.json 2> $O/bench_c5w.err; cut -c1-300 $O/bench_c5w.json
