# update-kernel round: ballot sort, a1 unroll, item_size shifts, fill without acquire, restructure L2 prefetch
O=gpurun_out/v3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in c5w c4-8 c3; do echo "== $w"; python scripts/kprof.py $w 5 2>/dev/null; done
python bench.py --no-cpu-baseline --steps 10 > $O/bench_c5w.json 2> $O/bench_c5w.err; cut -c1-400 $O/bench_c5w.json
if [ -d _old ]; then (cd _old && python -c "import __graft_entry__ as g; g.build()" > ../$O/old_build.log 2>&1 && echo "== OLD fef6f4b c5w" && python scripts/kprof.py c5w 5 2>/dev/null | grep -E 'eval|restruct|total'); fi
echo "== HEAD again"; python scripts/kprof.py c5w 5 2>/dev/null | grep -E 'eval|restruct|total'
