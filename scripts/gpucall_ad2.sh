O=gpurun_out/ad2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_adaptive.py tests/test_gpu_adaptive_mode.py -q -x --timeout 600 > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in c3-adaptive-t4 c3-adaptive-t16 c3-adaptive-t64; do
  timeout 300 python scripts/kprof.py $w 5 redundant,indexed 2>/dev/null | grep -v Memset > $O/kprof_$w.txt
  timeout 300 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
