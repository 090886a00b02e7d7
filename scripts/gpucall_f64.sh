O=gpurun_out/f64; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -k "f64 or float64 or fp64 or double or pairrec or multirank or adaptive" > $O/tests.log 2>&1; tail -3 $O/tests.log
python bench.py --precision fp64 --no-cpu-baseline --steps 10 > $O/bench_c5w_fp64.json 2> $O/bench_c5w_fp64.err
