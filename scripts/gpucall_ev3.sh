O=gpurun_out/${1:-ev3}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_faces.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py tests/test_gpu_multiproc.py tests/test_gpu_adaptive.py -m gpu -q -x --timeout 300 > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in ${WLS:-c3 c5w c3dense c4-8 c4-64}; do t=$(python scripts/kprof.py $w 5 redundant 2>/dev/null | grep "k_eval_gravity" | awk '{print $1}'); echo "$w eval_us $t"; done
