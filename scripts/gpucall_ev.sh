# eval experiment: build, gravity parity tests, CUPTI kernel times of the REDUNDANT and INDEXED evals
O=gpurun_out/${1:-ev}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_faces.py tests/test_gpu_fullsize.py tests/test_gpu_adaptive.py tests/test_gpu_multirank.py -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in ${WLS:-c5w c4-8 c3 c4-128}; do
  echo "== $w"; python scripts/kprof.py $w 3 redundant,indexed 2>/dev/null | grep -E "eval|restruct|total"
done
