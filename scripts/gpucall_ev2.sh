O=gpurun_out/${1:-ev2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_faces.py tests/test_gpu_adaptive.py -m gpu -q -x > $O/tests.log 2>&1; tail -2 $O/tests.log
for w in c5w c4-8 c3; do echo "== $w"; python scripts/kprof.py $w 3 redundant 2>/dev/null | grep -E "eval"; done
for w in c4-8 c3; do
  ncu --set full --import-source on --clock-control none -k regex:"k_eval_gravity" -c 1 -o $O/ev_$w python scripts/profile_step.py $w 1 redundant > $O/ncu_$w.log 2>&1
done
