O=gpurun_out/rs2; mkdir -p $O
for v in 0 1; do
 for w in c3 c4-8 c4-64 c5w c3-adaptive-t4 c3-adaptive-t16 c3-adaptive-t64; do
  for rep in 1 2; do
   echo "static=$v $w $(P2P_RS_STATIC=$v timeout 300 python scripts/kprof.py $w 5 redundant 2>/dev/null | grep restructure | awk '{print $1}' | tr '\n' ' ')"
  done
 done
done > $O/rs.txt
timeout 900 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_adaptive_mode.py tests/test_gpu_fullsize.py -q -x --timeout 600 > $O/tests.log 2>&1; tail -3 $O/tests.log
