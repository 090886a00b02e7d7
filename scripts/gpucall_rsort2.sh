# radix pass: larger tiles with dynamic shared staging
O=gpurun_out/rsort2; mkdir -p $O
for spec in "i20=-DP2P_RS_ITEMS=20" "i24m2=-DP2P_RS_ITEMS=24 -DP2P_RS_MINB=2" "i32m2=-DP2P_RS_ITEMS=32 -DP2P_RS_MINB=2"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; tail -3 $O/build_$name.log; continue; }
  for w in c5w c4-8 c3; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'radix_pass')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_helmholtz.py -m gpu -q -x 2>&1 | tail -2
