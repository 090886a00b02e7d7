# restructure build variants (c5w, c4-8): register cap, level-2 prefetch, unroll
O=gpurun_out/rsv; mkdir -p $O
for spec in "base=" "pf=-DP2P_RS_PF" "pf_u2=-DP2P_RS_PF -DP2P_RS_UNR=2" "minb3=-DP2P_RS_MINB=3" "pf_minb3=-DP2P_RS_PF -DP2P_RS_MINB=3"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep restructure)"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_fullsize.py tests/test_gpu_faces.py -m gpu -q -x 2>&1 | tail -2
