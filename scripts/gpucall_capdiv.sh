# eval item cost cap: items per nominal warp the work-scaled cap aims at
O=gpurun_out/capdiv; mkdir -p $O
for spec in "d4=-DP2P_CAP_DIV=4" "d2=-DP2P_CAP_DIV=2" "d1=-DP2P_CAP_DIV=1" "d8="; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c3 c4-8 c3-adaptive-t16 c3-adaptive-t4 c5w; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
