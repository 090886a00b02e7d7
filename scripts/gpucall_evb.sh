# eval work items claimed per queue atomic
O=gpurun_out/evb; mkdir -p $O
for spec in "b2=" "b1=-DP2P_EV_BATCH=1" "b3=-DP2P_EV_BATCH=3" "b2b="; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c3 c4-8 c3-adaptive-t16; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
