# eval hot loop: S-specialised copies vs one runtime-stride loop
O=gpurun_out/hotrt; mkdir -p $O
for spec in "base=" "rt=-DP2P_EV_HOT_RT" "base2=" "rt2=-DP2P_EV_HOT_RT"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8 c3 c4-32 c4-128 c3-adaptive-t16; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
