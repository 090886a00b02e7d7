# eval warps per CTA (2 x 10 CTAs vs 4 x 5) and restructure windows in flight (UNR 4 / 6 / 8)
O=gpurun_out/ewu; mkdir -p $O
for spec in "base=" "ew2=-DP2P_EV_WARPS=2" "unr6=-DP2P_RS_UNR=6" "unr8=-DP2P_RS_UNR=8" "base2="; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c3 c4-8; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity|k_restructure_gravity' | tr -s ' ' | tr '\n' ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
