# eval: warps per CTA that start on the small boxes (the others on items)
O=gpurun_out/sw; mkdir -p $O
for spec in "w1=" "w2=-DP2P_SMALL_WARPS=2" "w0=-DP2P_SMALL_WARPS=0" "w1b="; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c3 c4-8; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
