# eval small-box path thresholds (targets <= SMALL_NT and sources <= SMALL_R: thread-per-target-pair path)
O=gpurun_out/small; mkdir -p $O
for spec in "base=" "w6_256=-DP2P_SMALL_NT2=6 -DP2P_SMALL_R2=256" "r192=-DP2P_SMALL_R=192" "base2=" "w6_256b=-DP2P_SMALL_NT2=6 -DP2P_SMALL_R2=256"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c3 c4-16; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
