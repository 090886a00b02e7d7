# eval knob sweep: item cost cap, a third small-path window (same box, base twice)
O=gpurun_out/evk2; mkdir -p $O
for spec in "base=" "cap16=-DP2P_ITEM_COSTCAP=65536ull" "cap18=-DP2P_ITEM_COSTCAP=262144ull" "s3_512=-DP2P_SMALL_NT3=3 -DP2P_SMALL_R3=512" "s2_1024=-DP2P_SMALL_NT3=2 -DP2P_SMALL_R3=1024" "base2="; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; tail -2 $O/build_$name.log; continue; }
  for w in c5w c3 c4-8 c4-32; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
