# radix pass tuning after the ballot ranking: items per thread, CTAs per SM, look-back width
O=gpurun_out/rsort; mkdir -p $O
for spec in "base=" "i12=-DP2P_RS_ITEMS=12" "i20=-DP2P_RS_ITEMS=20" "i24=-DP2P_RS_ITEMS=24 -DP2P_RS_MINB=2" "mb4=-DP2P_RS_ITEMS=12 -DP2P_RS_MINB=4" "lb16=-DP2P_RS_LB=16" "i8mb6=-DP2P_RS_ITEMS=8 -DP2P_RS_MINB=6"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; tail -3 $O/build_$name.log; continue; }
  for w in c5w c4-8 c3; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'radix_pass')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
