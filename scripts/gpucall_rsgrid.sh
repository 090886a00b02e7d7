# restructure grid size (CTAs per SM in the launch; 4 are resident)
O=gpurun_out/rsgrid; mkdir -p $O
for spec in "g16=" "g4=-DP2P_RS_CTAS_PER_SM=4" "g8=-DP2P_RS_CTAS_PER_SM=8" "g32=-DP2P_RS_CTAS_PER_SM=32" "g16b="; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8 c3 c4-128; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_restructure_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
