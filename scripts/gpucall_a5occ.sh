# a5 occupancy: k_nbr_count / k_nbr_fill register caps
O=gpurun_out/a5occ; mkdir -p $O
for spec in "base=" "c3=-DP2P_NC_MINB=3" "c4=-DP2P_NC_MINB=4" "c5=-DP2P_NC_MINB=5" "f4=-DP2P_NB_MINB=4" "c4f4=-DP2P_NC_MINB=4 -DP2P_NB_MINB=4"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8 c3; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_nbr_count|k_nbr_fill' | tr -s ' ' | tr '\n' ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
