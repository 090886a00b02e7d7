# a1 particles in flight per thread, a3 records in flight per thread
O=gpurun_out/pu; mkdir -p $O
for spec in "base=" "bin8=-DP2P_BIN_U=8" "bin2=-DP2P_BIN_U=2" "perm8=-DP2P_PERM_U=8" "perm2=-DP2P_PERM_U=2" "base2="; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_bin|k_permute' | tr -s ' ' | tr '\n' ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
