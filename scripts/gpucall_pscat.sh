# a3 permute as a scatter through the inverse permutation (P2P_PERMUTE_SCATTER) vs the gather
O=gpurun_out/pscat; mkdir -p $O
for spec in "base=" "scat=-DP2P_PERMUTE_SCATTER"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; tail -5 $O/build_$name.log; continue; }
  for w in c5w c4-8 c3; do echo "== $name $w"; python scripts/kprof.py $w 5 2>/dev/null | grep -E 'radix_pass|permute|total'; done
  [ $name = scat ] && P2P_NVCC_FLAGS="$flags" timeout 600 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -2
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
