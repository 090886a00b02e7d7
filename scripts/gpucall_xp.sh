# radix ranking: XOR-accumulated digit peers vs the select form
O=gpurun_out/xp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_fullsize.py tests/test_gpu_helmholtz.py -m gpu -q -x 2>&1 | tail -1
for spec in "xor=" "sel=-DP2P_SORT_XORPEERS=0" "xor2=" "sel2=-DP2P_SORT_XORPEERS=0"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8 c3; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_radix_pass' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
