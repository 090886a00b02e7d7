# a1: 4 consecutive particles per thread with 16-byte loads / key stores vs the strided scalar kernel
O=gpurun_out/bv; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
for spec in "vec=" "sca=-DP2P_BIN_VEC=0" "vec2=" "sca2=-DP2P_BIN_VEC=0"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8 c3; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_bin' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
