# restructure fast32 rebase with FADD2 pairs vs scalar
O=gpurun_out/rsminb; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_fullsize.py tests/test_gpu_faces.py -m gpu -q -x 2>&1 | tail -1
for spec in "m0=" "m5=-DP2P_RS_MINB=5" "m6=-DP2P_RS_MINB=6" "m0b=" "m5b=-DP2P_RS_MINB=5"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c3 c4-128; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_restructure_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
