# eval small-box path: software-pipelined source loads vs four in flight
O=gpurun_out/sp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_mbquad.py -m gpu -q -x 2>&1 | tail -1
for spec in "pipe=" "flat=-DP2P_SMALL_PIPE=0" "pipe2=" "flat2=-DP2P_SMALL_PIPE=0"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c3 c4-8; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_eval_gravity' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
