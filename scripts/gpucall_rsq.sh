# restructure: static chunk stride vs dynamic batches of B chunks per queue atomic
O=gpurun_out/rsq; mkdir -p $O
for spec in "base=" "b4=-DP2P_RS_BATCH=4" "b8=-DP2P_RS_BATCH=8" "b16=-DP2P_RS_BATCH=16" "b32=-DP2P_RS_BATCH=32"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8 c3 c4-128 c3-adaptive-t16; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'restructure')"; done
done
P2P_NVCC_FLAGS="-DP2P_RS_BATCH=16" python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
P2P_NVCC_FLAGS="-DP2P_RS_BATCH=16" timeout 600 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_fullsize.py tests/test_gpu_faces.py -m gpu -q -x 2>&1 | tail -2
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
