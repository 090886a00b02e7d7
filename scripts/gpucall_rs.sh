# restructure experiment: kprof of both kernels + the red[]-parity tests
O=gpurun_out/${1:-rs}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for w in c5w c4-8 c3; do
  echo "== $w"; P2P_RS=legacy python scripts/kprof.py $w 3 2>/dev/null | grep -i "restruct"
  python scripts/kprof.py $w 3 2>/dev/null | grep -i "restruct"
done
timeout 900 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_faces.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3
