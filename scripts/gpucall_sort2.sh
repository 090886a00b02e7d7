# sort v2 (ballot ranking, unrolled colscan) + a1 unroll: parity + per-kernel times
O=gpurun_out/sort2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_fullsize.py tests/test_gpu_faces.py tests/test_gpu_helmholtz.py -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in c5w c4-8 c3; do
  echo "== $w rts"; python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_rs|radix|total|bin|permute|scan'
  echo "== $w onesweep"; P2P_SORT=onesweep python scripts/kprof.py $w 5 2>/dev/null | grep -E 'radix|total'
done
