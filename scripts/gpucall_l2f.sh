# L2 fetch-granularity hint experiment + current per-kernel times (c5w, c4-8, c3)
O=gpurun_out/l2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for w in c5w c4-8; do
  for f in none 32 64 128; do
    if [ $f = none ]; then python scripts/kprof.py $w 5 > $O/${w}_$f.txt 2>&1
    else P2P_L2_FETCH=$f python scripts/kprof.py $w 5 > $O/${w}_$f.txt 2>&1; fi
    echo "== $w $f"; cat $O/${w}_$f.txt
  done
done
timeout 600 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
