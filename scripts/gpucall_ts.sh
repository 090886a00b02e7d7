# a5 fill without its in-kernel look-back (k_tile_scan, chunked): full GPU suite + per-kernel times
O=gpurun_out/ts4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in c5w c4-8 c3; do echo "== $w"; python scripts/kprof.py $w 5 2>/dev/null | grep -v xyz; done
