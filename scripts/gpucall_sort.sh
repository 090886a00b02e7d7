# reduce-then-scan sort: parity + per-kernel times vs the Onesweep pass; bench c5w; ncu of the a1-a5 kernels
O=gpurun_out/sort; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gravity.py tests/test_gpu_fullsize.py tests/test_gpu_faces.py tests/test_gpu_helmholtz.py tests/test_gpu_multiproc.py -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
for w in c5w c4-8 c3 c4-128; do
  echo "== $w rts"; python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_rs|radix|total|bin|permute|scan'
  echo "== $w onesweep"; P2P_SORT=onesweep python scripts/kprof.py $w 5 2>/dev/null | grep -E 'radix|total'
done
python bench.py --no-cpu-baseline --steps 10 > $O/bench_c5w.json 2> $O/bench_c5w.err; cut -c1-600 $O/bench_c5w.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_nbr|k_bin|k_permute|k_rs_|k_scan|k_boxinfo" -c 12 \
    -o $O/a15 python scripts/profile_step.py c5w 1 redundant > $O/ncu.log 2>&1; tail -2 $O/ncu.log
