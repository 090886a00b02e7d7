O=gpurun_out/ad1; mkdir -p $O
for w in c3 c3-adaptive-t4 c3-adaptive-t16 c3-adaptive-t64; do
  echo "== $w"; timeout 300 python scripts/kprof.py $w 5 redundant,indexed 2>&1 | tail -40
done > $O/kprof.txt
