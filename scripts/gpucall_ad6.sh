O=gpurun_out/ad6; mkdir -p $O
for v in "P2P_ADAPT_CAP=0 P2P_NO_MB=1" "P2P_ADAPT_CAP=0 P2P_NO_MB=0" "P2P_ADAPT_CAP=1 P2P_NO_MB=1" "P2P_ADAPT_CAP=1 P2P_NO_MB=0"; do
 for w in c3-adaptive-t4 c3-adaptive-t16 c3-adaptive-t64; do
  for rep in 1 2; do
   echo "$v $w $(env $v timeout 300 python scripts/kprof.py $w 5 redundant,indexed 2>/dev/null | grep eval_gravity | awk '{print $1}' | tr '\n' ' ')"
  done
 done
done > $O/matrix.txt
