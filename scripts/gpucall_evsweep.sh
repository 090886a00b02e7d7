# eval build-option sweep: CUPTI eval times per workload for each P2P_NVCC_FLAGS variant
O=gpurun_out/${1:-evs}; mkdir -p $O
shift
for FL in "$@"; do
  tag=$(echo "$FL" | tr -c 'A-Za-z0-9=_' '_')
  P2P_NVCC_FLAGS="$FL" python -c "import __graft_entry__ as g; g.build()" > $O/build_$tag.log 2>&1 || { echo "build failed $FL"; tail -5 $O/build_$tag.log; continue; }
  for w in ${WLS:-c5w c4-8 c3}; do
    t=$(python scripts/kprof.py $w 5 redundant 2>/dev/null | grep "k_eval_gravity" | awk '{print $1}')
    echo "flags [$FL] $w eval_us $t"
  done
done
