# a1 register cap sweep + Helmholtz bench at the current code
O=gpurun_out/bin; mkdir -p $O
for spec in "base=" "m6=-DP2P_BIN_MINB=6" "m8=-DP2P_BIN_MINB=8"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for w in c5w c4-8 c3; do echo "== $name $w: $(python scripts/kprof.py $w 5 2>/dev/null | grep -E 'k_bin' | tr -s ' ')"; done
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
python scripts/bench_helmholtz.py c2a c2b > $O/bench_helmholtz.jsonl 2> $O/bench_helmholtz.err
P2P_HELM_SIMT=1 python scripts/bench_helmholtz.py c2a c2b >> $O/bench_helmholtz.jsonl 2>> $O/bench_helmholtz.err
wc -l $O/bench_helmholtz.jsonl
