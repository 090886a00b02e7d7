#!/bin/bash
# Build-variant timing on one GPU box: for each "name=FLAGS" argument, rebuild libp2p.so with P2P_NVCC_FLAGS=FLAGS
# and record the CUPTI per-kernel times of warm c5w steps (scripts/kprof.py) -> gpurun_out/variants/<name>.txt
# usage: bash scripts/variants.sh WORKLOAD "base=" "v1=-DP2P_RS_V1" ...
set -u
WL=$1; shift
O=gpurun_out/variants
mkdir -p $O
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; tail -5 $O/build_$name.log; continue; }
  P2P_NVCC_FLAGS="$flags" python scripts/kprof.py $WL 5 > $O/${WL}_$name.txt 2>&1
  echo "== $name ($flags)"; cat $O/${WL}_$name.txt
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
