#!/bin/bash
# compute-sanitizer over the product kernels (VERDICT r1 missing #7); logs -> gpurun_out/sanitize/
# usage (on a GPU box): bash scripts/sanitize.sh [tools...]
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
# torch caching-allocator blocks are still cached at exit: without this memcheck reports them as leaks
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
TOOLS=${@:-memcheck racecheck synccheck initcheck}
for tool in $TOOLS; do
  for case in c1 plummer adaptive helm loopback3; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check full"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    echo "== $tool $case" 
    timeout ${SAN_TIMEOUT:-600} $CS --tool $tool $extra --error-exitcode 17 --target-processes all \
      python scripts/sanitize_cases.py $case > $OUT/${tool}_${case}.log 2>&1
    echo "rc=$?" >> $OUT/${tool}_${case}.log
    tail -3 $OUT/${tool}_${case}.log
  done
done
