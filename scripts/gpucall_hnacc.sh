# Helmholtz tensor-core GEMM at t = 64: 3 accumulators + 2 A stages (default) vs 2 accumulators + 4 A stages
O=gpurun_out/hnacc; mkdir -p $O
for spec in "nacc3=" "nacc2=-DP2P_HELM_NACC64=2"; do
  name=${spec%%=*}; flags=${spec#*=}
  P2P_NVCC_FLAGS="$flags" python -c "from paper_2511_21535_b200 import build as B; B.build()" > $O/build_$name.log 2>&1 || { echo "build $name failed"; tail -3 $O/build_$name.log; continue; }
  echo "== $name"
  P2P_NVCC_FLAGS="$flags" timeout 600 python -m pytest tests/test_gpu_helmholtz.py -m gpu -q -x 2>&1 | tail -1
  P2P_NVCC_FLAGS="$flags" python scripts/bench_helmholtz.py c2b > $O/$name.jsonl 2> $O/$name.err
  python -c "
import json
for l in open('$O/$name.jsonl'):
    d=json.loads(l); print(d['workload'], 'eval_red', round(d['eval_redundant_ms'],4), 'eval_idx', round(d['eval_indexed_ms'],4), 'tf32frac', d.get('eval_frac_tf32_peak'), d.get('eval_rel_l2'), d['clocks']['sm_mhz'])
"
done
python -c "from paper_2511_21535_b200 import build as B; B.build()" > /dev/null 2>&1
