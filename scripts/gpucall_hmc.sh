# Helmholtz tensor-core GEMM: W multicast over clusters of 1 / 2 / 4 CTAs
O=gpurun_out/hmc; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for c in 2 4 1; do
  echo "== cluster $c"
  P2P_HELM_CLUSTER=$c timeout 600 python -m pytest tests/test_gpu_helmholtz.py -m gpu -q -x > $O/tests_$c.log 2>&1; tail -1 $O/tests_$c.log
  P2P_HELM_CLUSTER=$c timeout 300 python scripts/bench_helmholtz.py c2a c2b > $O/cl$c.jsonl 2> $O/cl$c.err
  python -c "
import json
for l in open('$O/cl$c.jsonl'):
    d=json.loads(l); print(d['workload'], 'eval_red', round(d['eval_redundant_ms'],4), 'eval_idx', round(d['eval_indexed_ms'],4), 'tf32frac', d.get('eval_frac_tf32_peak'), d['clocks']['sm_mhz'])
"
done
