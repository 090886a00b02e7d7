# Helmholtz tensor-core GEMM, t = 64: outputs split over two CTAs (default) vs one CTA per tile
O=gpurun_out/hsplit; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_helmholtz.py -m gpu -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
python scripts/bench_helmholtz.py c2a c2b > $O/split.jsonl 2> $O/split.err
P2P_HELM_NSPLIT=1 python scripts/bench_helmholtz.py c2a c2b > $O/nosplit.jsonl 2> $O/nosplit.err
for f in split nosplit; do echo "== $f"; python -c "
import json,sys
for l in open('$O/$f.jsonl'):
    d=json.loads(l); print(d['workload'], 'eval_red', round(d['eval_redundant_ms'],4), 'eval_idx', round(d['eval_indexed_ms'],4), 'tf32frac', d.get('eval_frac_tf32_peak'), d['clocks']['sm_mhz'])
"; done
