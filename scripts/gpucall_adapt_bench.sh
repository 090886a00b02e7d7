O=gpurun_out/${1:-ab}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for w in c3 c3-adaptive-t4 c3-adaptive-t16 c3-adaptive-t64; do
  python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 > $O/bench_$w.json 2> $O/bench_$w.err
  python -c "
import json,sys
d=json.load(open('$O/bench_$w.json'))
p=d['phases']
print('$w', 'value %.3e'%d['value'], 'ms %.3f'%d['ms_per_step'], 'upd %.3f rs %.3f ev %.3f'%(p['update_a1_a5_ms'],p['restructure_ms'],p['eval_ms']), 'frac %.3f'%d['roofline']['frac'], 'red/idx kernel %.2f e2e %.2f'%(p['redundant_kernel_vs_indexed'],p['redundant_e2e_vs_indexed']), 'pairs', d['config']['pairs_per_gpu_per_step'], 'clk', d['clocks']['sm_mhz'])
" || tail -5 $O/bench_$w.err
done
