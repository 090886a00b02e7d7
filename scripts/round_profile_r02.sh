#!/bin/bash
# Round-2 measurement call (one gpurun): GPU tests + smoke, compute-sanitizer (4 tools), ncu --set full of the hot
# kernels on c5w (eval REDUNDANT / INDEXED, restructure, sort, permute, a5) and of the tensor-core Helmholtz GEMM
# (both layouts, c2b), the bench lines (default c5w with cpu_baseline, fp64, the density sweep, c3 grid + adaptive,
# c5s, c3dense, reference arm, 2-process IPC on one GPU), Helmholtz, locality model, pair records, kernel split,
# the bench's ncu launch list.  usage: bash scripts/round_profile_r02.sh TAG
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
python bench.py > $O/bench_c5w.json 2> $O/bench_c5w.err
python bench.py --precision fp64 --no-cpu-baseline --steps 10 > $O/bench_c5w_fp64.json 2> $O/bench_c5w_fp64.err
for w in c4-8 c4-16 c4-32 c4-64 c4-128 c3 c3-adaptive-t4 c3-adaptive-t16 c3-adaptive-t64 c3dense; do
    python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
done
python bench.py --workload c5s --no-cpu-baseline --steps 5 > $O/bench_c5s.json 2> $O/bench_c5s.err
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus 2 --comm ipc --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_ipc2.json 2> $O/bench_ipc2.err
python scripts/bench_helmholtz.py c2a c2b > $O/bench_helmholtz.jsonl 2> $O/bench_helmholtz.err
P2P_HELM_SIMT=1 python scripts/bench_helmholtz.py c2a c2b >> $O/bench_helmholtz.jsonl 2>> $O/bench_helmholtz.err
python scripts/bench_pairrec.py > $O/bench_pairrec.jsonl 2> $O/bench_pairrec.err
python scripts/locality_model.py > $O/locality.jsonl 2> $O/locality.err
python scripts/kprof.py c5w 5 > $O/kprof_c5w.txt 2>/dev/null
ncu --set full --import-source on --clock-control none \
    -k regex:"k_eval_gravity|k_restructure_gravity|k_nbr_count|k_nbr_fill|k_radix_pass|k_permute|k_bin_gravity" -c 10 \
    -o $O/full_c5w python scripts/profile_step.py c5w 1 redundant,indexed > $O/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_helm_tc" -c 2 \
    -o $O/full_helm_tc python scripts/helm_prof.py c2b > $O/ncu_helm.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
# compute-sanitizer: closed on the GPU pool since late round 2 (runs refused); profiles/r02_sanitize_summary.txt is
# the earlier clean run -- re-enable with RUN_SANITIZE=1 where the tool is available
if [ "${RUN_SANITIZE:-0}" = 1 ]; then
  SAN_TIMEOUT=500 bash scripts/sanitize.sh > $O/sanitize_run.txt 2>&1
  cp -r gpurun_out/sanitize $O/
fi
echo done
