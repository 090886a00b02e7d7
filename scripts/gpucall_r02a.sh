set -x
mkdir -p gpurun_out/r02a
nvidia-smi > gpurun_out/r02a/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02a/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02a/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r02a/gpu_tests.log
python bench.py > gpurun_out/r02a/bench_c5w.json 2> gpurun_out/r02a/bench_c5w.err; echo bench rc=$?
cat gpurun_out/r02a/bench_c5w.json
SAN_TIMEOUT=400 bash scripts/sanitize.sh > gpurun_out/r02a/sanitize_summary.txt 2>&1
cp -r gpurun_out/sanitize gpurun_out/r02a/ 2>/dev/null
cat gpurun_out/r02a/sanitize_summary.txt | tail -70
