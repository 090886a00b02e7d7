set -x
O=gpurun_out/r02b; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubm scripts/ubench_evalmix.cu && /tmp/ubm > $O/ubench_evalmix.txt 2>&1
cat $O/ubench_evalmix.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -5 $O/gpu_tests.log
SAN_TIMEOUT=400 bash scripts/sanitize.sh memcheck initcheck > $O/sanitize_summary.txt 2>&1
cp -r gpurun_out/sanitize $O/
tail -40 $O/sanitize_summary.txt
