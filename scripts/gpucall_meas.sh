O=gpurun_out/${1:-meas}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubd scripts/ubench_fp64.cu && /tmp/ubd > $O/ubench_fp64.txt 2>&1; cat $O/ubench_fp64.txt
python bench.py > $O/bench_c5w.json 2> $O/bench_c5w.err; tail -c 1500 $O/bench_c5w.json; echo
python bench.py --precision fp64 --no-cpu-baseline --steps 10 > $O/bench_c5w_fp64.json 2> $O/bench_c5w_fp64.err; tail -c 1200 $O/bench_c5w_fp64.json; tail -3 $O/bench_c5w_fp64.err
python scripts/bench_helmholtz.py c2a c2b > $O/bench_helmholtz.jsonl 2> $O/bench_helmholtz.err; cat $O/bench_helmholtz.jsonl; tail -3 $O/bench_helmholtz.err
