for w in "$@"; do python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/pf_$w.json 2>gpurun_out/pf_$w.err; done
