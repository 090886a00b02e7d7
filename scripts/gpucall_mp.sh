O=gpurun_out/${1:-mp}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_abi.py -m gpu -q -x > $O/tests.log 2>&1; tail -15 $O/tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --comm ipc --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_ipc2.json 2> $O/bench_ipc2.err; echo "bench rc=$?"; tail -c 2500 $O/bench_ipc2.json; tail -5 $O/bench_ipc2.err
