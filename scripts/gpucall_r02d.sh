set -x
O=gpurun_out/r02d; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubm scripts/ubench_evalmix.cu && /tmp/ubm > $O/ubench_evalmix.txt 2>&1
cat $O/ubench_evalmix.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
P2P_RS=legacy python scripts/kprof.py c5w 3 2>/dev/null | grep -i restruct
python scripts/kprof.py c5w 3 2>/dev/null | grep -i restruct
ncu --set full --import-source on --clock-control none -k regex:"k_restructure" -c 1 -o $O/rs_pipe python scripts/profile_step.py c5w 1 redundant > $O/ncu_pipe.log 2>&1
P2P_RS=legacy ncu --set full --import-source on --clock-control none -k regex:"k_restructure" -c 1 -o $O/rs_legacy python scripts/profile_step.py c5w 1 redundant > $O/ncu_legacy.log 2>&1
ls -la $O
