# ncu --set full (+source) of the update kernels: RTS sort (default), the Onesweep pass, a5 kernels, bin, permute
O=gpurun_out/ncua15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rs_|k_bin|k_nbr|k_boxinfo|k_scan" -c 16 \
    -o $O/rts python scripts/profile_step.py c5w 1 redundant > $O/ncu1.log 2>&1; tail -1 $O/ncu1.log
P2P_SORT=onesweep timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_radix_pass|k_restructure" -c 4 \
    -o $O/os python scripts/profile_step.py c5w 1 redundant > $O/ncu2.log 2>&1; tail -1 $O/ncu2.log
