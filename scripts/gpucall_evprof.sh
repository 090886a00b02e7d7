# ncu --set full of the REDUNDANT eval on c3 and c4-8 (tails, overheads)
O=gpurun_out/evprof; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
for w in c3 c4-8; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_eval_gravity" -c 1 \
    -o $O/ev_$w python scripts/profile_step.py $w 1 redundant > $O/ncu_$w.log 2>&1; tail -1 $O/ncu_$w.log
done
