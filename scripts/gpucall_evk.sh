# K=8 vs K=4 eval: ncu --set full of the REDUNDANT eval on c4-128 and c5w
O=gpurun_out/${1:-evk}; mkdir -p $O
for K in 8 4; do
  P2P_NVCC_FLAGS="-DP2P_EVAL_K=$K" python -c "import __graft_entry__ as g; g.build()" > $O/build$K.log 2>&1
  for w in c4-128 c5w; do
    ncu --set full --import-source on --clock-control none -k regex:"k_eval_gravity" -c 1 -o $O/ev_K${K}_$w python scripts/profile_step.py $w 1 redundant > $O/ncu_K${K}_$w.log 2>&1
  done
done
ls $O
