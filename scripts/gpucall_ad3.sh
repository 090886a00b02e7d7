O=gpurun_out/ad3; mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"k_eval_gravity|k_adapt_restructure" -c 3 \
    -o $O/full_ad_t4 python scripts/profile_step.py c3-adaptive-t4 1 redundant,indexed > $O/ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_eval_gravity|k_adapt_restructure" -c 3 \
    -o $O/full_ad_t16 python scripts/profile_step.py c3-adaptive-t16 1 redundant,indexed >> $O/ncu.log 2>&1
