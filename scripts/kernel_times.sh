#!/bin/bash
# per-kernel device times (ncu gpu__time_duration, serialised) of one plan build + restructure + eval
# usage: bash scripts/kernel_times.sh WORKLOAD OUT.csv
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$2" python scripts/profile_step.py "$1" 1 > /dev/null 2>&1
