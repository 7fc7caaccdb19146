#!/bin/bash
# block-order band experiment: launch lists of both solvers for TEM_BAND values
for b in "$@"; do
  TEM_BAND=$b scripts/launch_list.sh split gpurun_out/ll_split_b$b.csv
  TEM_BAND=$b scripts/launch_list.sh two_sweep gpurun_out/ll_two_b$b.csv
done
