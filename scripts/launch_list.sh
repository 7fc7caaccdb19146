#!/bin/bash
# ncu launch list of a few sweep launches of a probe solve (experiments):
#   scripts/launch_list.sh <solver> <out.csv> [config]
cfg=${3:-large}
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:'k_(sweep|delta|pass1)' --launch-skip 10 --launch-count 6 --csv \
  python scripts/probe_solvers.py $cfg 1e-10 $1 40 > $2 2>&1
