#!/bin/bash
# z-chunk experiment: TEM_FORCE_NZC values vs the automatic choice (large-fit, split)
for n in auto "$@"; do
  if [ "$n" = auto ]; then unset TEM_FORCE_NZC; else export TEM_FORCE_NZC=$n; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:'k_(sweep|delta)' --launch-skip 10 --launch-count 6 --csv \
    python scripts/probe_solvers.py large-fit 1e-10 split 40 > gpurun_out/ll_nzc_$n.csv 2>&1
done
