#!/bin/bash
# A/B of library build variants on the bench workload (experiments):
#   scripts/ab_variants.sh base ml ...      (libtem_b200_<v>.so; "base" = libtem_b200.so)
# Per variant: a timed 480-iteration probe (SUI/s, no profiler) and an ncu
# launch list with DRAM bytes of six pass launches -> gpurun_out/ab_<v>.{txt,csv}
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2506_11657_b200/libtem_b200_$v.so
  [ "$v" = base ] && lib=paper_2506_11657_b200/libtem_b200.so
  export TEM_LIB=$PWD/$lib
  for rep in 1 2; do
    timeout 300 python scripts/probe_solvers.py large-fit 1e-10 split 480 2>&1 | grep -E "^split|Error|error" >> gpurun_out/ab_$v.txt
  done
  scripts/launch_list.sh split gpurun_out/ab_$v.csv large-fit
  echo "== $v"; cat gpurun_out/ab_$v.txt
done
