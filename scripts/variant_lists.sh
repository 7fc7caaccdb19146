#!/bin/bash
# launch lists of library build variants (experiments): scripts/variant_lists.sh v00 v11 ...
for v in "$@"; do
  TEM_LIB=paper_2506_11657_b200/libtem_b200_$v.so scripts/launch_list.sh split gpurun_out/ll_split_$v.csv
  TEM_LIB=paper_2506_11657_b200/libtem_b200_$v.so scripts/launch_list.sh two_sweep gpurun_out/ll_two_$v.csv
done
