#!/bin/bash
# experiments: build variants on the small configs (plain 1e-10 solves, 3 repeats each)
mkdir -p gpurun_out
for cfg in block-fit layered-fit hetero-fit; do
  for v in "$@"; do
    lib=paper_2506_11657_b200/libtem_b200_$v.so
    [ "$v" = base ] && lib=paper_2506_11657_b200/libtem_b200.so
    for rep in 1 2 3; do
      TEM_LIB=$PWD/$lib timeout 300 python scripts/probe_solvers.py $cfg 1e-10 split 2>&1 | grep -E "^split" | sed -E "s/iters \[[^]]*\]//; s/^/$cfg $v /" >> gpurun_out/abs.log
    done
  done
done
cat gpurun_out/abs.log | cut -c1-220
