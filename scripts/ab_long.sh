#!/bin/bash
# Same-box A/B under the power cap (experiments): alternate build variants on
# 2000-iteration probes of the bench workload (~7 s each), three rounds.
#   scripts/ab_long.sh head base ...   -> gpurun_out/abl_<v>.txt
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in "$@"; do
    lib=paper_2506_11657_b200/libtem_b200_$v.so
    [ "$v" = base ] && lib=paper_2506_11657_b200/libtem_b200.so
    TEM_LIB=$PWD/$lib timeout 300 python scripts/probe_solvers.py large-fit 1e-10 split 2000 2>&1 | grep -E "^split" | sed -E 's/iters \[[^]]*\]//' >> gpurun_out/abl_$v.txt
  done
done
for v in "$@"; do echo "== $v"; cat gpurun_out/abl_$v.txt; done
