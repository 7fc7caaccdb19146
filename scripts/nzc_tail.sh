#!/bin/bash
# experiments: z-chunk count for few active slots on `large` (ms per 16-iteration graph)
mkdir -p gpurun_out
for sh in 0 0,1 0,1,2; do
  for nzc in 0 2 3 4 5 6 7 9 12; do
    if [ $nzc = 0 ]; then unset TEM_FORCE_NZC; else export TEM_FORCE_NZC=$nzc; fi
    TEM_TRACE=1 python scripts/traffic_probe.py large $sh 160 2>&1 | grep "tem trace" | tail -6 | awk -v s=$sh -v n=$nzc '{split($8,a,"="); t+=a[2]; c++; g=$5" "$6} END {printf "shifts %s force_nzc %s %s graphs %d mean_ms %.4f\n", s, n, g, c, t/c}'
  done
done
