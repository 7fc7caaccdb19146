#!/bin/bash
# split-scheme launch lists for several TEM_BAND values (experiments)
for b in "$@"; do TEM_BAND=$b scripts/launch_list.sh split gpurun_out/ll_band_$b.csv; done
