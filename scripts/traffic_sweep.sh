#!/bin/bash
# DRAM bytes per pass for shift subsets of the bench family (experiments)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
run() {  # name, shifts, env...
  n=$1; sh=$2; shift 2
  env "$@" timeout 300 ncu --metrics $M --clock-control none -k regex:'k_(sweep|delta)' --launch-skip 10 --launch-count 4 --csv \
    python scripts/traffic_probe.py large $sh 40 > gpurun_out/tr_$n.csv 2>&1
}
run c1 0 A=1
run c3 0,1,2 A=1
run r1 10 A=1
run r4 10,11,12,13 A=1
run c10 0,1,2,3,4,5,6,7,8,9 A=1
run c10_nzc1 0,1,2,3,4,5,6,7,8,9 TEM_FORCE_NZC=1
run c10_b16 0,1,2,3,4,5,6,7,8,9 TEM_BAND=16
run c10_b4 0,1,2,3,4,5,6,7,8,9 TEM_BAND=4
