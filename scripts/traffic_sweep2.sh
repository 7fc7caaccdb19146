#!/bin/bash
# experiments: mass hit rate vs L2 set-aside; odd pass with own z from staging
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
run() {  # name, shifts, env...
  n=$1; sh=$2; shift 2
  env "$@" timeout 300 ncu --metrics $M --clock-control none -k regex:'k_(sweep|delta)' --launch-skip 10 --launch-count 4 --csv \
    python scripts/traffic_probe.py large $sh 40 > gpurun_out/tr_$n.csv 2>&1
}
all=0,1,2,3,4,5,6,7,8,9,10,11,12,13
run a14 $all A=1
run a14_p32 $all TEM_L2_PERSIST_MB=32
run a14_p64 $all TEM_L2_PERSIST_MB=64
run a14_z4 $all TEM_LIB=$PWD/paper_2506_11657_b200/libtem_b200_z4.so
run a14_z4b4 $all TEM_LIB=$PWD/paper_2506_11657_b200/libtem_b200_z4.so TEM_BAND=4
run a14_b4 $all TEM_BAND=4
