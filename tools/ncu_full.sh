#!/bin/bash
# usage: tools/ncu_full.sh <g> <what> <kernel-regex> <skip> <count> <out>
g=$1; what=$2; k=$3; s=$4; c=$5; out=$6
python tools/region_driver.py $g $what > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -s $s -c $c -o gpurun_out/$out python tools/region_driver.py $g $what > gpurun_out/ncu_full_$out.log 2>&1
tail -3 gpurun_out/ncu_full_$out.log
