#!/bin/bash
# Generator (NEXT-2) profiles under gpurun: launch list of one C3 generator-mode step and
# ncu --set full of each generator kernel (after the same command exited 0 without ncu).
set -e
OUT=${1:-gpurun_out}
mkdir -p $OUT
python tools/step_loop.py C3 2 auto 1 > $OUT/net_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file $OUT/net_launches.csv python tools/step_loop.py C3 1 auto 1 > /dev/null 2>&1
python tools_launches.py $OUT/net_launches.csv > $OUT/net_launch_summary.txt
ncu --set full --clock-control none --cache-control none --import-source on \
    -k "regex:k_net" -s 12 -c 6 -o $OUT/prof_net python tools/step_loop.py C3 1 auto 1 > $OUT/ncu_net.log 2>&1
python tools_ncu.py $OUT/prof_net.ncu-rep 6 > $OUT/prof_net_summary.txt 2>&1 || true
ncu -i $OUT/prof_net.ncu-rep --page raw --csv > $OUT/prof_net_raw.csv 2>/dev/null || true
rm -f $OUT/prof_net.ncu-rep
