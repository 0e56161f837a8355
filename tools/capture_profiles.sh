#!/bin/bash
# Round profile captures (run under gpurun, after the same commands exited 0 without ncu):
#   1. launch list of one bench step (per-kernel device time, warm caches as in the pipeline)
#   2. ncu --set full of the dominant fused kernel of each engine at C3, in pipeline cache state
set -e
OUT=${1:-gpurun_out}
mkdir -p $OUT
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
python tools_launches.py $OUT/launches.csv > $OUT/launch_summary.txt
python tools/prof_kaf.py C3 1 > $OUT/plain_prof.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base mangled \
    -k "regex:5k_lrtILi10ELi1" -s 2 -c 1 -o $OUT/prof_lrt python tools/prof_kaf.py C3 1 > $OUT/ncu_lrt.log 2>&1
SQNGD_ENGINE=fft ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base mangled \
    -k "regex:4k_afINS.*Li3ELi2EE" -s 1 -c 1 -o $OUT/prof_af python tools/prof_kaf.py C3 1 > $OUT/ncu_af.log 2>&1
# text summaries on the box (the .ncu-rep files are large); keep only the summaries + traffic numbers
for k in lrt af; do
  python tools_ncu.py $OUT/prof_$k.ncu-rep 1 > $OUT/prof_${k}_summary.txt 2>&1 || true
  ncu -i $OUT/prof_$k.ncu-rep --page source --csv --print-source sass > $OUT/prof_${k}_sass.csv 2>/dev/null || true
  python tools/sass_stalls.py $OUT/prof_${k}_sass.csv 40 > $OUT/prof_${k}_stalls.txt 2>&1 || true
  ncu -i $OUT/prof_$k.ncu-rep --page raw --csv > $OUT/prof_${k}_raw.csv 2>/dev/null || true
  rm -f $OUT/prof_${k}_sass.csv
done
rm -f $OUT/*.ncu-rep
