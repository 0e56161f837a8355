# C5 evidence (SURVEY §8(d) "ncu --set full ... at C3 and C5"): step launch list, ncu of k_lrt<ADJ>, k_node, k_adj_gc
OUT=gpurun_out/r02h_c5; mkdir -p $OUT
python tools/step_loop.py C5 1 > $OUT/sl_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_step_c5.csv python tools/step_loop.py C5 1 > $OUT/ncu_ll.log 2>&1
echo "ll rc=$?"; python tools_launches.py $OUT/launches_step_c5.csv > $OUT/launch_summary_step.txt 2>&1; gzip -f $OUT/launches_step_c5.csv
python tools/prof_kaf.py C5 1 > $OUT/plain_prof.log 2>&1; echo "plain rc=$?"; cat $OUT/plain_prof.log | tail -2
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base mangled \
    -k "regex:5k_lrtILi10ELi1ELb0ELi1E" -s 2 -c 1 -o $OUT/prof_lrt -f python tools/prof_kaf.py C5 1 > $OUT/ncu_lrt.log 2>&1
echo "ncu lrt rc=$?"
ncu --set full --clock-control none --cache-control none --import-source on \
    -k "regex:^(k_node|k_adj_gc|k_adj_g)$" -s 3 -c 3 -o $OUT/prof_tails -f python tools/prof_kaf.py C5 1 > $OUT/ncu_tails.log 2>&1
echo "ncu tails rc=$?"
for k in lrt tails; do
  python tools_ncu.py $OUT/prof_$k.ncu-rep 3 > $OUT/prof_${k}_summary.txt 2>&1 || true
  ncu -i $OUT/prof_$k.ncu-rep --page raw --csv > $OUT/prof_${k}_raw.csv 2>/dev/null || true
  gzip -f $OUT/prof_${k}_raw.csv
  rm -f $OUT/prof_$k.ncu-rep
done
ncu_sass() { :; }
du -sh gpurun_out; echo done
