# round-end evidence (r02l): full GPU suite + parity record, smoke, default bench, other configs, reference
# arm, C3 step launch list (ncu, cold + serialised: shares only), device timeline, ncu --set full of the
# dominant kernel of each engine (summaries, stall mix, DRAM traffic)
OUT=gpurun_out/r02l; mkdir -p $OUT
export SQNGD_PARITY_LOG=$OUT/parity_full.json
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $OUT/gputest.log 2>&1
echo "rc=$?" >> $OUT/gputest.log; tail -3 $OUT/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 $OUT/bench_full.log > $OUT/bench_c3.json
for cfg in C1 C2 C4 C5; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded 2>/dev/null | tail -1 >> $OUT/bench_configs.jsonl
done
echo "configs done"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 $OUT/bench_ref.log > $OUT/bench_ref.json
python tools/step_loop.py C3 3 > $OUT/sl_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_step_c3.csv python tools/step_loop.py C3 3 > $OUT/ncu_ll.log 2>&1
echo "ll rc=$?"; python tools_launches.py $OUT/launches_step_c3.csv > $OUT/launch_summary_step.txt 2>&1; gzip -f $OUT/launches_step_c3.csv
timeout 300 python tools/timeline.py C3 3 auto $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1; echo "tl rc=$?"
python tools/prof_kaf.py C3 1 > $OUT/plain_prof.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base mangled \
    -k "regex:5k_lrtILi10ELi1ELb0ELi1E" -s 2 -c 1 -o $OUT/prof_lrt -f python tools/prof_kaf.py C3 1 > $OUT/ncu_lrt.log 2>&1
echo "ncu lrt rc=$?"
SQNGD_ENGINE=fft ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base mangled \
    -k "regex:4k_afINS.*Li3ELi2EE" -s 1 -c 1 -o $OUT/prof_af -f python tools/prof_kaf.py C3 1 > $OUT/ncu_af.log 2>&1
echo "ncu af rc=$?"
for k in lrt af; do
  python tools_ncu.py $OUT/prof_$k.ncu-rep 1 > $OUT/prof_${k}_summary.txt 2>&1 || true
  ncu -i $OUT/prof_$k.ncu-rep --page source --csv --print-source sass > $OUT/prof_${k}_sass.csv 2>/dev/null || true
  python tools/sass_stalls.py $OUT/prof_${k}_sass.csv 40 > $OUT/prof_${k}_stalls.txt 2>&1 || true
  ncu -i $OUT/prof_$k.ncu-rep --page raw --csv > $OUT/prof_${k}_raw.csv 2>/dev/null || true
  gzip -f $OUT/prof_${k}_raw.csv
  rm -f $OUT/prof_${k}_sass.csv $OUT/prof_$k.ncu-rep
done
du -sh gpurun_out
echo "done"
