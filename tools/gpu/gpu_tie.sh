# TIE flag build: full GPU suite + smoke + short C3 bench
OUT=gpurun_out/tie; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > $OUT/gputest.log 2>&1; echo "rc=$?" >> $OUT/gputest.log; tail -3 $OUT/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > $OUT/bench.log 2>&1; echo "bench rc=$?"; tail -1 $OUT/bench.log | head -c 400; echo
grep -o '"fft_engine": {"value": [0-9.]*' $OUT/bench.log
