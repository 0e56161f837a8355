# round-end evidence: full GPU suite + parity record, smoke, default bench, other configs, reference arm,
# C3 step launch list (ncu, cold + serialised: shares only)
export SQNGD_PARITY_LOG=gpurun_out/parity_full.json
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/full.log 2>&1
echo "rc=$?" >> gpurun_out/full.log; tail -3 gpurun_out/full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
for cfg in C1 C2 C4 C5; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded 2>/dev/null | tail -1 >> gpurun_out/bench_configs.jsonl
done
echo "configs done"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python tools/step_loop.py C3 3 > gpurun_out/sl_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step_c3.csv python tools/step_loop.py C3 3 > gpurun_out/ncu_ll.log 2>&1
echo "ll rc=$?"
timeout 300 python tools/timeline.py C3 3 auto gpurun_out/timeline_c3.json > gpurun_out/timeline_c3.txt 2>&1; echo "tl rc=$?"
