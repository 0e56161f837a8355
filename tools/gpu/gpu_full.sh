# full GPU suite + smoke + default bench (round-end equivalent)
export SQNGD_PARITY_LOG=gpurun_out/parity_full.json
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/full.log 2>&1
echo "rc=$?" >> gpurun_out/full.log; tail -6 gpurun_out/full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -c 300 gpurun_out/bench_full.log
