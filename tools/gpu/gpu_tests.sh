export SQNGD_PARITY_LOG=gpurun_out/parity_r02a.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/gputest_r02a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_r02a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02a.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 > gpurun_out/bench_r02a.log 2>&1
tail -5 gpurun_out/gputest_r02a.log
