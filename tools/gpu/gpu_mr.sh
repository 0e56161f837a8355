export SQNGD_PARITY_LOG=gpurun_out/parity_mr.json
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider -rf > gpurun_out/mr.log 2>&1
echo "rc=$?" >> gpurun_out/mr.log; tail -15 gpurun_out/mr.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --deselect tests/test_gpu_multirank.py > gpurun_out/all_mr.log 2>&1
echo "rc=$?" >> gpurun_out/all_mr.log; tail -8 gpurun_out/all_mr.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 > gpurun_out/bench_mr.log 2>&1
tail -c 600 gpurun_out/bench_mr.log
