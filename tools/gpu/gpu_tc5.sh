# tcgen05 Chebyshev kernel: correctness first (short timeouts: a protocol bug would hang)
export SQNGD_PARITY_LOG=gpurun_out/parity_tc5.json
timeout 120 python -m pytest tests/test_gpu_chebyshev.py -q -x -p no:cacheprovider -k "forward_map_and_metrics and C1" > gpurun_out/tc5_a.log 2>&1
echo "rc=$?" >> gpurun_out/tc5_a.log
tail -3 gpurun_out/tc5_a.log
timeout 600 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -rf > gpurun_out/tc5_b.log 2>&1
echo "rc=$?" >> gpurun_out/tc5_b.log
tail -25 gpurun_out/tc5_b.log
