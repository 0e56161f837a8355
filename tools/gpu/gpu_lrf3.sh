timeout 900 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_parity.py tests/test_gpu_run.py tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/lrf_tests.log 2>&1
echo "tests rc=$?"; tail -6 gpurun_out/lrf_tests.log
bash tools/gpu/gpu_lrf2.sh | tail -2
