# balanced k_lrt launch: Chebyshev/coverage/full-size/multirank/status GPU tests, then A/B
timeout 1200 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py tests/test_gpu_status.py tests/test_gpu_run.py -q -p no:cacheprovider -rf -x > gpurun_out/bal_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/bal_tests.log
AB_ARMS="default SQNGD_LRT_BAL=0 lib:nodepk" bash tools/gpu/gpu_ab_env.sh
