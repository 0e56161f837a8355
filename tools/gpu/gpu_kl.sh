timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chebyshev.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -q -p no:cacheprovider -x > gpurun_out/kl_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/kl_tests.log
AB_ARMS="default SQNGD_COMB_KL=8" bash tools/gpu/gpu_ab_env.sh
