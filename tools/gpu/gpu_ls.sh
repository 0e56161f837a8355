SQNGD_LSPLIT=4 timeout 600 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/ls_tests.log 2>&1; echo "ls4 tests rc=$?"; tail -1 gpurun_out/ls_tests.log
AB_ARMS="default SQNGD_LSPLIT=2 SQNGD_LSPLIT=4 SQNGD_LSPLIT=8" bash tools/gpu/gpu_ab_env.sh
