timeout 1500 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_status.py tests/test_gpu_run.py tests/test_gpu_net.py -q -p no:cacheprovider -rf -x > gpurun_out/cl_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/cl_tests.log
SQNGD_DEBUG=1 python tools/step_loop.py C3 1 2>&1 | grep sqngd: | head -2
AB_ARMS="default SQNGD_ADJ_CL=0" bash tools/gpu/gpu_ab_env.sh
timeout 300 python tools/timeline.py C3 3 auto gpurun_out/timeline_c3.json > gpurun_out/timeline_c3.txt 2>&1; echo "tl rc=$?"; sed -n 4,22p gpurun_out/timeline_c3.txt
