timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_status.py tests/test_gpu_run.py tests/test_gpu_net.py tests/test_gpu_chebyshev.py -q -p no:cacheprovider -rf -x > gpurun_out/rho_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/rho_tests.log
AB_ARMS="default SQNGD_RHO_ONEPASS=0" bash tools/gpu/gpu_ab_env.sh
timeout 300 python tools/timeline.py C3 3 auto gpurun_out/timeline_c3.json > gpurun_out/timeline_c3.txt 2>&1; echo "tl rc=$?"; sed -n 4,20p gpurun_out/timeline_c3.txt
