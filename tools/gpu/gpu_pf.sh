timeout 900 python -m pytest tests/test_gpu_run.py -q -p no:cacheprovider -x > gpurun_out/run_tests.log 2>&1; echo "run tests rc=$?"; tail -1 gpurun_out/run_tests.log
AB_ARMS="default lib:pf1" bash tools/gpu/gpu_ab_env.sh
