# packed-FP32 k_lrt epilogue: Chebyshev parity tests, then A/B bench against the scalar build
timeout 900 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -rf -x > gpurun_out/pk_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/pk_tests.log
AB_VARIANTS="nopk" bash tools/gpu/gpu_ab.sh
