# packed complex arithmetic in the FFTs: full GPU suite, then A/B bench against the scalar build
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/cp_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/cp_tests.log
AB_VARIANTS="nocp" bash tools/gpu/gpu_ab.sh
